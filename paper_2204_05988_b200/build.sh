#!/bin/bash
# Build libsg.so for sm_100a (B200).  Usage: build.sh [extra nvcc flags]
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
cd "$HERE/csrc"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $*"
OBJS=""
PIDS=""
for f in mesh assemble kernels xfanin xfanin_tma vmoment d1fused setup solver strip_solver api; do
  $NVCC $FLAGS -dc -o "$f.o" "$f.cu" &
  PIDS="$PIDS $!"
  OBJS="$OBJS $f.o"
done
for p in $PIDS; do wait $p; done   # set -e: any failed compile aborts the build
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$HERE/libsg.so" $OBJS -lcudart
rm -f $OBJS
echo "built $HERE/libsg.so"
# measured fp64 peaks (the roofline denominator bench.py reports against)
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -o "$HERE/../tools/fp64_peak" "$HERE/../tools/fp64_peak.cu"
echo "built tools/fp64_peak"
