mkdir -p gpurun_out/dbg
cd $GRAFT_REPO_ROOT
for env in "" "SG_SERIAL_CROSS=1" "SG_SERIAL_APPLIES=1" "SG_SERIAL_CROSS=1 SG_SERIAL_APPLIES=1" "SG_NO_GRAPHS=1"; do
  echo "== $env" >> gpurun_out/dbg/out.log
  env $env timeout 120 python tools/repro_solve.py c0_2d_const 6 >> gpurun_out/dbg/out.log 2>&1; echo "rc=$?" >> gpurun_out/dbg/out.log
done
timeout 300 /usr/local/cuda/bin/cuda-gdb -batch -ex run -ex bt --args python tools/repro_solve.py c0_2d_const 6 > gpurun_out/dbg/gdb.log 2>&1
