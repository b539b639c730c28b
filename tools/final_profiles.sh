# end-of-round evidence: full GPU tests, bench lines of all configs, DRAM traffic, ncu --set full of the
# top kernels, ncu launch list of the bench command.  usage: tools/final_profiles.sh OUTDIR
O=${1:-gpurun_out/final}
mkdir -p $O
if [ "$2" = "bench" ]; then
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python tools/apply_bench.py --config c3_4d_lshape --prof > $O/apply_c3_4d_lshape.jsonl 2>/dev/null; tail -1 $O/apply_c3_4d_lshape.jsonl
python tools/apply_bench.py --config c4_6d_stream --prof > $O/apply_c4_6d_stream.jsonl 2>/dev/null; tail -1 $O/apply_c4_6d_stream.jsonl
python tools/apply_bench.py --config c2_4d_stream --prof > $O/apply_c2_4d_stream.jsonl 2>/dev/null; tail -1 $O/apply_c2_4d_stream.jsonl
fi
if [ "$2" = "bench" ]; then bash tools/final_benches.sh $O > $O/final_benches.log 2>&1; cat $O/final_benches.log; exit 0; fi
if [ "$2" = "traffic" ]; then bash tools/traffic_capture.sh $O > $O/traffic.log 2>&1; tail -5 $O/traffic.log; exit 0; fi
for k in k_xfanin_tma k_vfan_st; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/ncu_${k}_c4g3 -f python tools/apply_bench.py --config c4_6d_stream --grids 3 --reps 2 > $O/ncu_$k.log 2>&1
  python tools/ncu_summary.py $O/ncu_${k}_c4g3.ncu-rep > $O/ncu_full_${k}_c4g3.txt 2>/dev/null
  ncu -i $O/ncu_${k}_c4g3.ncu-rep --page source --csv --print-source sass > /tmp/sass_$k.csv 2>/dev/null
  python tools/sass_mix.py /tmp/sass_$k.csv > $O/sass_mix_${k}_c4g3.txt 2>/dev/null
done
timeout 600 ncu --set full --clock-control none -k regex:k_fwhole -s 2 -c 1 -o $O/ncu_k_fwhole_c4g0 -f python tools/apply_bench.py --config c4_6d_stream --grids 0 --reps 2 > $O/ncu_fwhole.log 2>&1
python tools/ncu_summary.py $O/ncu_k_fwhole_c4g0.ncu-rep > $O/ncu_full_k_fwhole_c4g0.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_gather_s2c -s 2 -c 1 -o $O/ncu_k_gather_s2c_c3g4 -f python tools/apply_bench.py --config c3_4d_lshape --grids 4 --reps 2 > $O/ncu_gs2c.log 2>&1
python tools/ncu_summary.py $O/ncu_k_gather_s2c_c3g4.ncu-rep > $O/ncu_full_k_gather_s2c_c3g4.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_vmom -s 2 -c 1 -o $O/ncu_k_vmom_c2g5 -f python tools/apply_bench.py --config c2_4d_stream --grids 5 --reps 2 > $O/ncu_vmom.log 2>&1
python tools/ncu_summary.py $O/ncu_k_vmom_c2g5.ncu-rep > $O/ncu_full_k_vmom_c2g5.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_xfanin_tma -s 2 -c 1 -o $O/ncu_k_xfanin_tma_c2g5 -f python tools/apply_bench.py --config c2_4d_stream --grids 5 --reps 2 > $O/ncu_xft2.log 2>&1
python tools/ncu_summary.py $O/ncu_k_xfanin_tma_c2g5.ncu-rep > $O/ncu_full_k_xfanin_tma_c2g5.txt 2>/dev/null
# launch list of the bench command (first strips; the strip solve is a CUDA graph: kernel nodes are profiled one by one)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 15000 -c 3000 --csv --log-file $O/launches_bench_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --secondary none > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches_bench_c4.csv > $O/launches_bench_c4_summary.txt 2>&1; head -20 $O/launches_bench_c4_summary.txt
rm -f $O/*.ncu-rep $O/*.ncu-rep.tmp   # (summaries only: gpurun copies back at most 64 MiB)
ls -la $O | head -60
