timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_strip or cross_grid" 2>&1 | tail -5 > gpurun_out/t_apply.log
for c in c4_6d_stream c2_4d_stream; do
timeout 300 python tools/apply_bench.py --config $c --reps 3 --prof > gpurun_out/abp_$c.log 2>&1
done
cat gpurun_out/t_apply.log
