# pass-1 rows-per-thread experiment on 3D v-lattices (SG_VF_R = 2/3/4)
mkdir -p gpurun_out/r1h
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "kernel_paths and SG_VF_R" > gpurun_out/r1h/pytest_vfr.log 2>&1
for r in 2 3 4 2; do
  SG_VF_R=$r timeout 300 python tools/apply_bench.py --config c4_6d_stream --reps 5 --prof > gpurun_out/r1h/apply_vfr$r.jsonl 2>&1
done
SG_VF_R=4 timeout 600 python bench.py --no-cpu > gpurun_out/r1h/bench_c4_vfr4.json 2>gpurun_out/r1h/bench_c4_vfr4.err
tail -2 gpurun_out/r1h/pytest_vfr.log; for r in 2 3 4; do tail -1 gpurun_out/r1h/apply_vfr$r.jsonl; done; tail -c 300 gpurun_out/r1h/bench_c4_vfr4.json
