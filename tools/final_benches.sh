# end-of-session bench lines for all five configs (default K/W), c4 first
mkdir -p gpurun_out/r1h
for c in c4_6d_stream c3_4d_lshape c1_2d_rot c0_2d_const c2_4d_stream; do
  timeout 900 python bench.py --config $c > gpurun_out/r1h/final_bench_$c.json 2> gpurun_out/r1h/final_bench_$c.err
done
for c in c4_6d_stream c3_4d_lshape c1_2d_rot c0_2d_const c2_4d_stream; do tail -c 200 gpurun_out/r1h/final_bench_$c.json; echo; done
