set -x
mkdir -p gpurun_out/r1h
for c in c4_6d_stream c2_4d_stream c3_4d_lshape c1_2d_rot c0_2d_const; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r1h/traffic_$c.csv python tools/apply_bench.py --config $c --reps 1 > gpurun_out/r1h/traffic_$c.log 2>&1
done
ls -la gpurun_out/r1h
