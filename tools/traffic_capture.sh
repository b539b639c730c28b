# DRAM traffic of the strip-operator apply (ncu, cold-cache serialised replay) for all five configs
# usage: tools/traffic_capture.sh OUTDIR ; then tools/apply_traffic.py per config (see profiles/README.md)
O=${1:-gpurun_out/traffic}
mkdir -p $O
for c in c4_6d_stream c2_4d_stream c3_4d_lshape c1_2d_rot c0_2d_const; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/traffic_$c.csv python tools/apply_bench.py --config $c --reps 1 > $O/traffic_$c.log 2>&1
  dof=$(tail -1 $O/traffic_$c.log | python -c "import json,sys; print(json.loads(sys.stdin.read())['total_dof'])")
  python tools/apply_traffic.py $O/traffic_$c.csv $c $dof 2 $O/traffic_$c.json
  gzip -f $O/traffic_$c.csv
done
