# L2-resident chunked apply: per-grid times for several chunk budgets, parity, DRAM traffic
# usage: tools/chunk_experiment.sh OUTDIR
O=${1:-gpurun_out/r2f}
mkdir -p $O
for mb in 0 24 40 64; do
  for c in c4_6d_stream c2_4d_stream; do
    SG_L2_MB=$mb timeout 600 python tools/apply_bench.py --config $c --prof > $O/apply_${c}_mb$mb.jsonl 2> $O/apply_${c}_mb$mb.err
    tail -1 $O/apply_${c}_mb$mb.jsonl
  done
done
SG_L2_MB=40 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply or full" > $O/pytest_chunk40.log 2>&1; tail -3 $O/pytest_chunk40.log
for mb in 0 40; do
  SG_L2_MB=$mb timeout 600 ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/traffic_c4_mb$mb.csv python tools/apply_bench.py --config c4_6d_stream --reps 1 > $O/traffic_c4_mb$mb.log 2>&1
  python tools/apply_traffic.py $O/traffic_c4_mb$mb.csv c4_6d_stream 261111171 2 $O/traffic_c4_mb$mb.json
  gzip -f $O/traffic_c4_mb$mb.csv
done
