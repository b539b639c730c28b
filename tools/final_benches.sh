# bench lines for all five configs (default K/W), c4 first; usage: tools/final_benches.sh OUTDIR
O=${1:-gpurun_out/final}
mkdir -p $O
for c in c4_6d_stream c3_4d_lshape c1_2d_rot c0_2d_const c2_4d_stream; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --impl reference > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err
for c in c4_6d_stream c3_4d_lshape c1_2d_rot c0_2d_const c2_4d_stream; do python - <<PY
import json
try:
    d=json.load(open("$O/bench_$c.json"))
    print("$c", "%.3e"%d["value"], round(d["ms_per_step"],1), round(d["roofline"]["frac"],4), round(d["roofline"]["hbm_view"]["frac"],4), round(d["roofline"]["share_of_step"],3), "%.3e"%d["e2e"]["value"], d["outer_iters"], d["inner_iters"], d["flagged_unconverged"])
except Exception as e: print("$c", "failed", e)
PY
done
