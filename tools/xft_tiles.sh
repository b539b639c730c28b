# pass-2 tile sweep (TMA line sweep), per-grid kernel times
O=${1:-gpurun_out/r2g}
mkdir -p $O
run() { # name wc kb nst cta
  SG_VERBOSE=1 SG_XFT_WC=$2 SG_XFT_KB=$3 SG_XFT_NST=$4 SG_XFT_CTA=$5 timeout 300 python tools/apply_bench.py --config c4_6d_stream --grids 2,3,4,5 --prof > $O/tiles_$1.jsonl 2> $O/tiles_$1.err
  echo "== $1 wc=$2 kb=$3 nst=$4 cta=$5"; grep -h "^xft" $O/tiles_$1.err | sort -u | head -4
  python - <<PY
import json
for l in open("$O/tiles_$1.jsonl"):
    if l.startswith("{") and "grid" in l:
        d=json.loads(l); print(d["l1"],d["l2"],d["ms"],[v for k,v in d["kernels_ms"].items() if "xfanin" in k])
PY
}
run A 4 16 3 3
run A4 4 16 4 3
run B 2 20 3 3
run B4 2 20 4 3
run B6 2 20 6 3
run C 1 28 3 3
run C4 1 28 4 3
run D 4 40 3 3
run D4 4 40 4 3
run E 2 32 3 3
run E4 2 32 4 3
run F 1 16 4 3
run Bc2 2 20 4 2
run Bc6 2 20 4 6
