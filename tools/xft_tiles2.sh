O=${1:-gpurun_out/r2m}
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
run G3 4 24 3 3
run G4 4 24 4 3
run H3 4 32 3 3
run H2 4 32 2 3
run I4 2 12 4 3
run I6 2 12 6 3
run J4 2 16 4 3
run J6 2 16 6 3
