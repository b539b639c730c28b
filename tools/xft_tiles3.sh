O=${1:-gpurun_out/r2o}
mkdir -p $O
run() { # name wc kb nst np
  SG_VERBOSE=1 SG_XFT_WC=$2 SG_XFT_KB=$3 SG_XFT_NST=$4 SG_XFT_NP=$5 timeout 300 python tools/apply_bench.py --config c4_6d_stream --grids 2,3,4,5 --prof > $O/tiles_$1.jsonl 2> $O/tiles_$1.err
  echo "== $1 wc=$2 kb=$3 nst=$4 np=$5"; grep -h "^xft" $O/tiles_$1.err | sort -u | head -4
  python - <<PY
import json
for l in open("$O/tiles_$1.jsonl"):
    if l.startswith("{") and "grid" in l:
        d=json.loads(l); print(d["l1"],d["l2"],d["ms"],[v for k,v in d["kernels_ms"].items() if "xfanin" in k], [v for k,v in d["kernels_ms"].items() if "vfan" in k])
PY
}
run A 4 16 3 1
run Anp2 4 16 3 2
run Anp4 4 16 3 4
run Dnp1 4 40 3 1
run Dnp2 4 40 3 2
run Dnp3 4 40 3 3
run Dnp6 4 40 3 6
run Dnp6s4 4 40 4 6
run Gnp3 4 24 3 3
run Gnp6 4 24 3 6
run W8np1 8 32 3 1
run W8np2 8 32 3 2
run W8np4 8 32 3 4
