O=${1:-gpurun_out/r2p}
mkdir -p $O
run() { # name cfg grids wc kb nst
  SG_VERBOSE=1 SG_XFT_WC=$4 SG_XFT_KB=$5 SG_XFT_NST=$6 timeout 300 python tools/apply_bench.py --config $2 --grids $3 --prof > $O/tiles_$1.jsonl 2> $O/tiles_$1.err
  echo "== $1 $2 wc=$4 kb=$5 nst=$6"; grep -h "^xft" $O/tiles_$1.err | sort -u | head -8
  python - <<PY
import json
for l in open("$O/tiles_$1.jsonl"):
    if l.startswith("{") and "grid" in l:
        d=json.loads(l); print(d["l1"],d["l2"],d["ms"],[v for k,v in d["kernels_ms"].items() if "xfanin" in k])
PY
}
run c4W8s2 c4_6d_stream 2,3,4,5,6 8 32 2
run c4W8s3 c4_6d_stream 2,3,4,5,6 8 32 3
run c4W8s4 c4_6d_stream 2,3,4,5,6 8 32 4
run c4W8k48 c4_6d_stream 2,3,4,5,6 8 48 3
run c4W8k48s2 c4_6d_stream 2,3,4,5,6 8 48 2
run c2base c2_4d_stream 2,3,4,5,6,7,8 4 8 4
run c2W8k12 c2_4d_stream 2,3,4,5,6,7,8 8 12 4
run c2W8k16 c2_4d_stream 2,3,4,5,6,7,8 8 16 4
run c2W8k24 c2_4d_stream 2,3,4,5,6,7,8 8 24 4
run c2W8k24s3 c2_4d_stream 2,3,4,5,6,7,8 8 24 3
run c2W4k16 c2_4d_stream 2,3,4,5,6,7,8 4 16 4
