"""Instruction mix and stall samples per opcode from `ncu -i REP --page source --csv --print-source sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {k: i for i, k in enumerate(hdr)}
ops = collections.defaultdict(lambda: [0, 0, 0])
tot = [0, 0]
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
stalls = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ci["Source"]].strip()
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0] + ("." + ".".join(op.split(".")[1:2]) if op.startswith(("LD", "ST")) else "")
    n = int(r[ci["Instructions Executed"]] or 0)
    s = int(r[ci["# Samples"]] or 0)
    ops[op][0] += n
    ops[op][1] += s
    tot[0] += n
    tot[1] += s
    for k in stall_cols:
        stalls[k] += int(r[ci[k]] or 0)
print("total inst", tot[0], "samples", tot[1])
for op, (n, s, _) in sorted(ops.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{op:14s} inst {n:12d} {100*n/tot[0]:5.1f}%  samples {100*s/max(tot[1],1):5.1f}%")
print({k: round(100 * v / max(tot[1], 1), 1) for k, v in stalls.most_common(8)})
