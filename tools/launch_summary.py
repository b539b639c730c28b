"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ni, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in rows[start + 1:]:
    if len(r) <= vi: continue
    k = r[ni].split("(")[0]
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    if v != v:   # nan: the launch that was cut off when ncu stopped
        continue
    agg[k][0] += 1; agg[k][1] += v; tot += v
print(f"launches {sum(a[0] for a in agg.values())}, device time {tot/1e6:.2f} ms (serialised, cold-cache)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:6d} {t/1e6:9.3f} ms {100*t/tot:6.2f}%  {k}")
