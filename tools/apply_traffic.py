"""DRAM traffic of the strip-operator apply, per DOF, from an ncu metrics CSV.

Input: the CSV of
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      python tools/apply_bench.py --config C --reps 1
which runs 1 + reps applies on every active grid.  Only the library's own kernels
(namespace sg::) after the first torch randn launch are counted: the mesh/assembly
setup before it and torch's own kernels are dropped.

Usage: apply_traffic.py CSV CONFIG TOTAL_DOF APPLIES_PER_GRID OUT_JSON
TOTAL_DOF = sum of S*n1*n2 over the grids (apply_bench's last line).  The result
(bytes per DOF-apply) is what bench.py multiplies by its mean DOF per apply to
report roofline.traffic."""
import csv, json, sys
from collections import defaultdict

path, config, total_dof, per_grid, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ii, ni, mi, ui, vi = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
per = defaultdict(dict)
names = {}
started = False
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    if "distribution" in r[ni]:
        started = True
    if not started or "sg::" not in r[ni]:
        continue
    try:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    except ValueError:
        continue
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ni].split("(")[0]
rd = sum(m.get("dram__bytes_read.sum", 0.0) for m in per.values())
wr = sum(m.get("dram__bytes_write.sum", 0.0) for m in per.values())
t = sum(m.get("gpu__time_duration.sum", 0.0) for m in per.values())
by_kernel = defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    e = by_kernel[names[k]]
    e[0] += 1
    e[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    e[2] += m.get("gpu__time_duration.sum", 0.0)
dof_applied = total_dof * per_grid
res = {"config": config, "launches": len(per), "dof_applied": dof_applied,
       "dram_read_bytes": rd, "dram_write_bytes": wr,
       "dram_bytes_per_dof": (rd + wr) / dof_applied, "ncu_time_s": t,
       "dram_gbs_serialised": (rd + wr) / t / 1e9 if t else None,
       "by_kernel": {k: {"launches": n, "dram_bytes": b, "time_s": s} for k, (n, b, s) in
                     sorted(by_kernel.items(), key=lambda x: -x[1][1])},
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on tools/apply_bench.py "
                 f"--config {config} ({per_grid} applies per grid, cold-cache serialised replay)"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: res[k] for k in ("launches", "dram_bytes_per_dof", "dram_gbs_serialised")}))
