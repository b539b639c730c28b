"""Per-kernel device-time breakdown of one bench step (torch.profiler / CUPTI activity
records, no kernel replay): python tools/step_prof.py --config c4_6d_stream"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2204_05988_b200 import Problem
from sginputs import get_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4_6d_stream")
ap.add_argument("--L", type=int, default=None)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--inner-rtol", type=float, default=1e-2)
a = ap.parse_args()
cfg = get_config(a.config, **({} if a.L is None else {"L": a.L}))
prob = Problem(cfg, stream=torch.cuda.current_stream())
tr = torch.zeros(prob.set_size(0, 1), dtype=torch.float64, device="cuda")
prob.sg_interp_u0(tr)
j = 1
for _ in range(a.warmup):
    prob.sg_step(j, 1, tr, 1e-10, a.inner_rtol); j += 1
torch.cuda.synchronize()
prob.reset_stats()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as pr:
    ev0.record()
    prob.sg_step(j, 1, tr, 1e-10, a.inner_rtol)
    ev1.record()
    torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1)
rows = []
for ev in pr.key_averages():
    t = getattr(ev, "device_time_total", 0)
    if t > 0:
        rows.append((t / 1e3, ev.count, ev.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(json.dumps({"config": cfg["name"], "L": cfg["L"], "step_ms": ms, "kernel_ms_total": tot, "stats": prob.stats()}))
for t, c, k in rows[:30]:
    print(f"{t:10.2f} ms {100 * t / tot:6.2f}% {c:8d}  {k[:90]}")
