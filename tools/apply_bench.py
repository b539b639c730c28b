"""Time the per-grid strip-operator apply (sg_apply_strip_operator) on every active grid."""
import os, sys, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_05988_b200 import Problem
from sginputs import get_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4_6d_stream")
ap.add_argument("--L", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--grids", default="all")
ap.add_argument("--prof", action="store_true", help="per-kernel device times (torch.profiler / CUPTI, no replay)")
a = ap.parse_args()
cfg = get_config(a.config, **({} if a.L is None else {"L": a.L}))
prob = Problem(cfg)
S = prob.S
grids = range(prob.num_grids(0)) if a.grids == "all" else [int(x) for x in a.grids.split(",")]
tot_ms = 0; tot_dof = 0
for g in grids:
    l1, l2, n1, n2 = prob.grid_info(0, g)
    n = S * n1 * n2
    X = torch.randn(n, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    prob.sg_apply_strip_operator(0, g, X, Y)
    torch.cuda.synchronize()
    prob.reset_stats(); prob.set_timing(True)
    for _ in range(a.reps):
        prob.sg_apply_strip_operator(0, g, X, Y)
    kt = prob.kernel_time(); prob.set_timing(False)
    kern = None
    if a.prof:
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as pr:
            for _ in range(a.reps):
                prob.sg_apply_strip_operator(0, g, X, Y)
            torch.cuda.synchronize()
        kern = {}
        for ev in pr.key_averages():
            if ev.device_type.name == "CUDA" and ev.count:
                kern[ev.key[:40]] = round(getattr(ev, "device_time_total", 0) / 1e3 / a.reps, 4)
    ms = kt["ms"] / a.reps
    tot_ms += ms; tot_dof += n
    print(json.dumps(dict(grid=g, l1=l1, l2=l2, n1=n1, n2=n2, dof=n, ms=round(ms, 4),
                          gdof_s=round(n / ms / 1e6, 3), alg_gbs=round(kt["bytes"] / a.reps / ms / 1e6, 1),
                          gflops=round(kt["flops"] / a.reps / ms / 1e6, 1), kernels_ms=kern)), flush=True)
print(json.dumps(dict(total_ms=tot_ms, total_dof=tot_dof, gdof_s=tot_dof / tot_ms / 1e6)))
