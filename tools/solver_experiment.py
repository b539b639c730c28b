"""Inner/outer iteration trade-off of the strip solver on the GPU (one strip)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_05988_b200 import Problem
from sginputs import get_config

IRTS = [float(x) for x in os.environ.get("IRTS", "1e-10,1e-6,1e-3,1e-2").split(",")]
cases = [("c4_6d_stream", 6), ("c2_4d_stream", 8), ("c3_4d_lshape", 7), ("c1_2d_rot", 10)]
if len(sys.argv) > 1:
    cases = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]
for name, L in cases:
    for pre in [int(x) for x in os.environ.get("PRE", "1,0").split(",")]:
        if pre: os.environ.pop("SG_NO_PRECOND", None)
        else: os.environ["SG_NO_PRECOND"] = "1"
        prob = Problem(get_config(name, L=L))
        for irt in IRTS:
            tr = torch.zeros(prob.set_size(0, 1), dtype=torch.float64, device="cuda")
            prob.sg_interp_u0(tr)
            b = torch.zeros(prob.set_size(0, prob.S), dtype=torch.float64, device="cuda")
            prob.sg_rhs(1, tr, b)
            u = torch.zeros_like(b)
            prob.reset_stats(); torch.cuda.synchronize(); t0 = time.perf_counter()
            try:
                it, last = prob.sg_solve_strip(b, u, rtol=1e-10, inner_rtol=irt, max_iter=300)
            except Exception as e:
                it, last = -1, str(e)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            st = prob.stats()
            print(json.dumps(dict(cfg=name, L=L, precond=pre, inner_rtol=irt, outer=it, last=last,
                                  inner=st["inner_iters"], applies=st["applies"], dof=st["dof_applied"],
                                  sec=round(dt, 3), dof_per_s=st["dof_applied"] / dt)), flush=True)
        del prob
