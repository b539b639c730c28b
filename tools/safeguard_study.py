#!/usr/bin/env python
"""When does the minimal-residual safeguard (reading R13) engage?  Runs the first
strips of a configuration and prints, per strip, the outer iterations, whether the update
norm ever grew (the safeguard's trigger) and the norm history.

  python tools/safeguard_study.py c1_2d_rot 5 3 1e-12
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_05988_b200 import Problem  # noqa: E402
from sginputs import get_config  # noqa: E402

name, L, nst, inner = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
cfg = get_config(name, L=L)
g = Problem(cfg)
tr = torch.zeros(g.set_size(0, 1), dtype=torch.float64, device="cuda")
g.sg_interp_u0(tr)
for j in range(1, nst + 1):
    g.reset_stats()
    g.sg_step(j, 1, tr, 1e-10, inner)
    nd, om = g.solve_history()
    st = g.stats()
    grew = [i + 1 for i in range(1, len(nd)) if nd[i] > nd[i - 1]]
    print(json.dumps(dict(config=name, L=L, strip=j, inner_rtol=inner, outer_iters=len(nd),
                          inner_iters=st["inner_iters"], mr_switches=st["outer_mr_switches"],
                          growth_at=grew, first_growth_ratio=(nd[grew[0] - 1] / nd[grew[0] - 2]) if grew else None,
                          nd=[float("%.3e" % x) for x in nd], omega=[round(x, 3) for x in om])), flush=True)
