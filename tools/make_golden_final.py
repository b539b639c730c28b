#!/usr/bin/env python
"""Write tests/golden/final_<config>_L<L>.npz: the oracle's solution at the final time T
(all N = round(T/tau) strips, direct-LU Richardson at rtol 1e-13) for the final-time
parity test (tests/test_gpu_parity.py::test_final_time).  Calls only oracle/ and the
input module sginputs/ (no CUDA path).

  python tools/make_golden_final.py c0_2d_const 6
  python tools/make_golden_final.py c1_2d_rot 5
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.sgrid import SGProblem  # noqa: E402
from sginputs import get_config  # noqa: E402


def main(name, L, nsteps=None):
    cfg = get_config(name, L=L)
    o = SGProblem(cfg)
    N = int(round(cfg["T"] / cfg["tau"])) if nsteps is None else nsteps
    t0 = time.time()
    tr, _, its = o.run(nsteps=N, rtol=1e-13)
    out = {"nsteps": N, "full": o.to_full(tr), "iters": np.asarray(its)}
    for (l1, l2), u in tr.items():
        out[f"block_{l1}_{l2}"] = u
    tag = "final" if nsteps is None else f"strips{nsteps}"
    path = os.path.join(ROOT, "tests", "golden", f"{tag}_{name}_L{L}.npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {N} strips in {time.time() - t0:.1f}s, outer its {min(its)}-{max(its)}, "
          f"||U(T)|| = {o.spatial_l2(tr):.6e}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else None)
