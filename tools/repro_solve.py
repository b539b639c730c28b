"""Minimal strip solve on a small configuration (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_05988_b200 import Problem
from sginputs import get_config
name = sys.argv[1] if len(sys.argv) > 1 else "c0_2d_const"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
g = Problem(get_config(name, L=L))
n = g.set_size(0, g.S)
b = torch.randn(n, dtype=torch.float64, device="cuda")
u = torch.zeros_like(b)
print("created", flush=True)
it, last = g.sg_solve_strip(b, u, rtol=1e-10, inner_rtol=1e-10, max_iter=50)
print("solved", it, last, flush=True)
