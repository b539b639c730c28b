"""Problem data and seeded input generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no meshes, no matrices, no
quadrature): only the five BASELINE.json configurations written out as plain
data, small variants of them for parity tests, and seeded random block
vectors.  Both `oracle/` and `paper_2204_05988_b200/` read it; neither reads
the other.

Conventions:
  * level l of a factor mesh has nc * 2**(l-1) cells per axis (nc = 2, i.e.
    "2^l cells", BASELINE configs[0]);
  * a combination level L has active component grids |l|_1 = L and coarse
    (preconditioner) grids |l|_1 = L-1 ("l1+l2 in {6,5}" for L=6, configs[0]);
    this is the paper's eq. (3)/(sec. 4.1) V_L with its L shifted by one;
  * polynomials are dicts {exponent tuple: coefficient} in the coordinates of
    one factor domain (x for a(x), v for b(v));
  * beta = sum_r a_r(x) b_r(v) e_{axis_r}   (sec. 4.2 l.486), axis in
    0..2d-1 (0..d-1 are x axes, d..2d-1 are v axes);
  * u0 = sum of rank-1 terms, each a product of per-factor Gaussians
    scale * exp(-|y - c|^2 / w).
"""
from __future__ import annotations

import copy
import math

import numpy as np


def _gauss(center, w, scale=1.0):
    return {"center": list(map(float, center)), "w": float(w), "scale": float(scale)}


def _poly_const(d, c):
    return {(0,) * d: float(c)}


def _poly_coord(d, i, c=1.0):
    e = [0] * d
    e[i] = 1
    return {tuple(e): float(c)}


# --------------------------------------------------------------------------
# BASELINE.json configs (indices 0..4).  Plain data.
# --------------------------------------------------------------------------
CONFIGS = {
    # configs[0]: 2D phase space, constant beta, inflow g = u0(r - beta t)
    "c0_2d_const": dict(
        d=1,
        xmesh=dict(kind="box", lo=[0.0], hi=[1.0]),
        vmesh=dict(kind="box", lo=[0.0], hi=[1.0]),
        nc=2, L=6, q=0, tau=1.0 / 64, T=0.5, sigma=0.0,
        beta=[(0, _poly_const(1, 1.0), _poly_const(1, 1.0)),
              (1, _poly_const(1, 1.0), _poly_const(1, 0.5))],
        u0=[(1.0, _gauss([0.3], 0.01), _gauss([0.3], 0.01))],
        g="shifted_u0",
    ),
    # configs[1]: 2D rotation beta = (v, -x), dG(1)
    "c1_2d_rot": dict(
        d=1,
        xmesh=dict(kind="box", lo=[-1.0], hi=[1.0]),
        vmesh=dict(kind="box", lo=[-1.0], hi=[1.0]),
        nc=2, L=14, q=1, tau=2.0 ** -8, T=math.pi / 2, sigma=0.0,
        beta=[(0, _poly_const(1, 1.0), _poly_coord(1, 0, 1.0)),
              (1, _poly_coord(1, 0, -1.0), _poly_const(1, 1.0))],
        u0=[(1.0, _gauss([0.4], 0.02), _gauss([0.0], 0.02))],
        g=None,
    ),
    # configs[2]: 4D free streaming beta = (v, 0), sigma = 0.1
    "c2_4d_stream": dict(
        d=2,
        xmesh=dict(kind="box", lo=[0.0, 0.0], hi=[1.0, 1.0]),
        vmesh=dict(kind="box", lo=[-1.0, -1.0], hi=[1.0, 1.0]),
        nc=2, L=12, q=0, tau=2.0 ** -7, T=0.25, sigma=0.1,
        beta=[(0, _poly_const(2, 1.0), _poly_coord(2, 0)),
              (1, _poly_const(2, 1.0), _poly_coord(2, 1))],
        u0=[(1.0, _gauss([0.5, 0.5], 0.01), _gauss([0.3, 0.2], 0.01))],
        g=None,
    ),
    # configs[3]: 4D L-shaped x domain, harmonic force beta = (v, -x), dG(1)
    "c3_4d_lshape": dict(
        d=2,
        xmesh=dict(kind="lshape", lo=[-1.0, -1.0], hi=[1.0, 1.0]),
        vmesh=dict(kind="box", lo=[-4.0, -4.0], hi=[4.0, 4.0]),
        nc=2, L=11, q=1, tau=2.0 ** -7, T=0.5, sigma=0.0,
        beta=[(0, _poly_const(2, 1.0), _poly_coord(2, 0)),
              (1, _poly_const(2, 1.0), _poly_coord(2, 1)),
              (2, _poly_coord(2, 0, -1.0), _poly_const(2, 1.0)),
              (3, _poly_coord(2, 1, -1.0), _poly_const(2, 1.0))],
        u0=[(1.0, _gauss([-0.5, 0.5], 0.05), _gauss([0.0, 0.0], 2.0, 1.0 / (2 * math.pi)))],
        g=None,
    ),
    # configs[4]: 6D free streaming beta = (v, 0)
    "c4_6d_stream": dict(
        d=3,
        xmesh=dict(kind="box", lo=[0.0] * 3, hi=[1.0] * 3),
        vmesh=dict(kind="box", lo=[-4.0] * 3, hi=[4.0] * 3),
        nc=2, L=8, q=0, tau=2.0 ** -6, T=0.125, sigma=0.0,
        beta=[(i, _poly_const(3, 1.0), _poly_coord(3, i)) for i in range(3)],
        u0=[(1.0, _gauss([0.5] * 3, 0.02), _gauss([0.0] * 3, 2.0, (2 * math.pi) ** -1.5))],
        g=None,
    ),
}

CONFIG_ORDER = ["c0_2d_const", "c1_2d_rot", "c2_4d_stream", "c3_4d_lshape", "c4_6d_stream"]


def get_config(name: str, **over) -> dict:
    """Return a deep copy of a config with overrides (e.g. L=4, nsteps=2)."""
    cfg = copy.deepcopy(CONFIGS[name])
    cfg["name"] = name
    cfg.update(over)
    return cfg


def seeded_block(rng_seed: int, shape, scale=1.0) -> np.ndarray:
    """Seeded standard-normal fp64 array (input generator for parity tests)."""
    rng = np.random.default_rng(rng_seed)
    return scale * rng.standard_normal(shape)
