"""Exact characteristic solutions and L2 errors (oracle; used by pins and bench notes).

PAPER.md eq. (1) l.36-42 with f = 0, g = exact trace: the solution is
transported along the characteristics of beta and damped by exp(-sigma t):
  constant beta (configs[0]):  u(t,r) = u0(r - beta t)
  rotation beta = (v,-x) (configs[1]): u(t,x,v) = u0(x cos t - v sin t, x sin t + v cos t)
  free streaming beta = (v,0), sigma: u(t,x,v) = exp(-sigma t) u0(x - v t, v)
Errors are L2 norms over Omega computed with 4x4 Gauss-Legendre on every cell
of the full fine grid (d = 1), on which the sparse-grid function is bilinear.
"""
from __future__ import annotations

import math

import numpy as np

from .fem import gaussian_factor, gl01


def u0_fun(cfg):
    terms = [(c, gaussian_factor(gx), gaussian_factor(gv)) for c, gx, gv in cfg["u0"]]
    d = cfg["d"]

    def f(x, v):
        return sum(c * fx(x) * fv(v) for c, fx, fv in terms)
    return f


def exact_fun(cfg, t):
    name = cfg.get("exact", cfg["name"])
    u0 = u0_fun(cfg)
    d = cfg["d"]
    if name.startswith("c0"):
        beta = np.zeros(2 * d)
        for ax, a, b in cfg["beta"]:
            beta[ax] += list(a.values())[0] * list(b.values())[0]
        return lambda x, v: u0(x - beta[:d] * t, v - beta[d:] * t)
    if name.startswith("c1"):
        c, s = math.cos(t), math.sin(t)
        return lambda x, v: u0(x * c - v * s, x * s + v * c)
    if name.startswith("c2") or name.startswith("c4"):
        sig = cfg["sigma"]
        return lambda x, v: math.exp(-sig * t) * u0(x - v * t, v)
    raise ValueError(name)


def l2_error_2d(P, Ufull, fun):
    """||U - fun||_{L2(Omega)} and ||fun|| for d = 1, Ufull nodal values on the (F,F) grid."""
    mx = P.Hx.meshes[P.F]; mv = P.Hv.meshes[P.F]
    xs = mx.coords[:, 0]; vs = mv.coords[:, 0]
    g, w = gl01(4)
    err2 = 0.0; nrm2 = 0.0
    for i in range(mx.n - 1):
        hx = xs[i + 1] - xs[i]
        xq = xs[i] + hx * g
        for k in range(mv.n - 1):
            hv = vs[k + 1] - vs[k]
            vq = vs[k] + hv * g
            X, V = np.meshgrid(xq, vq, indexing="ij")
            a = (X - xs[i]) / hx; b = (V - vs[k]) / hv
            U = ((1 - a) * (1 - b) * Ufull[i, k] + a * (1 - b) * Ufull[i + 1, k]
                 + (1 - a) * b * Ufull[i, k + 1] + a * b * Ufull[i + 1, k + 1])
            E = fun(X.reshape(-1, 1), V.reshape(-1, 1)).reshape(X.shape)
            W = np.outer(w, w) * hx * hv
            err2 += np.sum(W * (U - E) ** 2)
            nrm2 += np.sum(W * E ** 2)
    return math.sqrt(err2), math.sqrt(nrm2)
