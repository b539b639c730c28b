"""Time basis and the Kronecker expansion of the strip operator A^(delta) (oracle).

PAPER.md sec. 4.2 l.440-477:  with time quadrature nodes tau_mu (exact here,
the configs' coefficients are time independent)

  A_{l,l'} = sum_mu w_mu [ (T^t_mu + delta C^t_mu) (x) M
                          + delta T^t_mu (x) (T^r)^T
                          + delta (T^t_mu)^T (x) (T^r + K^r)
                          + M^t_mu (x) (T^r + delta C^r + K^r + delta K~^r - G^r) ]
             + G^t (x) M

where the time blocks are M^t = [eta_s' eta_s], T^t = [eta'_s' eta_s],
C^t = [eta'_s' eta'_s] (row s = test, column s' = trial) and
G^t = [eta_s'(t_{j-1}) eta_s(t_{j-1})].  Reading R1: the paper
prints "+ K~" without delta; the weak form eq. (4) l.89 puts delta in front
of every test-function derivative, so (sigma U, delta d_beta w) = delta K~.

The space matrices are expanded into Kronecker products of factor matrices
(l.479-504) from beta = sum_r a_r(x) b_r(v) e_{axis_r}:
  d_beta phi = sum_r a_r b_r d_{axis_r} phi
  T^r = sum_r (a_r D_r^x phi', phi)_x (x) (b_r D_r^v phi', phi)_v
  C^r = sum_{r,r'} (a_r a_r' D_r^x phi', D_r'^x phi)_x (x) (b_r b_r' D_r^v phi', D_r'^v phi)_v
  K^r = sigma M,  K~^r = sigma (T^r)^T   (sigma constant in all configs)
  G^r = sum over faces of Omega = (dOmega1 x Omega2) u (Omega1 x dOmega2) of
        int_{face} (beta.n) chi_{beta.n<0} phi' phi, factorised as in l.706-716.
"""
from __future__ import annotations

import math
from collections import OrderedDict

import numpy as np

from .fem import MatSpec, face, vol, poly_key


# ----------------------------------------------------------------------------
# time basis: Legendre polynomials on the strip (reading R6)
# ----------------------------------------------------------------------------
def legendre(s: int, xi):
    xi = np.asarray(xi, float)
    if s == 0:
        return np.ones_like(xi)
    if s == 1:
        return xi
    if s == 2:
        return 1.5 * xi ** 2 - 0.5
    raise ValueError("dG order > 2 not needed")


def dlegendre(s: int, xi):
    xi = np.asarray(xi, float)
    if s == 0:
        return np.zeros_like(xi)
    if s == 1:
        return np.ones_like(xi)
    if s == 2:
        return 3.0 * xi
    raise ValueError


def time_blocks(q: int, tau: float):
    """Exact time blocks on a strip of length tau, eta_s(t) = P_s(xi), xi = 2(t-t_{j-1})/tau - 1.

    Integrals by Gauss-Legendre with q+2 points (exact for degree <= 2q+3).
    Returns dict Mt, Tt, Ct, Gt, eta_minus = eta(t_{j-1}^+), eta_plus = eta(t_j^-)."""
    xg, wg = np.polynomial.legendre.leggauss(q + 2)
    S = q + 1
    Mt = np.zeros((S, S)); Tt = np.zeros((S, S)); Ct = np.zeros((S, S))
    for s in range(S):          # test
        for sp_ in range(S):    # trial
            e_s, e_sp = legendre(s, xg), legendre(sp_, xg)
            de_s, de_sp = dlegendre(s, xg) * 2 / tau, dlegendre(sp_, xg) * 2 / tau
            jac = tau / 2
            Mt[s, sp_] = np.sum(wg * e_sp * e_s) * jac
            Tt[s, sp_] = np.sum(wg * de_sp * e_s) * jac
            Ct[s, sp_] = np.sum(wg * de_sp * de_s) * jac
    em = np.array([legendre(s, -1.0) for s in range(S)], float)
    ep = np.array([legendre(s, 1.0) for s in range(S)], float)
    Gt = np.outer(em, em)
    return dict(Mt=Mt, Tt=Tt, Ct=Ct, Gt=Gt, eta_minus=em, eta_plus=ep)


# ----------------------------------------------------------------------------
# polynomial helpers (dict {expo: coef})
# ----------------------------------------------------------------------------
def pmul(p: dict, q: dict) -> dict:
    out = {}
    for a, ca in p.items():
        for b, cb in q.items():
            k = tuple(x + y for x, y in zip(a, b))
            out[k] = out.get(k, 0.0) + ca * cb
    return {k: v for k, v in out.items() if v != 0.0}


def pscale(p: dict, c: float) -> dict:
    return {k: v * c for k, v in p.items() if v * c != 0.0}


def pconst(d: int, c: float) -> dict:
    return {(0,) * d: float(c)}


def p_is_const(p: dict):
    ks = [k for k, v in p.items() if v != 0.0]
    if not ks:
        return True, 0.0
    if len(ks) == 1 and sum(ks[0]) == 0:
        return True, p[ks[0]]
    return False, None


def p_single_coord(p: dict):
    """If p = c * y_i return (i, c) else None."""
    ks = [k for k, v in p.items() if v != 0.0]
    if len(ks) == 1 and sum(ks[0]) == 1:
        return int(np.argmax(ks[0])), p[ks[0]]
    return None


# ----------------------------------------------------------------------------
# space matrices as lists of (xspec, vspec, coef)
# ----------------------------------------------------------------------------
class SpaceTerms:
    def __init__(self, cfg: dict):
        self.cfg = cfg
        d = cfg["d"]
        self.d = d
        self.beta = [(ax, dict(a), dict(b)) for ax, a, b in cfg["beta"]]
        one = pconst(d, 1.0)
        self.M = [(vol(one), vol(one), 1.0)]
        # T^r: (d_beta phi', phi): derivative on the TRIAL function
        self.T = []
        for ax, a, b in self.beta:
            if ax < d:
                self.T.append((vol(a, trial_d=ax), vol(b), 1.0))
            else:
                self.T.append((vol(a), vol(b, trial_d=ax - d), 1.0))
        self.TT = [(x.transpose(), v.transpose(), c) for x, v, c in self.T]
        # C^r: (d_beta phi', d_beta phi)
        self.C = []
        for ax, a, b in self.beta:
            for ax2, a2, b2 in self.beta:
                xd, xd2 = (ax if ax < d else -1), (ax2 if ax2 < d else -1)
                vd, vd2 = (ax - d if ax >= d else -1), (ax2 - d if ax2 >= d else -1)
                self.C.append((vol(pmul(a, a2), trial_d=xd, test_d=xd2),
                               vol(pmul(b, b2), trial_d=vd, test_d=vd2), 1.0))
        self.G = self._inflow_terms()

    def _inflow_terms(self):
        """G^r = sum_faces int (beta.n) chi_{beta.n<0} phi' phi  (eq. (14) l.459, l.706-716).

        Face of Omega1 with normal s e_i:  beta.n = s * beta_{x_i} = s a(x) b(v);
        the configs have a constant there, so the x factor is the face mass
        (times s*a) and the v factor is int chi_{s a b(v) < 0} b(v) phi' phi.
        Face of Omega2 with normal s e_i: symmetric (b constant, chi on x)."""
        d = self.d
        out = []
        for ax in range(2 * d):
            terms = [(a, b) for bax, a, b in self.beta if bax == ax]
            if not terms:
                continue
            assert len(terms) == 1, "one beta term per axis (configs)"
            a, b = terms[0]
            for s in (-1, 1):
                if ax < d:            # x face, normal s e_ax on Omega1
                    const, ca = p_is_const(a)
                    assert const, "inflow factorisation needs a(x) constant on x faces"
                    wpoly = pscale(b, s * ca)               # beta.n = s*ca*b(v)
                    xs = face(ax, s)
                    vs = self._chi_weighted(wpoly, self.d)
                    if vs is not None:
                        out.append((xs, vs, 1.0))
                else:                 # v face, normal s e_{ax-d} on Omega2
                    const, cb = p_is_const(b)
                    assert const, "inflow factorisation needs b(v) constant on v faces"
                    wpoly = pscale(a, s * cb)
                    xs = self._chi_weighted(wpoly, self.d)
                    vs = face(ax - d, s)
                    if xs is not None:
                        out.append((xs, vs, 1.0))
        return out

    @staticmethod
    def _chi_weighted(w: dict, d: int):
        """vol spec int chi_{w<0} w phi' phi for w constant or c*y_i; None if empty."""
        const, c = p_is_const(w)
        if const:
            if c < 0:
                return vol(w)
            return None
        sc = p_single_coord(w)
        assert sc is not None, "inflow weight must be constant or c*y_i"
        i, c = sc
        # w < 0  <=>  c*y_i < 0  <=>  (-sign c) y_i > 0
        return vol(w, chi=(i, -int(np.sign(c))))


def strip_terms(cfg: dict, tau: float, delta: float):
    """Space-time terms (T_block, xspec, vspec) of A^(delta) (reading R1).

    Identical (xspec, vspec) pairs are merged by summing their time blocks;
    zero blocks are dropped.  Returns list of (Tblock (S,S), xspec, vspec)."""
    sig = float(cfg["sigma"])
    st = SpaceTerms(cfg)
    tb = time_blocks(cfg["q"], tau)
    Mt, Tt, Ct, Gt = tb["Mt"], tb["Tt"], tb["Ct"], tb["Gt"]
    acc = OrderedDict()

    def add(Tblk, lst, scale=1.0):
        for xs, vs, c in lst:
            xs, cx = canonical(xs)
            vs, cv = canonical(vs)
            key = (xs, vs)
            acc[key] = acc.get(key, 0.0) + scale * c * cx * cv * Tblk

    add(Tt + delta * Ct + Gt, st.M)                 # (T^t + delta C^t) (x) M  +  G^t (x) M
    add(delta * Tt, st.TT)                          # delta T^t (x) (T^r)^T
    add(delta * Tt.T, st.T)                         # delta (T^t)^T (x) T^r
    add(delta * sig * Tt.T, st.M)                   # delta (T^t)^T (x) K^r
    add(Mt, st.T)                                   # M^t (x) T^r
    add(delta * Mt, st.C)                           # M^t (x) delta C^r
    add(sig * Mt, st.M)                             # M^t (x) K^r
    add(delta * sig * Mt, st.TT)                    # M^t (x) delta K~^r   (reading R1)
    add(-Mt, st.G)                                  # M^t (x) (-G^r)
    terms = [(T, xs, vs) for (xs, vs), T in acc.items() if np.any(T != 0.0)]
    return terms


def canonical(spec: MatSpec):
    """Pull the scalar out of a vol weight: w = c * w^ with the first monomial of w^ equal to 1."""
    if spec.kind != "vol" or not spec.weight:
        return spec, 1.0
    c = spec.weight[0][1]
    w = tuple((k, v / c) for k, v in spec.weight)
    return MatSpec("vol", w, spec.trial_d, spec.test_d, spec.chi), c


def mass_terms(cfg: dict, Tblock: np.ndarray):
    """Single-term operator Tblock (x) M^x (x) M^v (jump load / L2 inner product)."""
    one = pconst(cfg["d"], 1.0)
    return [(np.asarray(Tblock, float), vol(one), vol(one))]


def delta_hmin(cfg: dict) -> float:
    """delta = edge length on the finest scale (configs 0/1 'delta=h_min', reading R5)."""
    if cfg.get("delta") is not None:
        return float(cfg["delta"])
    cells = cfg["nc"] * 2 ** (cfg["L"] - 2)
    h = [(hi - lo) / cells for m in (cfg["xmesh"], cfg["vmesh"]) for lo, hi in zip(m["lo"], m["hi"])]
    return min(h)


def n_strips(cfg: dict) -> int:
    """N = round(T / tau), tau kept exactly (reading R7)."""
    if cfg.get("nsteps") is not None:
        return int(cfg["nsteps"])
    return int(round(cfg["T"] / cfg["tau"]))
