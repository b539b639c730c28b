"""Pins of oracle/problem.py + the block apply of oracle/sgrid.py (no GPU).

(c) factored apply == explicitly formed dense Kronecker sum (tiny levels);
weak form: the Kronecker expansion (reading R1) equals a
direct space-time quadrature of a_j^(delta) (eq. (4) l.89-91) on one grid;
energy identity: U^T A U equals eq. (11) l.176-181 evaluated by quadrature.
"""
import itertools
import math

import numpy as np
import pytest

from sginputs import CONFIG_ORDER, get_config
from oracle.problem import time_blocks
from oracle.sgrid import SGProblem

SMALL = {"c0_2d_const": 4, "c1_2d_rot": 4, "c2_4d_stream": 3, "c3_4d_lshape": 3, "c4_6d_stream": 3}


def test_time_blocks_closed_form():
    tau = 0.3
    tb = time_blocks(0, tau)
    assert np.allclose(tb["Mt"], [[tau]]) and np.allclose(tb["Tt"], 0) and np.allclose(tb["Gt"], 1)
    tb = time_blocks(1, tau)
    # Legendre P0 = 1, P1 = xi on the strip
    assert np.allclose(tb["Mt"], tau * np.diag([1.0, 1.0 / 3.0]), atol=1e-15)
    assert np.allclose(tb["Tt"], [[0.0, 2.0], [0.0, 0.0]], atol=1e-15)
    assert np.allclose(tb["Ct"], (2.0 / tau) * np.diag([0.0, 2.0]), atol=1e-13)
    assert np.allclose(tb["Gt"], [[1.0, -1.0], [-1.0, 1.0]])
    # discrete integration by parts: T + T^T = eta(t_j)eta(t_j)^T - eta(t_{j-1})eta(t_{j-1})^T
    ep, em = tb["eta_plus"], tb["eta_minus"]
    assert np.allclose(tb["Tt"] + tb["Tt"].T, np.outer(ep, ep) - np.outer(em, em), atol=1e-14)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_factored_equals_dense_kron(name):
    """(c) A_{l,l'} u applied factored == dense kron(T, kron(X, V)) @ vec(u)."""
    P = SGProblem(get_config(name, L=SMALL[name]))
    rng = np.random.default_rng(7)
    for l in P.active[:2] + P.active[-1:]:
        for lp in (P.active[0], l, P.active[-1]):
            u = rng.standard_normal(P.shape(lp))
            y = P.apply_pair(P.terms, l, lp, u)
            # explicit dense Kronecker sum, formed term by term with numpy.kron
            D = 0
            for T, xs, vs in P.terms:
                X = P.factor("x", xs, l[0], lp[0]).toarray()
                V = P.factor("v", vs, l[1], lp[1]).toarray()
                D = D + np.kron(T, np.kron(X, V))
            y2 = (D @ u.ravel()).reshape(y.shape)
            assert np.abs(y - y2).max() <= 1e-13 * max(1.0, np.abs(y2).max())


# ------------------------------------------------------------------ weak form
def _beta_fun(cfg):
    d = cfg["d"]

    def poly(p, y):
        return sum(c * np.prod(y ** np.asarray(e)) for e, c in p.items())

    def beta(x, v):
        b = np.zeros(2 * d)
        for ax, a, bb in cfg["beta"]:
            b[ax] += poly(a, x) * poly(bb, v)
        return b
    return beta


@pytest.mark.parametrize("name,q", [("c0_2d_const", 0), ("c0_2d_const", 1), ("c1_2d_rot", 1),
                                    ("c1_2d_rot", 0)])
def test_kron_equals_direct_weak_form_1d(name, q):
    """Kronecker block A_{l,l} == direct quadrature of a_j^(delta)(U, w) (eq. (4)), d = 1.

    a(U,w) = int_I (dtU + b.grad U + s U, w + delta(dtw + b.grad w)) - <U,w>_{Gamma^-} dt
             + (U(t_{j-1}^+), w(t_{j-1}^+)), with sigma set to 0.3 to exercise K, K~."""
    cfg = get_config(name, L=4, q=q, sigma=0.3)
    P = SGProblem(cfg, galerkin="direct")
    tau, delta, sig = P.tau, P.delta, 0.3
    beta = _beta_fun(cfg)
    l = P.active[1]
    mx, mv = P.Hx.meshes[l[0]], P.Hv.meshes[l[1]]
    xs, vs = mx.coords[:, 0], mv.coords[:, 0]
    S = P.S
    n1, n2 = mx.n, mv.n
    N = S * n1 * n2
    A = np.zeros((N, N))
    gq, wq = np.polynomial.legendre.leggauss(4)
    from oracle.problem import dlegendre, legendre

    def idx(s, k, m):
        return (s * n1 + k) * n2 + m

    for i in range(n1 - 1):
        hx = xs[i + 1] - xs[i]
        for k in range(n2 - 1):
            hv = vs[k + 1] - vs[k]
            loc = [(s, a, b) for s in range(S) for a in range(2) for b in range(2)]
            for (qt, wt), (qx, wx), (qv, wv) in itertools.product(zip(gq, wq), zip(gq, wq), zip(gq, wq)):
                x = xs[i] + hx * (qx + 1) / 2; v = vs[k] + hv * (qv + 1) / 2
                w = wt * wx * wv * tau / 2 * hx / 2 * hv / 2
                bt = beta(np.array([x]), np.array([v]))
                px = [(xs[i + 1] - x) / hx, (x - xs[i]) / hx]; dpx = [-1 / hx, 1 / hx]
                pv = [(vs[k + 1] - v) / hv, (v - vs[k]) / hv]; dpv = [-1 / hv, 1 / hv]
                val, L_ = {}, {}
                for (s, a, b) in loc:
                    e, de = legendre(s, qt), dlegendre(s, qt) * 2 / tau
                    f = e * px[a] * pv[b]
                    dtf = de * px[a] * pv[b]
                    dbf = e * (bt[0] * dpx[a] * pv[b] + bt[1] * px[a] * dpv[b])
                    val[(s, a, b)] = (f, dtf + dbf)
                for trial in loc:
                    fU, DU = val[trial]
                    for test in loc:
                        fw, Dw = val[test]
                        A[idx(test[0], i + test[1], k + test[2]), idx(trial[0], i + trial[1], k + trial[2])] += \
                            w * (DU + sig * fU) * (fw + delta * Dw)
    # inflow boundary: -int_I <U,w>_{Gamma^-} = int_I int_{Gamma^-} |beta.n| U w
    for face_axis, s_face in itertools.product((0, 1), (-1, 1)):
        nodes_fixed = 0 if s_face < 0 else (n1 - 1 if face_axis == 0 else n2 - 1)
        other = vs if face_axis == 0 else xs
        for c in range(len(other) - 1):
            hc = other[c + 1] - other[c]
            for (qt, wt), (qy, wy) in itertools.product(zip(gq, wq), zip(gq, wq)):
                y = other[c] + hc * (qy + 1) / 2
                if face_axis == 0:
                    x, v = xs[nodes_fixed], y
                else:
                    x, v = y, vs[nodes_fixed]
                bn = s_face * beta(np.array([x]), np.array([v]))[face_axis]
                if bn >= 0:
                    continue
                w = wt * wy * tau / 2 * hc / 2
                ph = [(other[c + 1] - y) / hc, (y - other[c]) / hc]
                for s1, s2 in itertools.product(range(S), range(S)):
                    e1, e2 = legendre(s1, qt), legendre(s2, qt)
                    for a, b in itertools.product(range(2), range(2)):
                        if face_axis == 0:
                            r_, c_ = idx(s1, nodes_fixed, c + a), idx(s2, nodes_fixed, c + b)
                        else:
                            r_, c_ = idx(s1, c + a, nodes_fixed), idx(s2, c + b, nodes_fixed)
                        A[r_, c_] += w * (-bn) * e1 * e2 * ph[a] * ph[b]
    # jump (U(t_{j-1}^+), w(t_{j-1}^+)) = G^t (x) M
    Mx = np.zeros((n1, n1)); Mv = np.zeros((n2, n2))
    for Mm, zz, n in ((Mx, xs, n1), (Mv, vs, n2)):
        for c in range(n - 1):
            h = zz[c + 1] - zz[c]
            Mm[np.ix_([c, c + 1], [c, c + 1])] += h / 6 * np.array([[2, 1], [1, 2]])
    em = np.array([legendre(s, -1.0) for s in range(S)])
    A += np.kron(np.outer(em, em), np.kron(Mx, Mv))
    K = P.block_matrix(P.terms, l, l).toarray()
    assert np.abs(K - A).max() <= 1e-13 * np.abs(A).max()


# ------------------------------------------------------------ energy identity
def _boxes(spec):
    """Sub-boxes of a factor domain, split at 0 on every axis (|beta.n| is smooth on each)."""
    lo, hi = np.asarray(spec["lo"], float), np.asarray(spec["hi"], float)
    d = lo.size
    cuts = [sorted(set([lo[a], hi[a]] + ([0.0] if lo[a] < 0 < hi[a] else []))) for a in range(d)]
    out = []
    for idx in itertools.product(*[range(len(c) - 1) for c in cuts]):
        blo = np.array([cuts[a][i] for a, i in enumerate(idx)])
        bhi = np.array([cuts[a][i + 1] for a, i in enumerate(idx)])
        if spec["kind"] == "lshape" and (blo[0] + bhi[0]) / 2 > 0 and (blo[1] + bhi[1]) / 2 < 0:
            continue
        out.append((blo, bhi))
    return out


def _gl_box(lo, hi, n=3):
    g, w = np.polynomial.legendre.leggauss(n)
    d = lo.size
    pts, wts = [], []
    for idx in itertools.product(range(n), repeat=d):
        pts.append(lo + (hi - lo) * (g[list(idx)] + 1) / 2)
        wts.append(np.prod(w[list(idx)]) * np.prod((hi - lo) / 2))
    return np.array(pts), np.array(wts)


def _faces(spec, boxes):
    """Boundary (d-1)-faces of the union of boxes: (axis, sign, fixed value, lo, hi)."""
    out = []
    d = len(spec["lo"])
    for bi, (lo, hi) in enumerate(boxes):
        for ax in range(d):
            for s in (-1, 1):
                val = lo[ax] if s < 0 else hi[ax]
                shared = False
                for bj, (lo2, hi2) in enumerate(boxes):
                    if bj == bi:
                        continue
                    v2 = hi2[ax] if s < 0 else lo2[ax]
                    if abs(v2 - val) < 1e-12 and all(abs(lo2[a] - lo[a]) < 1e-12 and abs(hi2[a] - hi[a]) < 1e-12
                                                      for a in range(d) if a != ax):
                        shared = True
                if not shared:
                    out.append((ax, s, val, np.delete(lo, ax), np.delete(hi, ax)))
    return out


@pytest.mark.parametrize("name", ["c2_4d_stream", "c3_4d_lshape", "c0_2d_const", "c1_2d_rot"])
def test_energy_identity(name):
    """U^T A^(delta)_{l,l} U = eq. (11) for one strip (beta divergence free):
    int_I sigma||v||^2 + 1/2 |v|^2_{dOmega} + delta||dtv+dbv||^2 + delta sigma (v, dtv+dbv) dt
    + 1/2||v(t_{j-1}^+)||^2 + 1/2||v(t_j^-)||^2, for v = eta(t) p(x) r(v), p, r affine."""
    cfg = get_config(name, L=3, sigma=0.25)
    P = SGProblem(cfg, galerkin="direct")
    d, S, tau, delta, sig = P.d, P.S, P.tau, P.delta, 0.25
    beta = _beta_fun(cfg)
    l = P.active[0]
    mx, mv = P.Hx.meshes[l[0]], P.Hv.meshes[l[1]]
    rng = np.random.default_rng(11)
    ct = rng.standard_normal(S); ax_ = rng.standard_normal(d); cx = rng.standard_normal()
    av = rng.standard_normal(d); cv = rng.standard_normal()
    U = ct[:, None, None] * np.outer(mx.coords @ ax_ + cx, mv.coords @ av + cv)[None]
    lhs = float(np.vdot(U, P.apply_diag(l, U)))
    from oracle.problem import dlegendre, legendre
    gq, wq = np.polynomial.legendre.leggauss(3)

    def ev(t_xi, x, v):
        e = sum(ct[s] * legendre(s, t_xi) for s in range(S))
        de = sum(ct[s] * dlegendre(s, t_xi) for s in range(S)) * 2 / tau
        p, r = x @ ax_ + cx, v @ av + cv
        b = beta(x, v)
        grad = np.concatenate([ax_ * r, av * p])
        return e * p * r, de * p * r + e * (b @ grad)

    bx, bv = _boxes(cfg["xmesh"]), _boxes(cfg["vmesh"])
    rhs = 0.0
    for (xlo, xhi), (vlo, vhi) in itertools.product(bx, bv):
        X, WX = _gl_box(xlo, xhi); V, WV = _gl_box(vlo, vhi)
        for i, j in itertools.product(range(len(X)), range(len(V))):
            w = WX[i] * WV[j]
            for qt, wt in zip(gq, wq):
                f, D = ev(qt, X[i], V[j])
                rhs += w * wt * tau / 2 * (sig * f * f + delta * D * D + delta * sig * f * D)
            fm, _ = ev(-1.0, X[i], V[j]); fp, _ = ev(1.0, X[i], V[j])
            rhs += w * 0.5 * (fm * fm + fp * fp)
    # 1/2 int_I int_{dOmega} |beta.n| v^2
    for axis_set, boxes_a, boxes_b, is_x in ((0, bx, bv, True), (1, bv, bx, False)):
        for ax, s, val, flo, fhi in _faces(cfg["xmesh"] if is_x else cfg["vmesh"], boxes_a):
            for blo, bhi in boxes_b:
                if d == 1:
                    Fp, FW = np.zeros((1, 0)), np.ones(1)
                else:
                    Fp, FW = _gl_box(flo, fhi)
                Bp, BW = _gl_box(blo, bhi)
                for i, j in itertools.product(range(len(FW)), range(len(BW))):
                    y = np.insert(Fp[i], ax, val)
                    x, v = (y, Bp[j]) if is_x else (Bp[j], y)
                    bn = s * beta(x, v)[ax if is_x else d + ax]
                    for qt, wt in zip(gq, wq):
                        f, _ = ev(qt, x, v)
                        rhs += FW[i] * BW[j] * wt * tau / 2 * 0.5 * abs(bn) * f * f
    assert abs(lhs - rhs) <= 1e-11 * abs(rhs), (lhs, rhs)
