"""Direct-quadrature pins of SGProblem.l2_inner (the strip solver's stopping norm) and
SGProblem.inflow_load (reading R9), no GPU.

Both references evaluate the sparse-grid / boundary functions pointwise with an explicit
1D hat-function formula and integrate with Gauss rules on the finest cells; they use no
matrix of oracle/fem.py, no embedding E and no term list (d = 1 configurations, where the
factor meshes are intervals)."""
import numpy as np
import pytest

from oracle.problem import legendre
from oracle.sgrid import SGProblem
from sginputs import get_config


def _hat(nodes, k, y):
    """phi_k(y) on the uniform 1D mesh `nodes` (explicit formula)."""
    h = nodes[1] - nodes[0]
    return np.maximum(0.0, 1.0 - np.abs(y - nodes[k]) / h)


def _eval_block(P, l, u_s, x, v):
    """sum_{k1,k2} u_s[k1,k2] phi_k1(x) phi_k2(v) on the tensor points x (nx,), v (nv,)."""
    xn = P.Hx.meshes[l[0]].coords[:, 0]
    vn = P.Hv.meshes[l[1]].coords[:, 0]
    Px = np.stack([_hat(xn, k, x) for k in range(xn.size)])      # (n1, nx)
    Pv = np.stack([_hat(vn, k, v) for k in range(vn.size)])      # (n2, nv)
    return Px.T @ u_s @ Pv                                        # (nx, nv)


def _fine_gauss(P, which, nq):
    """Gauss points / weights on every cell of the finest mesh of one factor."""
    mesh = (P.Hx if which == "x" else P.Hv).meshes[P.F]
    nodes = mesh.coords[:, 0]
    g, w = np.polynomial.legendre.leggauss(nq)
    pts, wts = [], []
    for a, b in zip(nodes[:-1], nodes[1:]):
        pts.append(0.5 * (a + b) + 0.5 * (b - a) * g)
        wts.append(0.5 * (b - a) * w)
    return np.concatenate(pts), np.concatenate(wts)


@pytest.mark.parametrize("name,L", [("c1_2d_rot", 4), ("c0_2d_const", 5)])
def test_l2_inner_direct_quadrature(name, L):
    """(U, W)_{L2(I_j x Omega)} of two random sparse-grid functions of P^q(I_j, V_L) ==
    Gauss quadrature in (t, x, v) of the pointwise product (exact: piecewise polynomial
    integrands of degree <= 2 per direction on the finest cells, 3 points each)."""
    P = SGProblem(get_config(name, L=L))
    rng = np.random.default_rng(5)
    U = {l: rng.standard_normal(P.shape(l)) for l in P.active}
    W = {l: rng.standard_normal(P.shape(l)) for l in P.active}
    got = P.l2_inner(U, W)
    xq, xw = _fine_gauss(P, "x", 3)
    vq, vw = _fine_gauss(P, "v", 3)
    tg, tw = np.polynomial.legendre.leggauss(3)
    tw = tw * P.tau / 2
    ref = 0.0
    for mu in range(tg.size):
        eta = [float(legendre(s, tg[mu])) for s in range(P.S)]
        fu = sum(eta[s] * _eval_block(P, l, U[l][s], xq, vq) for l in P.active for s in range(P.S))
        fw = sum(eta[s] * _eval_block(P, l, W[l][s], xq, vq) for l in P.active for s in range(P.S))
        ref += tw[mu] * np.einsum("i,j,ij->", xw, vw, fu * fw)
    assert abs(got - ref) <= 1e-12 * abs(ref), (got, ref)


def _inflow_reference(P, t0, interpolate):
    """-int_{I_j} eta_s <g, phi_k phi_m>_{Gamma^-} dt by quadrature on the faces of the unit
    square (constant beta, d = 1).  interpolate=True: g(tau_mu, .) replaced by its nodal
    interpolant on the finest face mesh at the 4 Gauss times tau_mu (reading R9, the
    oracle's definition, evaluated independently); False: the exact g, 8-point Gauss in t."""
    cfg = P.cfg
    beta = P.beta_const()
    (c, gx, gv), = cfg["u0"]
    fx = lambda y: gx["scale"] * np.exp(-(y - gx["center"][0]) ** 2 / gx["w"])
    fv = lambda y: gv["scale"] * np.exp(-(y - gv["center"][0]) ** 2 / gv["w"])
    nt = 4 if interpolate else 8
    tg, tw = np.polynomial.legendre.leggauss(nt)
    tq, tw = t0 + P.tau * (tg + 1) / 2, tw * P.tau / 2
    out = {l: np.zeros(P.shape(l)) for l in P.active}
    xF = P.Hx.meshes[P.F].coords[:, 0]
    vF = P.Hv.meshes[P.F].coords[:, 0]
    xq, xw = _fine_gauss(P, "x", 6)
    vq, vw = _fine_gauss(P, "v", 6)

    def along(nodes_F, f, q):   # g on the face at points q (interpolated on the finest face mesh or exact)
        if not interpolate:
            return f(q)
        vals = f(nodes_F)
        return sum(vals[k] * _hat(nodes_F, k, q) for k in range(nodes_F.size))

    for mu in range(nt):
        t = tq[mu]
        eta = np.array([float(legendre(s, tg[mu])) for s in range(P.S)])
        # faces x = 0 / x = 1 (normal -e_x / +e_x), g(t, x_f, v) = c fx(x_f - b0 t) fv(v - b1 t)
        for sgn, xf in ((-1, 0.0), (1, 1.0)):
            bn = sgn * beta[0]
            if bn >= 0:
                continue
            gvals = c * fx(xf - beta[0] * t) * along(vF, lambda y: fv(y - beta[1] * t), vq)
            for l in P.active:
                vn = P.Hv.meshes[l[1]].coords[:, 0]
                k1 = 0 if sgn < 0 else P.Hx.n(l[0]) - 1
                for k2 in range(vn.size):
                    val = np.sum(vw * gvals * _hat(vn, k2, vq))
                    out[l][:, k1, k2] += -bn * tw[mu] * eta * val
        # faces v = 0 / v = 1
        for sgn, vf in ((-1, 0.0), (1, 1.0)):
            bn = sgn * beta[1]
            if bn >= 0:
                continue
            gvals = c * fv(vf - beta[1] * t) * along(xF, lambda y: fx(y - beta[0] * t), xq)
            for l in P.active:
                xn = P.Hx.meshes[l[0]].coords[:, 0]
                k2 = 0 if sgn < 0 else P.Hv.n(l[1]) - 1
                for k1 in range(xn.size):
                    val = np.sum(xw * gvals * _hat(xn, k1, xq))
                    out[l][:, k1, k2] += -bn * tw[mu] * eta * val
    return out


@pytest.mark.parametrize("q", [0, 1])
def test_inflow_load_direct_quadrature(q):
    """configs[0] (and the same data with dG(1)): SGProblem.inflow_load on strip 3 equals
    (a) the same functional (reading R9) evaluated independently to 1e-12, and (b) the exact
    boundary integral of the unmodified g within the interpolation error (a wide Gaussian,
    w = 0.5, so that the O(h_F^2) term is < 1e-3 of the load)."""
    cfg = get_config("c0_2d_const", L=6, q=q)
    P = SGProblem(cfg)
    t0 = 2 * P.tau
    got = P.inflow_load(t0)
    ref = _inflow_reference(P, t0, interpolate=True)
    scale = max(np.abs(ref[l]).max() for l in P.active)
    assert scale > 0
    for l in P.active:
        assert np.abs(got[l] - ref[l]).max() <= 1e-12 * scale, l
    wide = get_config("c0_2d_const", L=6, q=q)
    wide["u0"] = [(1.0, dict(center=[0.3], w=0.5, scale=1.0), dict(center=[0.3], w=0.5, scale=1.0))]
    Pw = SGProblem(wide)
    gw = Pw.inflow_load(t0)
    ex = _inflow_reference(Pw, t0, interpolate=False)
    sc = max(np.abs(ex[l]).max() for l in Pw.active)
    for l in Pw.active:
        assert np.abs(gw[l] - ex[l]).max() <= 1e-3 * sc, l
