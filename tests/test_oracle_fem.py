"""Pins of oracle/fem.py: exact factor matrices vs closed forms computed by an
independent method (tensor Gauss-Legendre over boxes), invariants, and the
Galerkin identity of PAPER.md l.506-509 (no GPU)."""
import itertools
import math

import numpy as np
import pytest

from oracle.fem import assemble, duffy_rule, face, load_vector, vol
from oracle.mesh import Hierarchy, build_mesh

SPECS = {
    "box1": dict(kind="box", lo=[-2.0], hi=[2.0]),
    "box2": dict(kind="box", lo=[0.0, -1.0], hi=[1.0, 1.0]),
    "lsh": dict(kind="lshape", lo=[-1.0, -1.0], hi=[1.0, 1.0]),
    "box3": dict(kind="box", lo=[-4.0, 0.0, -1.0], hi=[4.0, 1.0, 1.0]),
}


def boxes_of(spec):
    lo, hi = np.asarray(spec["lo"]), np.asarray(spec["hi"])
    if spec["kind"] == "lshape":
        return [([-1, -1], [0, 0]), ([-1, 0], [0, 1]), ([0, 0], [1, 1])]
    return [(lo, hi)]


def integrate(spec, f, n=4):
    """int_Omega f by tensor Gauss-Legendre on the boxes making up Omega (exact for poly deg <= 7)."""
    x, w = np.polynomial.legendre.leggauss(n)
    tot = 0.0
    for lo, hi in boxes_of(spec):
        lo, hi = np.asarray(lo, float), np.asarray(hi, float)
        d = lo.size
        for idx in itertools.product(range(n), repeat=d):
            y = lo + (hi - lo) * (x[list(idx)] + 1) / 2
            ww = np.prod(w[list(idx)]) * np.prod((hi - lo) / 2)
            tot += ww * f(y)
    return tot


def faces_of(spec, axis, sign):
    """(d-1)-boxes of the boundary part with outward normal sign*e_axis: (fixed value, lo, hi)."""
    if spec["kind"] == "lshape":
        table = {
            (0, -1): [(-1.0, [-1.0], [1.0])],
            (0, 1): [(1.0, [0.0], [1.0]), (0.0, [-1.0], [0.0])],
            (1, -1): [(-1.0, [-1.0], [0.0]), (0.0, [0.0], [1.0])],
            (1, 1): [(1.0, [-1.0], [1.0])],
        }
        return table[(axis, sign)]
    lo, hi = np.asarray(spec["lo"]), np.asarray(spec["hi"])
    others = [a for a in range(lo.size) if a != axis]
    val = lo[axis] if sign < 0 else hi[axis]
    return [(val, lo[others], hi[others])]


def face_integrate(spec, axis, sign, f, n=4):
    x, w = np.polynomial.legendre.leggauss(n)
    d = len(spec["lo"])
    tot = 0.0
    for val, flo, fhi in faces_of(spec, axis, sign):
        flo, fhi = np.asarray(flo, float), np.asarray(fhi, float)
        if d == 1:
            tot += f(np.array([val]))
            continue
        for idx in itertools.product(range(n), repeat=d - 1):
            yo = flo + (fhi - flo) * (x[list(idx)] + 1) / 2
            y = np.insert(yo, axis, val)
            tot += np.prod(w[list(idx)]) * np.prod((fhi - flo) / 2) * f(y)
    return tot


def affine(rng, d):
    a = rng.standard_normal(d); c = rng.standard_normal()
    return a, c, (lambda y: float(a @ y + c))


@pytest.fixture(scope="module")
def meshes():
    return {k: build_mesh(s, 2, 2) for k, s in SPECS.items()}


@pytest.mark.parametrize("key", list(SPECS))
def test_mass_exact(meshes, key):
    """(a) 1^T M 1 = |Omega|; u^T M w = int u w for affine u, w."""
    m = meshes[key]; spec = SPECS[key]; d = m.d
    M = assemble(m, vol({(0,) * d: 1.0}))
    assert abs(M.sum() - integrate(spec, lambda y: 1.0)) < 1e-12
    assert abs(M - M.T).max() < 1e-15
    rng = np.random.default_rng(2)
    a, c, u = affine(rng, d); b, e, w = affine(rng, d)
    U = m.coords @ a + c; W = m.coords @ b + e
    ref = integrate(spec, lambda y: u(y) * w(y))
    assert abs(W @ M @ U - ref) < 1e-12 * max(1, abs(ref))


@pytest.mark.parametrize("key", list(SPECS))
def test_derivative_and_stiffness(meshes, key):
    """(b) derivative matrices annihilate constants; exact on affine functions."""
    m = meshes[key]; spec = SPECS[key]; d = m.d
    one = {(0,) * d: 1.0}
    rng = np.random.default_rng(3)
    a, c, u = affine(rng, d); b, e, w = affine(rng, d)
    U = m.coords @ a + c; W = m.coords @ b + e
    ones = np.ones(m.n)
    for p in range(d):
        D = assemble(m, vol(one, trial_d=p))                 # int d_p phi' phi
        assert np.abs(D @ ones).max() < 1e-13
        ref = integrate(spec, lambda y: a[p] * w(y))
        assert abs(W @ D @ U - ref) < 1e-12 * max(1, abs(ref))
        Dt = assemble(m, vol(one, test_d=p))
        assert abs(Dt - D.T).max() < 1e-15
        for q in range(d):
            K = assemble(m, vol(one, trial_d=p, test_d=q))   # int d_p phi' d_q phi
            assert np.abs(K @ ones).max() < 1e-12 and np.abs(ones @ K).max() < 1e-12
            ref = a[p] * b[q] * integrate(spec, lambda y: 1.0)
            assert abs(W @ K @ U - ref) < 1e-12 * max(1, abs(ref))


@pytest.mark.parametrize("key", list(SPECS))
def test_weighted_exact(meshes, key):
    """Weights y_i, y_i y_j (the v_k, v_k v_l of the north star) and chi-weights, exact."""
    m = meshes[key]; spec = SPECS[key]; d = m.d
    rng = np.random.default_rng(4)
    a, c, u = affine(rng, d); b, e, w = affine(rng, d)
    U = m.coords @ a + c; W = m.coords @ b + e
    for i in range(d):
        ei = tuple(1 if k == i else 0 for k in range(d))
        V = assemble(m, vol({ei: 1.0}))
        ref = integrate(spec, lambda y: y[i] * u(y) * w(y))
        assert abs(W @ V @ U - ref) < 1e-12 * max(1, abs(ref))
        for j in range(d):
            eij = tuple(int(k == i) + int(k == j) for k in range(d))
            Wm = assemble(m, vol({eij: 1.0}))
            ref = integrate(spec, lambda y: y[i] * y[j] * u(y) * w(y))
            assert abs(W @ Wm @ U - ref) < 1e-11 * max(1, abs(ref))
            # weighted derivative (a_r a_r' d phi' phi-type terms)
            Dw = assemble(m, vol({ei: 1.0}, trial_d=j))
            ref = integrate(spec, lambda y: y[i] * a[j] * w(y))
            assert abs(W @ Dw @ U - ref) < 1e-12 * max(1, abs(ref))
        for s in (-1, 1):
            X = assemble(m, vol({ei: 1.0}, chi=(i, s)))
            ref = integrate(spec, lambda y: (s * y[i] > 0) * y[i] * u(y) * w(y), n=6) if spec["kind"] != "lshape" else None
            if ref is not None and m.lo[i] < 0 < m.hi[i] and abs(round(-m.lo[i] / m.h[i]) - (-m.lo[i] / m.h[i])) < 1e-12:
                # split the box at y_i = 0 so the indicator is smooth on each part
                lo, hi = np.array(spec["lo"], float), np.array(spec["hi"], float)
                part = dict(kind="box", lo=lo.copy(), hi=hi.copy())
                if s > 0:
                    part["lo"][i] = 0.0
                else:
                    part["hi"][i] = 0.0
                ref = integrate(part, lambda y: y[i] * u(y) * w(y))
                assert abs(W @ X @ U - ref) < 1e-12 * max(1, abs(ref))


@pytest.mark.parametrize("key", list(SPECS))
def test_face_mass(meshes, key):
    """Boundary factor of G^(r): int_{Gamma_{s e_i}} u w ds exact for affine u, w."""
    m = meshes[key]; spec = SPECS[key]; d = m.d
    rng = np.random.default_rng(5)
    a, c, u = affine(rng, d); b, e, w = affine(rng, d)
    U = m.coords @ a + c; W = m.coords @ b + e
    for ax in range(d):
        for s in (-1, 1):
            F = assemble(m, face(ax, s))
            ref = face_integrate(spec, ax, s, lambda y: u(y) * w(y))
            assert abs(W @ F @ U - ref) < 1e-12 * max(1, abs(ref))
            meas = face_integrate(spec, ax, s, lambda y: 1.0)
            assert abs(F.sum() - meas) < 1e-12


@pytest.mark.parametrize("key", ["box1", "lsh", "box2", "box3"])
def test_galerkin_identity(key):
    """A_{l,l'} = E_{F,l}^T A_{F,F} E_{F,l'} equals the direct
    assembly on level l, and A_l E_{l<-l'} / E^T A_l' for the cross levels."""
    spec = SPECS[key]
    F = 3 if key != "box3" else 2
    H = Hierarchy(spec, 2, F)
    d = len(spec["lo"])
    e0 = tuple(1 if k == 0 else 0 for k in range(d))
    specs = [vol({(0,) * d: 1.0}), vol({e0: 1.0}, trial_d=d - 1),
             vol({(0,) * d: 1.0}, trial_d=0, test_d=d - 1), face(0, -1),
             vol({e0: 2.0}, chi=(0, 1))]
    for sp_ in specs:
        AF = assemble(H.meshes[F], sp_)
        for l in range(1, F + 1):
            A = assemble(H.meshes[l], sp_)
            G = H.E(F, l).T @ AF @ H.E(F, l)
            assert abs(G - A).max() < 1e-13 * max(1, abs(A).max())
            for lp in range(1, F + 1):
                cross = H.E(F, l).T @ AF @ H.E(F, lp)
                Alp = assemble(H.meshes[lp], sp_)
                alt = A @ H.E(l, lp) if l >= lp else H.E(lp, l).T @ Alp
                assert abs(cross - alt).max() < 1e-13 * max(1, abs(A).max())


@pytest.mark.parametrize("d", [1, 2, 3])
def test_duffy_rule_exact(d):
    """Collapsed GL rule: weights sum to 1/d!, exact for monomials of degree <= 5."""
    xi, w = duffy_rule(d)
    assert abs(w.sum() - 1 / math.factorial(d)) < 1e-15
    for expo in itertools.product(range(4), repeat=d):
        if sum(expo) > 5:
            continue
        # int_{ref simplex} xi^a = a! / (d + |a|)!  (Dirichlet integral)
        ref = np.prod([math.factorial(k) for k in expo]) / math.factorial(d + sum(expo))
        got = np.sum(w * np.prod(xi ** np.asarray(expo), axis=1))
        assert abs(got - ref) < 1e-15


def test_load_vector_polynomial():
    """sum_k l_k = int f for polynomial f (partition of unity + rule exactness)."""
    for key in SPECS:
        spec = SPECS[key]; m = build_mesh(spec, 2, 2)
        f = lambda Y: 1.0 + Y[:, 0] ** 2 - 0.5 * Y[:, -1]
        lvec = load_vector(m, f)
        ref = integrate(spec, lambda y: 1.0 + y[0] ** 2 - 0.5 * y[-1])
        assert abs(lvec.sum() - ref) < 1e-12 * abs(ref)
