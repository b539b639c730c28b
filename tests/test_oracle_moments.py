"""Pin of the shifted-moment reading used by the GPU pass-1 kernel (DESIGN.md sec. 5,
`vmoment.cu`), checked on the ORACLE's exact matrices only (no GPU, no product code).

For a monomial weight y^n (|n| <= 2) the weighted P1 mass row of node a satisfies
    int y^n phi_a phi_b = sum_{m <= n} binom(n, m) y_a^(n-m) R_m^{cls(a)}[b - a],
    R_m^{cls}[k] = int (y - y_a)^m phi_a phi_{a+off_k} dy,
where R_m depends only on the boundary class of a (per axis: low face, interior,
high face) and scales as prod_q h_q^(1 + m_q) under uniform refinement.  The test
derives R_m from the level-1 lattice (one node per class, as the GPU setup does)
and reconstructs every row of the level-3 weighted masses, and the chi-weighted
inflow masses int y_i chi(s y_i > 0) phi phi (rows on the kept side = the y_i
row, on the other side zero, on the plane y_i = 0 the half stencil)."""
import itertools

import numpy as np
import pytest

from oracle.fem import assemble, vol
from oracle.mesh import build_mesh

DOMS = {
    2: dict(kind="box", lo=[-1.0, -1.0], hi=[1.0, 1.0]),
    3: dict(kind="box", lo=[-4.0, -4.0, -4.0], hi=[4.0, 4.0, 4.0]),
}


def monos(d):
    out = [()]
    out += [(i,) for i in range(d)]
    out += [(i, j) for i in range(d) for j in range(i, d)]
    return out


def expo(mono, d):
    e = [0] * d
    for a in mono:
        e[a] += 1
    return tuple(e)


def weight_of(mono, d):
    return {expo(mono, d): 1.0} if mono else {tuple([0] * d): 1.0}


def cls_of(z, m):
    return tuple(0 if zq == 0 else (2 if zq == m - 1 else 1) for zq in z)


def offsets(d):
    """Kuhn neighbour offsets: +-(sum of a subset of axes)."""
    offs = set()
    for r in range(d + 1):
        for sub in itertools.combinations(range(d), r):
            o = np.zeros(d, int)
            o[list(sub)] = 1
            offs.add(tuple(o))
            offs.add(tuple(-o))
    return sorted(offs)


def row_stencil(A, mesh, a, offs):
    z = mesh.lattice[a]
    out = np.zeros(len(offs))
    for k, o in enumerate(offs):
        zz = tuple(int(v) for v in z + np.asarray(o))
        b = mesh.node_id.get(zz)
        if b is not None:
            out[k] = A[a, b]
    return out


def shifted(M, mono, y):
    """R_m row from absolute-monomial rows M[n] at node coordinate y (exact identities)."""
    if len(mono) == 0:
        return M[()]
    if len(mono) == 1:
        (i,) = mono
        return M[(i,)] - y[i] * M[()]
    i, j = mono
    if i == j:
        return M[(i, i)] - 2 * y[i] * M[(i,)] + y[i] ** 2 * M[()]
    return M[(i, j)] - y[j] * M[(i,)] - y[i] * M[(j,)] + y[i] * y[j] * M[()]


def recon(R, mono, y):
    if len(mono) == 0:
        return R[()]
    if len(mono) == 1:
        (i,) = mono
        return y[i] * R[()] + R[(i,)]
    i, j = mono
    if i == j:
        return y[i] ** 2 * R[()] + 2 * y[i] * R[(i,)] + R[(i, i)]
    return y[i] * y[j] * R[()] + y[i] * R[(j,)] + y[j] * R[(i,)] + R[(i, j)]


@pytest.mark.parametrize("d,level", [(2, 3), (3, 2)])
def test_shifted_moments_reconstruct_weighted_masses(d, level):
    spec = DOMS[d]
    offs = offsets(d)
    m1 = build_mesh(spec, 2, 1)
    ml = build_mesh(spec, 2, level)
    ms = monos(d)
    A1 = {mo: assemble(m1, vol(weight_of(mo, d))).tocsr() for mo in ms}
    Al = {mo: assemble(ml, vol(weight_of(mo, d))).tocsr() for mo in ms}
    # level-1 class tables
    R1 = {}
    for a in range(m1.n):
        c = cls_of(m1.lattice[a], m1.m)
        rows = {mo: row_stencil(A1[mo], m1, a, offs) for mo in ms}
        R1[c] = {mo: shifted(rows, mo, m1.coords[a]) for mo in ms}
    ratio = ml.h / m1.h
    worst = 0.0
    for a in range(ml.n):
        c = cls_of(ml.lattice[a], ml.m)
        y = ml.coords[a]
        R = {mo: R1[c][mo] * np.prod(ratio) * np.prod([ratio[q] for q in mo]) for mo in ms}
        for mo in ms:
            ref = row_stencil(Al[mo], ml, a, offs)
            got = recon(R, mo, y)
            scale = max(np.abs(Al[mo]).max(), 1e-300)
            worst = max(worst, np.abs(got - ref).max() / scale)
    assert worst <= 1e-13, worst


@pytest.mark.parametrize("axis,sign", [(0, 1), (1, -1)])
def test_chi_weighted_rows(axis, sign):
    d, level = 2, 3
    spec = DOMS[d]
    offs = offsets(d)
    m1 = build_mesh(spec, 2, 1)
    ml = build_mesh(spec, 2, level)
    w = {expo((axis,), d): 1.0}
    chi1 = assemble(m1, vol(w, chi=(axis, sign))).tocsr()
    chil = assemble(ml, vol(w, chi=(axis, sign))).tocsr()
    plain = assemble(ml, vol(w)).tocsr()
    half = {}
    for a in range(m1.n):
        if m1.lattice[a][axis] == 1:            # the plane y_axis = 0 of the level-1 lattice
            half[cls_of(m1.lattice[a], m1.m)] = row_stencil(chi1, m1, a, offs)
    ratio = ml.h / m1.h
    for a in range(ml.n):
        y = ml.coords[a]
        ref = row_stencil(chil, ml, a, offs)
        if sign * y[axis] > 0:
            got = row_stencil(plain, ml, a, offs)
        elif y[axis] == 0.0:
            got = half[cls_of(ml.lattice[a], ml.m)] * np.prod(ratio) * ratio[axis]
        else:
            got = np.zeros(len(offs))
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(plain).max(), a
