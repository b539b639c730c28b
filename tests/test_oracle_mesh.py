"""Pins of oracle/mesh.py against closed forms and brute force (no GPU)."""
import math

import numpy as np
import pytest

from oracle.mesh import Hierarchy, build_mesh, locate, volumes

BOX1 = dict(kind="box", lo=[0.0], hi=[1.0])
BOX2 = dict(kind="box", lo=[-1.0, -1.0], hi=[1.0, 1.0])
LSH = dict(kind="lshape", lo=[-1.0, -1.0], hi=[1.0, 1.0])
BOX3 = dict(kind="box", lo=[-4.0] * 3, hi=[4.0] * 3)


@pytest.mark.parametrize("spec,d", [(BOX1, 1), (BOX2, 2), (LSH, 2), (BOX3, 3)])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_counts_closed_form(spec, d, level):
    """Node / element counts of the structured Kuhn meshes (2^l cells per axis)."""
    m = build_mesh(spec, 2, level)
    c = 2 ** level
    if spec["kind"] == "lshape":
        assert m.n == (c + 1) ** 2 - (c // 2) ** 2            # quadrant x>0,y<0 removed
        assert m.elems.shape[0] == 2 * (3 * c * c // 4)
    else:
        assert m.n == (c + 1) ** d
        assert m.elems.shape[0] == math.factorial(d) * c ** d
    # volumes sum to |Omega| (independent of the element construction)
    area = {1: 1.0, 2: 4.0}.get(d, 512.0) if spec["kind"] == "box" else 3.0
    assert abs(volumes(m).sum() - area) < 1e-12 * area
    # no degenerate simplices
    assert volumes(m).min() > 0


@pytest.mark.parametrize("spec,d", [(BOX1, 1), (BOX2, 2), (BOX3, 3), (LSH, 2)])
def test_pattern_is_kuhn_stencil(spec, d):
    """Interior rows have 2(2^d - 1) + 1 entries: z and z +- e_S (Kuhn edges)."""
    m = build_mesh(spec, 2, 3)
    rl = np.diff(m.pattern.indptr)
    assert rl.max() == 2 * (2 ** d - 1) + 1
    lat = m.lattice
    cells = m.m - 1
    interior = np.all((lat > 0) & (lat < cells), axis=1)
    if spec["kind"] == "lshape":
        c = cells // 2
        interior &= ~((lat[:, 0] >= c) & (lat[:, 1] <= c))
    assert np.all(rl[interior] == 2 * (2 ** d - 1) + 1)
    # symmetric pattern, diagonal present, sorted rows
    P = m.pattern
    assert (P != P.T).nnz == 0
    assert np.all(P.diagonal() == 1)
    for i in range(m.n):
        cols = P.indices[P.indptr[i]:P.indptr[i + 1]]
        assert np.all(np.diff(cols) > 0)
    # brute force: every pattern pair differs by a 0/+-1 vector with all nonzero entries of one sign
    rows = np.repeat(np.arange(m.n), rl)
    diff = lat[P.indices] - lat[rows]
    ok = np.all(diff >= 0, axis=1) | np.all(diff <= 0, axis=1)
    assert np.all(ok) and np.abs(diff).max() <= 1


@pytest.mark.parametrize("spec", [BOX1, BOX2, LSH, BOX3])
def test_embedding_reproduces_p1_functions(spec):
    """E_{l+1<-l} c represents the same function pointwise (nestedness)."""
    lmax = 3 if spec is not BOX3 else 2
    H = Hierarchy(spec, 2, lmax + 1)
    rng = np.random.default_rng(0)
    for l in range(1, lmax + 1):
        E = H.E1[l]
        assert np.allclose(np.asarray(E.sum(axis=1)).ravel(), 1.0, atol=1e-15)
        vals = np.unique(E.data)
        assert set(np.round(vals, 15)).issubset({0.5, 1.0})
        c = rng.standard_normal(H.n(l))
        f = E @ c
        # random points inside the domain
        pts = H.meshes[l + 1].coords[rng.integers(0, H.n(l + 1), 40)]
        pts = pts + 0.3 * H.meshes[l + 1].h * (rng.random(pts.shape) - 0.5)
        lo, hi = H.meshes[l].lo, H.meshes[l].hi
        pts = np.clip(pts, lo, hi)
        if spec["kind"] == "lshape":
            bad = (pts[:, 0] > 0) & (pts[:, 1] < 0)
            pts = pts[~bad]
        vc, lc = locate(H.meshes[l], pts)
        vf, lf = locate(H.meshes[l + 1], pts)
        assert np.allclose((c[vc] * lc).sum(1), (f[vf] * lf).sum(1), atol=1e-12)
        # affine functions are reproduced exactly
        a = rng.standard_normal(H.meshes[l].d)
        assert np.allclose(E @ (H.meshes[l].coords @ a + 0.7), H.meshes[l + 1].coords @ a + 0.7, atol=1e-13)


def test_embedding_composition_and_adjoint():
    H = Hierarchy(BOX2, 2, 4)
    rng = np.random.default_rng(1)
    c = rng.standard_normal(H.n(1)); dd = rng.standard_normal(H.n(4))
    E = H.E(4, 1)
    assert abs(dd @ (E @ c) - (E.T @ dd) @ c) < 1e-12 * np.abs(dd).sum() * np.abs(c).sum()
    assert np.allclose((H.E1[3] @ (H.E1[2] @ (H.E1[1] @ c))), E @ c, atol=1e-14)
