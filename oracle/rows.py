"""Sampled rows of factor matrices and of the strip operator on large levels (oracle).

TEST INFRASTRUCTURE ONLY: imported by tests/, never by the product path.

A P1 factor matrix row F[k, :] (eq. (14) l.450-461, factorised as in
l.484-504) is an integral over the elements in the support of phi_k.  On levels
too large to assemble whole (the level-7 factors of configs[4], 2.1 M nodes),
row k is assembled exactly on the PATCH of k: the global cells that have k as a
corner (same absolute coordinates, same Kuhn split, `mesh.build_mesh`'s
definitions), so every element containing k is present and `fem.assemble`
returns the global row.  Face integrals over patch facets that are not on the
domain boundary do not contain k (they lie on the planes z_k +- 1 where
phi_k = 0) and add nothing to row k.  Box lattices only (the large levels of
the configs are boxes).

`sampled_apply` evaluates y = sum_t (T_t x A_t x B_t) X (l.462-477) at the
outer product of sampled x-rows and v-rows, with each factor either assembled
whole (small levels) or by patch rows.  Pinned against whole assembly and
`SGProblem.apply_pair` in tests/test_oracle_rows.py.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

from .fem import assemble
from .mesh import Mesh, build_mesh, element_pattern


def _box_params(spec: dict, nc: int, level: int):
    lo = np.asarray(spec["lo"], float)
    hi = np.asarray(spec["hi"], float)
    cells = nc * 2 ** (level - 1)
    return lo, hi, cells, cells + 1, (hi - lo) / cells


def build_patches(spec: dict, nc: int, level: int, centers: np.ndarray):
    """Disjoint union of the patches of the lattice nodes `centers` (ncent, d).

    Returns (mesh, center_local_ids, local_to_global)."""
    assert spec["kind"] == "box"
    lo, hi, cells, m, h = _box_params(spec, nc, level)
    d = lo.size
    perms = list(itertools.permutations(range(d)))
    lat, elems, cids = [], [], []
    for z in np.asarray(centers, dtype=np.int64).tolist():
        local = {}

        def nid(v):
            v = tuple(v)
            if v not in local:
                local[v] = len(lat)
                lat.append(v)
            return local[v]

        corners = [[c for c in (zk - 1, zk) if 0 <= c <= cells - 1] for zk in z]
        for cell in itertools.product(*corners):
            for pi in perms:
                v = list(cell)
                verts = [nid(v)]
                for ax in pi:
                    v[ax] += 1
                    verts.append(nid(v))
                elems.append(verts)
        cids.append(local[tuple(z)])
    lattice = np.asarray(lat, dtype=np.int64)
    coords = lo + lattice * h
    elems = np.asarray(elems, dtype=np.int64)
    mesh = Mesh("box", d, level, lo, hi, m, h, lattice, coords, {}, elems)
    mesh.pattern = element_pattern(mesh)
    mesh.ecoords = coords[elems]
    strides = m ** np.arange(d)
    return mesh, np.asarray(cids), lattice @ strides


def factor_rows(spec: dict, nc: int, level: int, nodes: np.ndarray, matspec) -> sp.csr_matrix:
    """Rows `nodes` (global node ids, box lattice) of the factor matrix `matspec` at `level`,
    as a (len(nodes) x n) CSR matrix with global column ids."""
    lo, hi, cells, m, h = _box_params(spec, nc, level)
    d = lo.size
    nodes = np.asarray(nodes, dtype=np.int64)
    centers = np.stack([(nodes // m ** k) % m for k in range(d)], axis=1)
    mesh, cid, l2g = build_patches(spec, nc, level, centers)
    F = assemble(mesh, matspec).tocsr()
    R = F[cid].tocoo()
    return sp.csr_matrix((R.data, (R.row, l2g[R.col])), shape=(len(nodes), m ** d))


class FactorRows:
    """Row access to the factor matrices of one factor at one level: whole assembly when
    the level is small, patch rows otherwise."""

    def __init__(self, spec: dict, nc: int, level: int, rows: np.ndarray, whole_max: int = 40000):
        self.spec, self.nc, self.level = spec, nc, level
        self.rows = np.asarray(rows, dtype=np.int64)
        lo, hi, cells, m, h = _box_params(spec, nc, level) if spec["kind"] == "box" else (None,) * 5
        self.mesh = None
        if spec["kind"] != "box" or m ** lo.size <= whole_max:
            self.mesh = build_mesh(spec, nc, level)
        self._cache = {}

    def get(self, matspec) -> sp.csr_matrix:
        if matspec not in self._cache:
            if self.mesh is not None:
                self._cache[matspec] = assemble(self.mesh, matspec).tocsr()[self.rows]
            else:
                self._cache[matspec] = factor_rows(self.spec, self.nc, self.level, self.rows, matspec)
        return self._cache[matspec]


def sampled_apply(cfg: dict, terms, l, X: np.ndarray, xrows, vrows) -> np.ndarray:
    """y[s, i, a] = [sum_t (T_t x A_t x B_t) X]_{s, xrows[i], vrows[a]} on grid l = (l1, l2)
    (the diagonal block A^(delta)_{l,l}, l = l' so every factor lives on the grid's own level)."""
    S = X.shape[0]
    Ax = FactorRows(cfg["xmesh"], cfg["nc"], l[0], xrows)
    Bv = FactorRows(cfg["vmesh"], cfg["nc"], l[1], vrows)
    n1, n2 = X.shape[1], X.shape[2]
    y = np.zeros((S, len(xrows), len(vrows)))
    for T, xs, vs in terms:
        A = Ax.get(xs)
        B = Bv.get(vs)
        for sp_ in range(S):
            # W = A X B^T, through the smaller intermediate
            if len(xrows) * n2 <= n1 * len(vrows):
                W = np.asarray(B @ np.asarray(A @ X[sp_]).T).T
            else:
                W = np.asarray(A @ np.asarray(B @ X[sp_].T).T)
            for s in range(S):
                if T[s, sp_] != 0.0:
                    y[s] += T[s, sp_] * W
    return y
