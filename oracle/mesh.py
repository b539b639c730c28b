"""Nested structured P1 meshes on one factor domain Omega^(i) (oracle).

PAPER.md sec. 2 l.64-67: "V^(i)_1 subset V^(i)_2 subset ... by uniform
refinement" of conforming finite element spaces on polyhedral Omega^(i).
BASELINE configs: uniform 1D meshes of 2^l cells; structured P1 triangulations
(squares split along one diagonal); the L-shape [-1,1]^2 minus [0,1]x[-1,0];
Kuhn subdivision (6 tetrahedra per cube) in 3D.  All are the Kuhn (Freudenthal)
triangulation of a box lattice, which is nested under halving.

Definitions used here (plain; written for readability, not speed):
  * level l: nc * 2**(l-1) cells per axis, lattice nodes m = cells + 1 per axis;
  * a lattice node z (integer vector) is in the mesh iff it lies in the closed
    domain; for the L-shape the open quadrant {x>0, y<0} is removed;
  * node numbering: lexicographic in z with axis 0 fastest, skipping absent nodes;
  * a cell (lower corner z) is in the mesh iff its centre lies in the domain;
    each cell is split into d! Kuhn simplices, one per permutation pi of the
    axes (itertools order), with vertices v0 = z, v_k = v_{k-1} + e_{pi(k)};
  * the sparsity pattern of every factor matrix is {(a, b): a, b vertices of a
    common simplex} (the P1 stiffness/mass pattern), rows sorted ascending;
  * the embedding E_{l+1 <- l}[f, c] = phi^{(l)}_c(x_f), the coarse basis
    function evaluated at the fine node ("matrix representation
    of the embedding from V_l' in V_l").
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass
class Mesh:
    kind: str
    d: int
    level: int
    lo: np.ndarray
    hi: np.ndarray
    m: int                       # lattice nodes per axis
    h: np.ndarray                # cell edge per axis
    lattice: np.ndarray          # (n, d) int lattice coords of nodes, in node order
    coords: np.ndarray           # (n, d) float coordinates
    node_id: dict                # tuple(lattice) -> node index
    elems: np.ndarray            # (ne, d+1) node indices (Kuhn vertex order)
    pattern: sp.csr_matrix = field(default=None)  # boolean sparsity, sorted
    ecoords: np.ndarray = field(default=None)     # (ne, d+1, d) element vertex coordinates

    @property
    def n(self) -> int:
        return self.lattice.shape[0]


def _in_domain_closed(kind: str, frac: np.ndarray) -> np.ndarray:
    """frac: (..., d) point coordinates in [0,1]^d relative to the bounding box."""
    ok = np.all((frac >= -1e-12) & (frac <= 1 + 1e-12), axis=-1)
    if kind == "lshape":
        # removed: open quadrant x > 0, y < 0  (x = frac0 > 1/2, y = frac1 < 1/2)
        ok &= ~((frac[..., 0] > 0.5 + 1e-12) & (frac[..., 1] < 0.5 - 1e-12))
    return ok


def build_mesh(spec: dict, nc: int, level: int) -> Mesh:
    """Structured Kuhn P1 mesh of one factor domain at `level`."""
    kind = spec["kind"]
    lo = np.asarray(spec["lo"], float)
    hi = np.asarray(spec["hi"], float)
    d = lo.size
    cells = nc * 2 ** (level - 1)
    m = cells + 1
    h = (hi - lo) / cells
    if kind == "periodic":
        # 1D periodic interval (only for the paper's Table 1 pin, sec. 5.1 l.585):
        # node cells == node 0, element i = (i, i+1 mod cells)
        assert d == 1
        lattice = np.arange(cells)[:, None]
        node_id = {(i,): i for i in range(cells)}
        node_id[(cells,)] = 0
        coords = lo + lattice * h
        elems = np.array([[i, (i + 1) % cells] for i in range(cells)], dtype=np.int64)
        mesh = Mesh(kind, d, level, lo, hi, m, h, lattice, coords, node_id, elems)
        mesh.pattern = element_pattern(mesh)
        ii = np.arange(cells)
        mesh.ecoords = (lo + np.stack([ii, ii + 1], axis=1) * h)[:, :, None]   # unwrapped
        return mesh
    # all lattice points, lexicographic with axis 0 fastest
    grids = np.meshgrid(*[np.arange(m)] * d, indexing="ij")
    allz = np.stack([g.ravel(order="F") for g in grids], axis=1)  # axis0 fastest
    # order='F' on an 'ij' meshgrid makes axis 0 vary fastest
    keep = _in_domain_closed(kind, allz / cells)
    lattice = allz[keep]
    node_id = {tuple(z): i for i, z in enumerate(lattice.tolist())}
    coords = lo + lattice * h
    # cells
    cgrids = np.meshgrid(*[np.arange(cells)] * d, indexing="ij")
    allc = np.stack([g.ravel(order="F") for g in cgrids], axis=1)
    ckeep = _in_domain_closed(kind, (allc + 0.5) / cells)
    cell_list = allc[ckeep]
    elems = []
    perms = list(itertools.permutations(range(d)))
    for z in cell_list.tolist():
        for pi in perms:
            v = list(z)
            verts = [node_id[tuple(v)]]
            for ax in pi:
                v[ax] += 1
                verts.append(node_id[tuple(v)])
            elems.append(verts)
    elems = np.asarray(elems, dtype=np.int64)
    mesh = Mesh(kind, d, level, lo, hi, m, h, lattice, coords, node_id, elems)
    mesh.pattern = element_pattern(mesh)
    mesh.ecoords = coords[elems]
    return mesh


def element_pattern(mesh: Mesh) -> sp.csr_matrix:
    """Sparsity {(a,b): a,b in a common element}, canonical CSR (sorted, no dups)."""
    e = mesh.elems
    k = e.shape[1]
    rows = np.repeat(e, k, axis=1).ravel()
    cols = np.tile(e, (1, k)).ravel()
    P = sp.coo_matrix((np.ones(rows.size), (rows, cols)), shape=(mesh.n, mesh.n)).tocsr()
    P.sum_duplicates()
    P.sort_indices()
    P.data[:] = 1.0
    return P


def pattern_ell(mesh: Mesh, width: int) -> np.ndarray:
    """Pattern as padded ELL, row-major (n, width), sorted columns, -1 padding."""
    P = mesh.pattern
    out = -np.ones((mesh.n, width), dtype=np.int32)
    for i in range(mesh.n):
        cols = P.indices[P.indptr[i]:P.indptr[i + 1]]
        assert cols.size <= width
        out[i, :cols.size] = cols
    return out


def volumes(mesh: Mesh) -> np.ndarray:
    """|K| for every element: |det(v1-v0, ..., vd-v0)| / d!."""
    P = mesh.ecoords                          # (ne, d+1, d)
    J = P[:, 1:, :] - P[:, :1, :]              # (ne, d, d)
    return np.abs(np.linalg.det(J)) / math.factorial(mesh.d)


def locate(mesh: Mesh, pts: np.ndarray):
    """For points in the closed domain return (vertex node ids (np,d+1), barycentric (np,d+1)).

    Plain point location in the structured Kuhn mesh: find the containing cell
    (a cell that is in the mesh), then the Kuhn simplex by sorting the local
    coordinates in decreasing order; barycentric coordinates are the sorted
    differences."""
    d = mesh.d
    cells = mesh.m - 1
    if mesh.kind == "periodic":
        q = np.mod((pts[:, 0] - mesh.lo[0]) / mesh.h[0], cells)
        i0 = np.minimum(np.floor(q).astype(np.int64), cells - 1)
        f = q - i0
        verts = np.stack([i0, (i0 + 1) % cells], axis=1)
        lam = np.stack([1 - f, f], axis=1)
        return verts, lam
    q = (pts - mesh.lo) / mesh.h                  # lattice units
    base = np.floor(q + 1e-12).astype(np.int64)
    base = np.clip(base, 0, cells - 1)
    out_v = np.zeros((pts.shape[0], d + 1), np.int64)
    out_l = np.zeros((pts.shape[0], d + 1))
    for p in range(pts.shape[0]):
        b = base[p].copy()
        # choose a cell that is in the domain (L-shape: shift on cell faces)
        cand = [b]
        for shift in itertools.product(*[[0, -1]] * d):
            bb = b + np.asarray(shift)
            if np.all(bb >= 0) and np.all(bb <= cells - 1):
                cand.append(bb)
        chosen = None
        for bb in cand:
            f = q[p] - bb
            if np.any(f < -1e-9) or np.any(f > 1 + 1e-9):
                continue
            if _in_domain_closed(mesh.kind, (bb + 0.5) / cells):
                chosen = bb
                break
        assert chosen is not None, "point outside mesh"
        f = np.clip(q[p] - chosen, 0.0, 1.0)
        order = np.argsort(-f, kind="stable")
        fs = f[order]
        lam = np.empty(d + 1)
        lam[0] = 1.0 - fs[0]
        for k in range(1, d):
            lam[k] = fs[k - 1] - fs[k]
        lam[d] = fs[d - 1]
        v = chosen.copy()
        verts = [mesh.node_id[tuple(v.tolist())]]
        for ax in order:
            v[ax] += 1
            verts.append(mesh.node_id[tuple(v.tolist())])
        out_v[p] = verts
        out_l[p] = lam
    return out_v, out_l


def embedding(coarse: Mesh, fine: Mesh) -> sp.csr_matrix:
    """E[f, c] = phi^coarse_c(x_f)  (matrix of V_l' -> V_l)."""
    verts, lam = locate(coarse, fine.coords)
    rows = np.repeat(np.arange(fine.n), coarse.d + 1)
    E = sp.coo_matrix((lam.ravel(), (rows, verts.ravel())), shape=(fine.n, coarse.n)).tocsr()
    E.eliminate_zeros()
    E.sum_duplicates()
    E.sort_indices()
    return E


class Hierarchy:
    """Meshes of one factor for levels 1..lmax and the one-level embeddings."""

    def __init__(self, spec: dict, nc: int, lmax: int):
        self.spec = spec
        self.nc = nc
        self.lmax = lmax
        self.meshes = {l: build_mesh(spec, nc, l) for l in range(1, lmax + 1)}
        self.E1 = {l: embedding(self.meshes[l], self.meshes[l + 1]) for l in range(1, lmax)}
        self._Ecache = {}

    def n(self, l: int) -> int:
        return self.meshes[l].n

    def E(self, lf: int, lc: int) -> sp.csr_matrix:
        """E_{lf <- lc} = product of one-level embeddings (identity if equal)."""
        assert lf >= lc
        key = (lf, lc)
        if key not in self._Ecache:
            M = sp.identity(self.n(lc), format="csr")
            for l in range(lc, lf):
                M = self.E1[l] @ M
            self._Ecache[key] = M.tocsr()
        return self._Ecache[key]
