"""Exact P1 factor matrices and quadrature load vectors on one factor mesh (oracle).

PAPER.md eq. (14) l.450-461 defines the space matrices M, T, C, K, K~, G as L2
inner products of basis functions (and their beta-derivatives); l.484-504
reduce them, for tensor-product coefficients beta = sum a_i(x) b_i(v) e_i +
c_i(x) d_i(v) e_{i+d}, to sums of Kronecker products of d-dimensional factor
matrices such as (a_i d_{x_i} phi', phi)_{L2(Omega^(1))}.  This module computes
those factor matrices.

A factor matrix is described by a spec (see `MatSpec`):
    vol : F[k, k'] = int_Omega  w(y) chi(y) (D^p phi_k')(D^q phi_k) dy
          w a polynomial of degree <= 2, D^p in {identity, d/dy_p} acting on
          the TRIAL function phi_k' (column), D^q on the TEST function phi_k
          (row), chi an optional half-space indicator chi_{s*y_axis > 0}
    face: F[k, k'] = int_{Gamma_n} phi_k' phi_k ds over all boundary facets
          with outward normal n = s*e_axis.

Integration is EXACT: a polynomial weight of degree <= 2 is written in the
quadratic barycentric form w = sum_{e,f} C_ef lam_e lam_f on each simplex and
integrated with the closed formula
    int_K lam_0^a0 ... lam_d^ad = d! |K| a0! ... ad! / (d + sum a)!.
Indicators are aligned with mesh planes at every level (the half-space
boundaries y_axis = 0 are lattice planes), so chi is constant per element and
taken at the element centroid.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh, volumes


# ----------------------------------------------------------------------------
# specs
# ----------------------------------------------------------------------------
def poly_key(p: dict) -> tuple:
    return tuple(sorted((tuple(k), float(v)) for k, v in p.items() if v != 0.0))


@dataclass(frozen=True)
class MatSpec:
    kind: str                  # "vol" or "face"
    weight: tuple = ()         # poly_key of w (vol)
    trial_d: int = -1          # derivative axis on trial (column) function, -1 = none
    test_d: int = -1           # derivative axis on test (row) function
    chi: tuple = None          # (axis, sign) for chi_{sign*y_axis > 0}, or None
    axis: int = -1             # face: normal axis
    sign: int = 0              # face: normal sign

    def transpose(self) -> "MatSpec":
        if self.kind == "face":
            return self
        return MatSpec("vol", self.weight, self.test_d, self.trial_d, self.chi)


def vol(weight: dict, trial_d=-1, test_d=-1, chi=None) -> MatSpec:
    return MatSpec("vol", poly_key(weight), trial_d, test_d, chi)


def face(axis: int, sign: int) -> MatSpec:
    return MatSpec("face", axis=axis, sign=sign)


# ----------------------------------------------------------------------------
# barycentric monomial integrals
# ----------------------------------------------------------------------------
def _bary_integral_table(d: int, order: int) -> np.ndarray:
    """T[i1..i_order] = int_K lam_i1 ... lam_i_order / |K|  (closed formula)."""
    T = np.zeros((d + 1,) * order)
    for idx in itertools.product(range(d + 1), repeat=order):
        a = np.bincount(np.asarray(idx), minlength=d + 1)
        num = math.factorial(d) * np.prod([math.factorial(int(x)) for x in a])
        T[idx] = num / math.factorial(d + order)
    return T


def _weight_bary(weight: tuple, P: np.ndarray) -> np.ndarray:
    """Quadratic barycentric coefficient matrices C (ne, d+1, d+1), sym, for w on each element.

    With y = sum_e P_e lam_e and sum_e lam_e = 1:
      1       = sum_ef lam_e lam_f
      y_i     = sum_ef P_e,i lam_e lam_f           (symmetrised)
      y_i y_j = sum_ef P_e,i P_f,j lam_e lam_f     (symmetrised)
    """
    ne, dp1, d = P.shape
    C = np.zeros((ne, dp1, dp1))
    one = np.ones(dp1)
    for expo, c in weight:
        expo = np.asarray(expo)
        deg = int(expo.sum())
        if deg == 0:
            C += c * np.einsum("e,f->ef", one, one)[None]
        elif deg == 1:
            i = int(np.argmax(expo))
            u = P[:, :, i]
            C += c * 0.5 * (u[:, :, None] * one[None, None, :] + one[None, :, None] * u[:, None, :])
        elif deg == 2:
            idx = [ax for ax in range(d) for _ in range(expo[ax])]
            u, w = P[:, :, idx[0]], P[:, :, idx[1]]
            C += c * 0.5 * (u[:, :, None] * w[:, None, :] + w[:, :, None] * u[:, None, :])
        else:
            raise ValueError("weights of degree > 2 are not needed by the paper's configs")
    return C


def _grad_lambda(P: np.ndarray) -> np.ndarray:
    """G (ne, d+1, d): gradient of lam_e on each element."""
    J = P[:, 1:, :] - P[:, :1, :]               # rows: v_k - v_0
    Jinv = np.linalg.inv(J)
    # y - v0 = J^T xi  =>  xi = J^{-T} (y - v0), lam_k = xi_{k-1}
    # grad lam_k = row k-1 of J^{-T}
    G = np.zeros((P.shape[0], P.shape[1], P.shape[2]))
    G[:, 1:, :] = np.swapaxes(Jinv, 1, 2)
    G[:, 0, :] = -G[:, 1:, :].sum(axis=1)
    return G


def assemble_vol(mesh: Mesh, spec: MatSpec) -> sp.csr_matrix:
    """F[k,k'] = int w chi (D^p phi_k') (D^q phi_k), exact (eq. (14), l.491-503)."""
    d = mesh.d
    P = mesh.ecoords                 # (ne, d+1, d)
    volK = volumes(mesh)
    C = _weight_bary(spec.weight, P)            # (ne, d+1, d+1)
    if spec.chi is not None:
        ax, s = spec.chi
        cen = P.mean(axis=1)[:, ax]
        volK = volK * (s * cen > 0)
    G = _grad_lambda(P)
    p, q = spec.trial_d, spec.test_d
    if p < 0 and q < 0:
        T4 = _bary_integral_table(d, 4)
        loc = np.einsum("nef,abef->nab", C, T4)             # [test a, trial b]
    elif p >= 0 and q < 0:
        T3 = _bary_integral_table(d, 3)
        s3 = np.einsum("nef,aef->na", C, T3)                 # int w lam_a
        loc = s3[:, :, None] * G[:, None, :, p]              # test a, trial b: dlam_b/dp
    elif p < 0 and q >= 0:
        T3 = _bary_integral_table(d, 3)
        s3 = np.einsum("nef,bef->nb", C, T3)
        loc = G[:, :, None, q] * s3[:, None, :]
    else:
        T2 = _bary_integral_table(d, 2)
        s2 = np.einsum("nef,ef->n", C, T2)
        loc = s2[:, None, None] * G[:, :, None, q] * G[:, None, :, p]
    loc = loc * volK[:, None, None]
    e = mesh.elems
    rows = np.repeat(e[:, :, None], d + 1, axis=2).ravel()
    cols = np.repeat(e[:, None, :], d + 1, axis=1).ravel()
    F = sp.coo_matrix((loc.ravel(), (rows, cols)), shape=(mesh.n, mesh.n)).tocsr()
    F.sum_duplicates()
    return _on_pattern(mesh, F)


def boundary_facets(mesh: Mesh):
    """List of (node tuple, outward axis, sign) for facets not shared by two elements."""
    d = mesh.d
    count = {}
    owner = {}
    for ei, el in enumerate(mesh.elems.tolist()):
        for drop in range(d + 1):
            f = tuple(sorted(el[:drop] + el[drop + 1:]))
            count[f] = count.get(f, 0) + 1
            owner[f] = (ei, el[drop])
    out = []
    for f, c in count.items():
        if c != 1:
            continue
        lat = mesh.lattice[list(f)]
        opp = mesh.lattice[owner[f][1]]
        axes = [ax for ax in range(d) if np.all(lat[:, ax] == lat[0, ax])]
        assert len(axes) == 1, "boundary facet is not axis aligned"
        ax = axes[0]
        sign = 1 if opp[ax] < lat[0, ax] else -1
        out.append((f, ax, sign))
    return out


def assemble_face(mesh: Mesh, spec: MatSpec) -> sp.csr_matrix:
    """F[k,k'] = int_{Gamma_{s e_axis}} phi_k' phi_k ds (eq. (14) G^(r), l.459, l.706-716)."""
    d = mesh.d
    rows, cols, vals = [], [], []
    for f, ax, sign in boundary_facets(mesh):
        if ax != spec.axis or sign != spec.sign:
            continue
        if d == 1:
            rows.append(f[0]); cols.append(f[0]); vals.append(1.0)
            continue
        Pf = mesh.coords[list(f)]
        E = (Pf[1:] - Pf[:1]).T                      # d x (d-1)
        area = math.sqrt(abs(np.linalg.det(E.T @ E))) / math.factorial(d - 1)
        k = d - 1
        for a in range(d):
            for b in range(d):
                mult = 2 if a == b else 1
                rows.append(f[a]); cols.append(f[b])
                vals.append(math.factorial(k) * area * mult / math.factorial(k + 2))
    F = sp.coo_matrix((vals, (rows, cols)), shape=(mesh.n, mesh.n)).tocsr()
    F.sum_duplicates()
    return _on_pattern(mesh, F)


def _on_pattern(mesh: Mesh, F: sp.csr_matrix) -> sp.csr_matrix:
    """Return F stored on the mesh pattern (explicit zeros kept), canonical order."""
    P = mesh.pattern
    rows = np.repeat(np.arange(P.shape[0]), np.diff(P.indptr))
    vals = np.asarray(F[rows, P.indices]).ravel()
    assert abs(abs(vals).sum() - abs(F).sum()) <= 1e-12 * max(1.0, abs(F).sum()), \
        "entries outside the element pattern"
    G = sp.csr_matrix((vals, P.indices.copy(), P.indptr.copy()), shape=P.shape)
    return G


def assemble(mesh: Mesh, spec: MatSpec) -> sp.csr_matrix:
    if spec.kind == "vol":
        return assemble_vol(mesh, spec)
    return assemble_face(mesh, spec)


# ----------------------------------------------------------------------------
# quadrature for non-polynomial loads (u0, inflow g): collapsed Gauss-Legendre
# ----------------------------------------------------------------------------
NQ = 4  # Gauss-Legendre points per collapsed direction (reading R9)


def gl01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def duffy_rule(d: int, n: int = NQ):
    """Points xi (nq, d) in the reference simplex {xi>=0, sum xi<=1} and weights.

    Collapsed (Duffy) map from [0,1]^d:
      d=1: xi1 = u1
      d=2: xi1 = u1, xi2 = u2 (1-u1),                 J = (1-u1)
      d=3: xi1 = u1, xi2 = u2 (1-u1), xi3 = u3 (1-u1)(1-u2),  J = (1-u1)^2 (1-u2)
    weights are GL(n) tensor weights times J; they sum to 1/d!."""
    g, w = gl01(n)
    pts, wts = [], []
    for idx in itertools.product(range(n), repeat=d):
        u = [g[i] for i in idx]
        ww = np.prod([w[i] for i in idx])
        if d == 1:
            xi = [u[0]]; J = 1.0
        elif d == 2:
            xi = [u[0], u[1] * (1 - u[0])]; J = 1 - u[0]
        else:
            xi = [u[0], u[1] * (1 - u[0]), u[2] * (1 - u[0]) * (1 - u[1])]
            J = (1 - u[0]) ** 2 * (1 - u[1])
        pts.append(xi)
        wts.append(ww * J)
    return np.asarray(pts), np.asarray(wts)


def load_vector(mesh: Mesh, fun) -> np.ndarray:
    """l_k = int fun(y) phi_k(y) dy with the collapsed GL rule on every simplex.

    fun: callable on (np, d) -> (np,).  Element vertex order = Kuhn order
    (v0 = cell corner), physical point y = v0 + sum_i xi_i (v_i - v0),
    weight d! |K| w_q, basis lam_0 = 1 - sum xi, lam_i = xi_i."""
    d = mesh.d
    xi, wq = duffy_rule(d)
    lam = np.concatenate([1 - xi.sum(axis=1, keepdims=True), xi], axis=1)   # (nq, d+1)
    P = mesh.ecoords
    volK = volumes(mesh)
    out = np.zeros(mesh.n)
    for e in range(P.shape[0]):
        y = P[e, 0] + xi @ (P[e, 1:] - P[e, :1])
        fv = fun(y) * wq * math.factorial(d) * volK[e]
        np.add.at(out, mesh.elems[e], lam.T @ fv)
    return out


def gaussian_factor(g: dict):
    """Per-factor initial-value function: scale*exp(-|y-c|^2/w), or (pins only)
    {'type': 'sin'|'cos', 'k': k}: sin/cos(2 pi k sum_i y_i) (eq. (16) l.582)."""
    if g.get("type") == "sin":
        return lambda y: np.sin(2 * np.pi * g["k"] * np.sum(y, axis=1))
    if g.get("type") == "cos":
        return lambda y: np.cos(2 * np.pi * g["k"] * np.sum(y, axis=1))
    c = np.asarray(g["center"])
    return lambda y: g["scale"] * np.exp(-np.sum((y - c) ** 2, axis=1) / g["w"])
