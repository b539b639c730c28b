"""Sparse-grid combination-technique strip solver (oracle).

PAPER.md sec. 4.1-4.3:
  * l.392-418: a function of P^r(I_j, V_L) is stored on the spanning set of the
    component grids (eta_s x phi^(1)_{l1,k1} x phi^(2)_{l2,k2}); here the active
    grids are |l|_1 = L (reading R2), coefficient block u_l of shape (S, n1, n2),
    S = q+1, index order (s, k1, k2) = kron(time, x, v);
  * l.424-438: A^(delta) u = b blockwise; l.462-477 terms; l.506-509 the
    cross-level factor matrices A_{l,l'} = E_{F,l}^T A_{F,F} E_{F,l'} with F
    the finest level used (here L-1);
  * l.512-532: [A u]_l = sum_{l'} A_{l,l'} u_{l'}, each block applied as
    (S^t x Id x Id)(Id x S^1 x Id)(Id x Id x S^2) (factored);
  * l.540-566: Richardson u^{k+1} = u^k - P^{-1}(A u^k - b) with the combination
    technique P^{-1}: block solves (15) on |l|_1 = L and L-1, coarse residuals
    by the transpose of the x-embedding, and the combination
    du_l = dhat_l - (E^(1) x Id) dhat_{l1-1,l2} (l1 > 1);
  * eq. (4) l.82-95: the strip right-hand side is (U_{j-1}^-, w_{j-1}^+)
    - int <g, w>_{Gamma^-} (f = 0 in all configs), U_0^- = u0.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .fem import assemble, gaussian_factor, load_vector
from .mesh import Hierarchy
from .problem import delta_hmin, legendre, mass_terms, n_strips, strip_terms, time_blocks


class SGProblem:
    def __init__(self, cfg: dict, galerkin: str = "fine"):
        """galerkin='fine': cross-level factor matrices E^T A_F E (paper l.506-509);
        galerkin='direct': assembled directly on each level (equal by nestedness,
        pinned in tests/test_oracle_fem.py)."""
        self.cfg = cfg
        self.d = cfg["d"]
        self.L = cfg["L"]
        assert self.L >= 2
        self.q = cfg["q"]
        self.S = self.q + 1
        self.F = self.L - 1                    # finest level
        self.tau = float(cfg["tau"])
        self.delta = delta_hmin(cfg)
        self.N = n_strips(cfg)
        self.galerkin = galerkin
        self.Hx = Hierarchy(cfg["xmesh"], cfg["nc"], self.F)
        self.Hv = Hierarchy(cfg["vmesh"], cfg["nc"], self.F)
        self.active = [(l1, self.L - l1) for l1 in range(1, self.L)]
        self.coarse = [(l1, self.L - 1 - l1) for l1 in range(1, self.L - 1)]
        self.tb = time_blocks(self.q, self.tau)
        self.terms = strip_terms(cfg, self.tau, self.delta)
        self._fm = {}
        self._lu = {}

    # ------------------------------------------------------------------ shapes
    def shape(self, l):
        return (self.S, self.Hx.n(l[0]), self.Hv.n(l[1]))

    def zeros(self, grids=None):
        grids = self.active if grids is None else grids
        return {l: np.zeros(self.shape(l)) for l in grids}

    # ------------------------------------------------------- factor matrices
    def factor(self, which: str, spec, l: int, lp: int) -> sp.csr_matrix:
        """Cross-level factor matrix [a(phi_{lp,k'}, phi_{l,k})]."""
        key = (which, spec, l, lp)
        if key not in self._fm:
            H = self.Hx if which == "x" else self.Hv
            if self.galerkin == "fine":
                AF = self._direct(which, spec, self.F)
                A = (H.E(self.F, l).T @ AF @ H.E(self.F, lp)).tocsr()
            else:
                assert l == lp
                A = self._direct(which, spec, l)
            self._fm[key] = A
        return self._fm[key]

    def _direct(self, which, spec, l):
        key = ("direct", which, spec, l)
        if key not in self._fm:
            H = self.Hx if which == "x" else self.Hv
            self._fm[key] = assemble(H.meshes[l], spec)
        return self._fm[key]

    # ----------------------------------------------------------------- apply
    def apply_pair(self, terms, l, lp, u):
        """A_{l,l'} u_{l'} factored."""
        S = terms[0][0].shape[0]
        y = np.zeros((S, self.Hx.n(l[0]), self.Hv.n(l[1])))
        for T, xs, vs in terms:
            X = self.factor("x", xs, l[0], lp[0])
            V = self.factor("v", vs, l[1], lp[1])
            W = [X @ u[sp_] @ V.T for sp_ in range(u.shape[0])]
            for s in range(S):
                for sp_ in range(u.shape[0]):
                    if T[s, sp_] != 0.0:
                        y[s] += T[s, sp_] * W[sp_]
        return y

    def block_matrix(self, terms, l, lp) -> sp.csr_matrix:
        """Explicit sum_t kron(T_t, kron(X_t, V_t)) for the block (l, l')."""
        M = None
        for T, xs, vs in terms:
            X = self.factor("x", xs, l[0], lp[0])
            V = self.factor("v", vs, l[1], lp[1])
            K = sp.kron(sp.csr_matrix(T), sp.kron(X, V, format="csr"), format="csr")
            M = K if M is None else M + K
        return M.tocsr()

    def apply_full(self, terms, U, targets=None, sources=None):
        """[A u]_l = sum_{l'} A_{l,l'} u_{l'} over the active set."""
        targets = self.active if targets is None else targets
        sources = list(U.keys()) if sources is None else sources
        return {l: sum(self.apply_pair(terms, l, lp, U[lp]) for lp in sources) for l in targets}

    def apply_diag(self, l, u, terms=None):
        """Diagonal block A_{l,l} u_l (the per-component-grid strip operator)."""
        return self.apply_pair(self.terms if terms is None else terms, l, l, u)

    # ------------------------------------------------------------- transfers
    def prolong(self, which, u, lf, lc):
        """(Id x E x Id) or (Id x Id x E): coarse level lc -> fine level lf along x or v."""
        H = self.Hx if which == "x" else self.Hv
        E = H.E(lf, lc)
        if which == "x":
            return np.stack([E @ u[s] for s in range(u.shape[0])])
        return np.stack([u[s] @ E.T for s in range(u.shape[0])])

    def restrict(self, which, r, lc, lf):
        """Transpose of the embedding."""
        H = self.Hx if which == "x" else self.Hv
        E = H.E(lf, lc)
        if which == "x":
            return np.stack([E.T @ r[s] for s in range(r.shape[0])])
        return np.stack([r[s] @ E for s in range(r.shape[0])])

    # -------------------------------------------------------- preconditioner
    def block_solve(self, l, r):
        """Solve A^(delta)_{l,l} x = r directly (eq. (15) l.547-549, 'direct ... methods')."""
        if l not in self._lu:
            self._lu[l] = spla.splu(self.block_matrix(self.terms, l, l).tocsc())
        return self._lu[l].solve(r.ravel()).reshape(r.shape)

    def combine(self, dhat):
        """du_l = dhat_l - (E^(1) x Id) dhat_{l1-1,l2} for l1 > 1."""
        du = {}
        for l in self.active:
            du[l] = dhat[l].copy()
            if l[0] > 1:
                c = (l[0] - 1, l[1])
                du[l] -= self.prolong("x", dhat[c], l[0], c[0])
        return du

    def precondition(self, r):
        """P^{-1} r: block solves on |l| = L, L-1 and the combination."""
        dhat = {l: self.block_solve(l, r[l]) for l in self.active}
        for c in self.coarse:
            src = (c[0] + 1, c[1])
            rc = self.restrict("x", r[src], c[0], src[0])        # (Id x E^T x Id) r, l.552
            dhat[c] = self.block_solve(c, rc)
        return self.combine(dhat)

    # ---------------------------------------------------------------- norms
    def l2_inner(self, U, W):
        """(U, W)_{L2(I_j x Omega)} = sum_{l,l'} U_l^T (M^t x M_{l,l'}) W_{l'} (SPEC tensor_ops.l2_inner)."""
        MW = self.apply_full(mass_terms(self.cfg, self.tb["Mt"]), W)
        return sum(float(np.vdot(U[l], MW[l])) for l in self.active)

    def spatial_l2(self, U):
        """||U||_{L2(Omega)} of a spatial block vector (S=1)."""
        MW = self.apply_full(mass_terms(self.cfg, np.ones((1, 1))), U)
        return math.sqrt(max(sum(float(np.vdot(U[l], MW[l])) for l in self.active), 0.0))

    # ------------------------------------------------------------------- rhs
    def interp_u0(self):
        """U_0^- = I_L u0: nodal interpolants of u0 on the active and coarse grids,
        combined by the combination formula ("for interpolation
        such a scheme ... gives the exact result").  Reading R8: this
        is how the initial value u0 (eq. (4), U_0^- = u0) enters; it reproduces
        PAPER.md Table 1 (l.597-628) to within 10% (tests/test_oracle_sgrid.py::
        test_paper_table1_d1_r1)."""
        vals = {}
        for l in self.active + self.coarse:
            mx, mv = self.Hx.meshes[l[0]], self.Hv.meshes[l[1]]
            acc = np.zeros((1, mx.n, mv.n))
            for c, gx, gv in self.cfg["u0"]:
                acc[0] += c * np.outer(gaussian_factor(gx)(mx.coords), gaussian_factor(gv)(mv.coords))
            vals[l] = acc
        return self.combine(vals)

    def jump_load(self, trace_prev):
        """(U_{j-1}^-, w_{j-1}^+) = eta_s(t_{j-1}^+) [M U^-]_l (eq. (4) l.91-94)."""
        em = self.tb["eta_minus"]
        MU = self.apply_full(mass_terms(self.cfg, np.ones((1, 1))), trace_prev)
        return {l: em[:, None, None] * MU[l][0][None] for l in self.active}

    def beta_const(self):
        """Constant beta vector (configs with constant coefficients only)."""
        d = self.d
        b = np.zeros(2 * d)
        for ax, a, bb in self.cfg["beta"]:
            ka = list(a.items()); kb = list(bb.items())
            assert len(ka) == 1 and sum(ka[0][0]) == 0 and len(kb) == 1 and sum(kb[0][0]) == 0
            b[ax] += ka[0][1] * kb[0][1]
        return b

    def inflow_load(self, t0):
        """-int_{I_j} eta_s <g, phi_k phi_m>_{Gamma^-} dt,  g = u0(r - beta t), constant beta (configs[0]).

        <g,w>_{Gamma^-} = int_{Gamma^-} (beta.n) g w; only
        d = 1 (the faces of Omega1 are points).  Reading R9: time integral by
        4-point Gauss-Legendre on the strip; on each face g(tau_mu, .) is
        replaced by its nodal interpolant on the finest face mesh (level F), so
        that the load is ONE functional on V_L:
          face x = x_f:  row (s, k_f, m) += w_mu eta_s(tau_mu) |beta.n| (E_{F,l2}^T M^v_F g_F)_m
          face v = v_f:  row (s, k, m_f) += w_mu eta_s(tau_mu) |beta.n| (E_{F,l1}^T M^x_F g_F)_k
        """
        assert self.d == 1 and self.cfg.get("g") == "shifted_u0"
        beta = self.beta_const()
        xg, wg = np.polynomial.legendre.leggauss(4)
        tq = t0 + self.tau * (xg + 1) / 2
        wt = wg * self.tau / 2
        one = {(0,): 1.0}
        from .fem import vol
        mxF, mvF = self.Hx.meshes[self.F], self.Hv.meshes[self.F]
        MxF = self.factor("x", vol(one), self.F, self.F)
        MvF = self.factor("v", vol(one), self.F, self.F)
        out = {l: np.zeros(self.shape(l)) for l in self.active}
        for mu in range(4):
            eta = np.array([legendre(s, xg[mu]) for s in range(self.S)])
            t = tq[mu]
            for c, gx, gv in self.cfg["u0"]:
                fx, fv = gaussian_factor(gx), gaussian_factor(gv)
                for s_face, xpt in ((-1, mxF.lo[0]), (1, mxF.hi[0])):
                    bn = s_face * beta[0]
                    if bn < 0:
                        gF = c * fx(np.array([[xpt - beta[0] * t]]))[0] * fv(mvF.coords - beta[1] * t)
                        lF = MvF @ gF
                        for l in self.active:
                            node = 0 if s_face < 0 else self.Hx.n(l[0]) - 1
                            ll = self.Hv.E(self.F, l[1]).T @ lF
                            out[l][:, node, :] += -bn * wt[mu] * eta[:, None] * ll[None, :]
                for s_face, vpt in ((-1, mvF.lo[0]), (1, mvF.hi[0])):
                    bn = s_face * beta[1]
                    if bn < 0:
                        gF = c * fx(mxF.coords - beta[0] * t) * fv(np.array([[vpt - beta[1] * t]]))[0]
                        lF = MxF @ gF
                        for l in self.active:
                            node = 0 if s_face < 0 else self.Hv.n(l[1]) - 1
                            ll = self.Hx.E(self.F, l[0]).T @ lF
                            out[l][:, :, node] += -bn * wt[mu] * eta[:, None] * ll[None, :]
        return out

    def rhs(self, j, trace_prev):
        """b^(delta) for strip j (1-based) (eq. (4) l.92-94, f = 0); trace_prev = U_{j-1}^-."""
        b = self.jump_load(trace_prev)
        if self.cfg.get("g") == "shifted_u0":
            gl = self.inflow_load((j - 1) * self.tau)
            for l in self.active:
                b[l] += gl[l]
        return b

    # ---------------------------------------------------------------- solver
    def solve_strip(self, b, rtol=1e-12, atol=1e-300, max_iter=200, u_init=None):
        """Richardson with the combination preconditioner.

        Stops when ||du||_{L2(I_j x Omega)} <= atol + rtol ||u||_{L2(I_j x Omega)}."""
        u = self.zeros() if u_init is None else {l: u_init[l].copy() for l in self.active}
        hist = []
        for k in range(max_iter):
            Au = self.apply_full(self.terms, u)
            r = {l: Au[l] - b[l] for l in self.active}
            du = self.precondition(r)
            for l in self.active:
                u[l] -= du[l]
            nd = math.sqrt(max(self.l2_inner(du, du), 0.0))
            nu = math.sqrt(max(self.l2_inner(u, u), 0.0))
            hist.append(nd)
            if nd <= atol + rtol * nu:
                return u, k + 1, hist
        return u, max_iter, hist

    def trace(self, U):
        """U_j^- = sum_s eta_s(t_j^-) U_s (spatial block vector, S=1)."""
        ep = self.tb["eta_plus"]
        return {l: np.tensordot(ep, U[l], axes=(0, 0))[None] for l in self.active}

    def run(self, nsteps=None, rtol=1e-12, callback=None):
        nsteps = self.N if nsteps is None else nsteps
        tr = self.interp_u0()
        iters = []
        U = None
        for j in range(1, nsteps + 1):
            b = self.rhs(j, tr)
            U, it, _ = self.solve_strip(b, rtol=rtol)
            iters.append(it)
            tr = self.trace(U)
            if callback is not None:
                callback(j, U, tr)
        return tr, U, iters

    # ------------------------------------------------------------ evaluation
    def to_full(self, U, level=None):
        """Evaluate a (spatial, S=1) sparse-grid function on the full grid (F,F) nodes."""
        F = self.F if level is None else level
        out = np.zeros((self.Hx.n(F), self.Hv.n(F)))
        for l, u in U.items():
            Ex = self.Hx.E(F, l[0]); Ev = self.Hv.E(F, l[1])
            out += Ex @ u[0] @ Ev.T
        return out
