"""GPU parity: the CUDA path (libsg.so through the C ABI) vs the oracle.

Bars: bit-exact for meshes / patterns / transfer indices; fp64 relative
max-norm 1e-12 per operator apply (BASELINE north_star); 1e-9 relative on the
solution function after stepping.  Sizes span several tiles and ragged tails.
"""
import numpy as np
import pytest

from sginputs import CONFIG_ORDER, get_config
from tests.gpu_helpers import SET_ACTIVE, SET_COARSE, from_blocks, oracle_spec, relmax, to_blocks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = {"c0_2d_const": 6, "c1_2d_rot": 5, "c2_4d_stream": 4, "c3_4d_lshape": 4, "c4_6d_stream": 3}

_cache = {}


def pair(name, L=None):
    """(gpu Problem, oracle SGProblem) for a config at a small level."""
    L = SMALL[name] if L is None else L
    key = (name, L)
    if key not in _cache:
        from oracle.sgrid import SGProblem
        from paper_2204_05988_b200 import Problem
        cfg = get_config(name, L=L)
        _cache[key] = (Problem(cfg), SGProblem(cfg))
    return _cache[key]


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_meshes_bit_exact(name):
    from oracle.mesh import pattern_ell
    g, o = pair(name)
    for fac, H in ((0, o.Hx), (1, o.Hv)):
        for l in range(1, o.F + 1):
            lat, cols = g.mesh_export(fac, l)
            m = H.meshes[l]
            assert np.array_equal(lat, m.lattice.astype(np.int32)), (fac, l)
            assert np.array_equal(cols, pattern_ell(m, cols.shape[1])), (fac, l)
            if l >= 2:
                pc, pv, rc, rv = g.transfer_export(fac, l)
                E = H.E1[l - 1]
                Et = E.T.tocsr()
                for i in range(m.n):
                    cc = E.indices[E.indptr[i]:E.indptr[i + 1]]
                    vv = E.data[E.indptr[i]:E.indptr[i + 1]]
                    assert np.array_equal(pc[i][pc[i] >= 0], cc) and np.array_equal(pv[i][pc[i] >= 0], vv)
                for i in range(H.n(l - 1)):
                    cc = Et.indices[Et.indptr[i]:Et.indptr[i + 1]]
                    vv = Et.data[Et.indptr[i]:Et.indptr[i + 1]]
                    assert np.array_equal(rc[i][rc[i] >= 0], cc) and np.array_equal(rv[i][rc[i] >= 0], vv)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_factor_matrices(name):
    from oracle.fem import assemble
    g, o = pair(name)
    d = o.d
    for fac, H in ((0, o.Hx), (1, o.Hv)):
        for sp in range(g.num_specs(fac)):
            spec = oracle_spec(g.spec_info(fac, sp), d)
            for l in range(1, o.F + 1):
                vals = g.factor_export(fac, sp, l)
                A = assemble(H.meshes[l], spec)
                _, cols = g.mesh_export(fac, l)
                ref = np.zeros_like(vals)
                for i in range(A.shape[0]):
                    k = cols[i] >= 0
                    ref[i, k] = A[i, cols[i][k]].toarray().ravel()
                scale = max(np.abs(ref).max(), 1e-300)
                assert np.abs(vals - ref).max() <= 1e-13 * scale, (fac, sp, l, spec)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_term_expansion_same_operator(name):
    """sum_t T_t (x) X_t (x) V_t from the GPU term list == the oracle's (dense, one grid)."""
    from oracle.fem import assemble
    g, o = pair(name)
    l = o.active[len(o.active) // 2]
    mx, mv = o.Hx.meshes[l[0]], o.Hv.meshes[l[1]]
    D1 = 0
    for T, xs, vs in g.terms():
        X = assemble(mx, oracle_spec(g.spec_info(0, xs), o.d)).toarray()
        V = assemble(mv, oracle_spec(g.spec_info(1, vs), o.d)).toarray()
        D1 = D1 + np.kron(T, np.kron(X, V))
    D2 = o.block_matrix(o.terms, l, l).toarray()
    assert relmax(D1, D2) <= 1e-13


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_apply_strip_operator(name):
    """Per-grid strip operator (the hot path) on every active and coarse grid."""
    g, o = pair(name)
    rng = np.random.default_rng(0)
    for set_, grids in ((SET_ACTIVE, o.active), (SET_COARSE, o.coarse)):
        for gi, l in enumerate(grids):
            X = rng.standard_normal(o.shape(l))
            Xt = torch.from_numpy(X.ravel()).cuda()
            Yt = torch.zeros_like(Xt)
            g.sg_apply_strip_operator(set_, gi, Xt, Yt)
            Y = Yt.cpu().numpy().reshape(X.shape)
            ref = o.apply_diag(l, X)
            assert relmax(Y, ref) <= 1e-12, (set_, l)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_apply_full_cross_grid(name):
    g, o = pair(name)
    rng = np.random.default_rng(1)
    U = {l: rng.standard_normal(o.shape(l)) for l in o.active}
    Xt = from_blocks(g, U)
    Yt = torch.zeros_like(Xt)
    g.sg_apply_full(Xt, Yt)
    Y = to_blocks(g, Yt)
    ref = o.apply_full(o.terms, U)
    for l in o.active:
        assert relmax(Y[l], ref[l]) <= 1e-12, l


@pytest.mark.parametrize("env", ["SG_NO_CROSS_BATCH", "SG_NO_TMA"])
@pytest.mark.parametrize("name", ["c2_4d_stream", "c4_6d_stream"])
def test_apply_full_cross_grid_paths(name, env, monkeypatch):
    """Cross-grid apply on the per-group path and with the batched lower part's kernel variants."""
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    monkeypatch.setenv(env, "1")
    cfg = get_config(name, L=SMALL[name])
    g, o = Problem(cfg), SGProblem(cfg)
    rng = np.random.default_rng(11)
    U = {l: rng.standard_normal(o.shape(l)) for l in o.active}
    Xt = from_blocks(g, U)
    Yt = torch.zeros_like(Xt)
    g.sg_apply_full(Xt, Yt)
    Y = to_blocks(g, Yt)
    ref = o.apply_full(o.terms, U)
    for l in o.active:
        assert relmax(Y[l], ref[l]) <= 1e-12, l


@pytest.mark.parametrize("name", ["c1_2d_rot", "c3_4d_lshape", "c4_6d_stream"])
def test_apply_mass_full(name):
    from oracle.problem import mass_terms
    g, o = pair(name)
    rng = np.random.default_rng(2)
    Tb = rng.standard_normal((o.S, 1))
    U = {l: rng.standard_normal((1,) + o.shape(l)[1:]) for l in o.active}
    Xt = from_blocks(g, U, S=1)
    Yt = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
    g.sg_apply_mass_full(Tb, Xt, Yt)
    Y = to_blocks(g, Yt)
    ref = o.apply_full(mass_terms(o.cfg, Tb), U)
    for l in o.active:
        assert relmax(Y[l], ref[l]) <= 1e-12, l


@pytest.mark.parametrize("name", ["c0_2d_const", "c3_4d_lshape", "c4_6d_stream"])
def test_transfers_and_combine(name):
    g, o = pair(name)
    rng = np.random.default_rng(3)
    S = o.S
    for fac, which in ((0, "x"), (1, "v")):
        for lf in range(2, o.F + 1):
            lo_ = 1
            n_o = (o.Hv if fac == 0 else o.Hx).n(lo_)
            nc, nf = (o.Hx if fac == 0 else o.Hv).n(lf - 1), (o.Hx if fac == 0 else o.Hv).n(lf)
            shp_c = (S, nc, n_o) if fac == 0 else (S, n_o, nc)
            shp_f = (S, nf, n_o) if fac == 0 else (S, n_o, nf)
            u = rng.standard_normal(shp_c)
            out = torch.zeros(int(np.prod(shp_f)), dtype=torch.float64, device="cuda")
            g.sg_prolongate(fac, lf, lf - 1, lo_, S, torch.from_numpy(u.ravel()).cuda(), out)
            ref = o.prolong(which, u, lf, lf - 1)
            assert np.array_equal(out.cpu().numpy().reshape(shp_f), ref)       # exact: weights 1, 1/2
            r = rng.standard_normal(shp_f)
            out2 = torch.zeros(int(np.prod(shp_c)), dtype=torch.float64, device="cuda")
            g.sg_restrict(fac, lf - 1, lf, lo_, S, torch.from_numpy(r.ravel()).cuda(), out2)
            assert relmax(out2.cpu().numpy().reshape(shp_c), o.restrict(which, r, lf - 1, lf)) <= 1e-15
    dh = {l: rng.standard_normal(o.shape(l)) for l in o.active + o.coarse}
    du = torch.zeros(g.set_size(SET_ACTIVE, S), dtype=torch.float64, device="cuda")
    g.sg_combine(from_blocks(g, dh), from_blocks(g, dh, SET_COARSE), du)
    ref = o.combine(dh)
    got = to_blocks(g, du)
    for l in o.active:
        assert relmax(got[l], ref[l]) <= 1e-15


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_interp_u0_and_rhs(name):
    g, o = pair(name)
    u0 = torch.zeros(g.set_size(SET_ACTIVE, 1), dtype=torch.float64, device="cuda")
    g.sg_interp_u0(u0)
    ref = o.interp_u0()
    got = to_blocks(g, u0, S=1)
    for l in o.active:
        assert relmax(got[l], ref[l]) <= 1e-14, l
    for j in (1, 3):
        b = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
        g.sg_rhs(j, u0, b)
        rb = o.rhs(j, ref)
        gb = to_blocks(g, b)
        for l in o.active:
            assert relmax(gb[l], rb[l]) <= 1e-12, (j, l)


def _full(o, blocks):
    return o.to_full(blocks)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_solve_strip(name):
    """Richardson + combination preconditioner: same FUNCTION as the oracle (coefficients
    are a spanning-set representation, not unique)."""
    g, o = pair(name)
    tr0 = o.interp_u0()
    b = o.rhs(1, tr0)
    U, it, _ = o.solve_strip(b, rtol=1e-13)
    bt = from_blocks(g, b)
    ut = torch.zeros_like(bt)
    git, last = g.sg_solve_strip(bt, ut, rtol=1e-13, inner_rtol=1e-13, max_iter=200)
    G = to_blocks(g, ut)
    for s in range(o.S):
        f_ref = _full(o, {l: U[l][s:s + 1] for l in o.active})
        f_gpu = _full(o, {l: G[l][s:s + 1] for l in o.active})
        assert relmax(f_gpu, f_ref) <= 1e-9, (s, it, git)


@pytest.mark.parametrize("name", ["c2_4d_stream", "c4_6d_stream", "c1_2d_rot", "c3_4d_lshape"])
@pytest.mark.parametrize("env", ["SG_OUTER=2", "SG_OUTER=1", "SG_NO_GRAPHS=1"])
def test_solve_strip_solver_variants(name, env, monkeypatch):
    """SG_OUTER=2 (residual-minimising step lengths from the first iteration, the safeguard's
    mode), SG_OUTER=1 (the paper's plain Richardson, no safeguard) and SG_NO_GRAPHS (the
    uncaptured host-loop driver of the same device kernels): the same converged strip
    solution as the oracle's plain Richardson."""
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    k, v = env.split("=")
    monkeypatch.setenv(k, v)
    cfg = get_config(name, L=SMALL[name])
    g, o = Problem(cfg), SGProblem(cfg)
    tr0 = o.interp_u0()
    b = o.rhs(1, tr0)
    U, it, _ = o.solve_strip(b, rtol=1e-13)
    ut = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
    git, _ = g.sg_solve_strip(from_blocks(g, b), ut, rtol=1e-13, inner_rtol=1e-13, max_iter=200)
    assert git < 200
    G = to_blocks(g, ut)
    for s in range(o.S):
        f_ref = _full(o, {l: U[l][s:s + 1] for l in o.active})
        f_gpu = _full(o, {l: G[l][s:s + 1] for l in o.active})
        assert relmax(f_gpu, f_ref) <= 1e-9, (s, it, git)


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_step_matches_oracle(name):
    g, o = pair(name)
    nst = 3
    tr_ref, _, _ = o.run(nsteps=nst, rtol=1e-13)
    u0 = torch.zeros(g.set_size(SET_ACTIVE, 1), dtype=torch.float64, device="cuda")
    g.sg_interp_u0(u0)
    g.sg_step(1, nst, u0, rtol=1e-13, inner_rtol=1e-13)
    f_ref = _full(o, tr_ref)
    f_gpu = _full(o, to_blocks(g, u0, S=1))
    assert relmax(f_gpu, f_ref) <= 1e-9
    # host-buffer path (e2e) gives the same result
    h = np.zeros(g.set_size(SET_ACTIVE, 1))
    g.sg_interp_u0(u0)
    h[:] = u0.cpu().numpy()
    g.sg_step(1, nst, h, rtol=1e-13, inner_rtol=1e-13)
    f_h = _full(o, to_blocks(g, torch.from_numpy(h), S=1))
    assert relmax(f_h, f_ref) <= 1e-9


def test_single_grid_edge_case():
    """L = 2: one component grid, no coarse grids; the preconditioner is exact."""
    g, o = pair("c1_2d_rot", L=2)
    assert g.num_grids(SET_COARSE) == 0
    tr0 = o.interp_u0()
    b = o.rhs(1, tr0)
    U, it, _ = o.solve_strip(b, rtol=1e-13)
    ut = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
    git, _ = g.sg_solve_strip(from_blocks(g, b), ut, rtol=1e-13, inner_rtol=1e-13)
    assert git <= 3
    G = to_blocks(g, ut)
    for l in o.active:
        assert relmax(G[l], U[l]) <= 1e-10


def test_zero_rhs_gives_zero():
    g, o = pair("c2_4d_stream")
    b = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
    u = torch.zeros_like(b)
    it, last = g.sg_solve_strip(b, u)
    assert it == 1 and float(u.abs().max()) == 0.0


@pytest.mark.parametrize("env", ["SG_NO_TMA", "SG_NO_FUSED"])
@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_apply_strip_operator_kernel_paths(name, env, monkeypatch):
    """Same parity on the fallbacks: of the TMA line sweep (register line sweep k_xfanin) and
    of the fused whole-x apply (moment pass 1 + whole-x pass 2)."""
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    for kv in env.split(";"):
        key, _, val = kv.partition("=")
        monkeypatch.setenv(key, val or "1")
    cfg = get_config(name, L=SMALL[name])
    g, o = Problem(cfg), SGProblem(cfg)
    rng = np.random.default_rng(5)
    for set_, grids in ((SET_ACTIVE, o.active), (SET_COARSE, o.coarse)):
        for gi, l in enumerate(grids):
            X = rng.standard_normal(o.shape(l))
            Xt = torch.from_numpy(X.ravel()).cuda()
            Yt = torch.zeros_like(Xt)
            g.sg_apply_strip_operator(set_, gi, Xt, Yt)
            assert relmax(Yt.cpu().numpy().reshape(X.shape), o.apply_diag(l, X)) <= 1e-12, (set_, l)


def _full_size_oracle(name, l):
    """Oracle for one grid of a full-size config: meshes up to the grid's own levels,
    factor matrices assembled directly on them (equal to the Galerkin products by
    nestedness, pinned in test_oracle_fem.py), the oracle's own delta and terms."""
    from oracle.problem import delta_hmin, strip_terms
    from oracle.sgrid import SGProblem
    cfg = get_config(name)
    o = SGProblem(get_config(name, L=max(l) + 1), galerkin="direct")
    o.tau, o.delta = cfg["tau"], delta_hmin(cfg)        # the oracle's own delta (reading R5)
    o.terms = strip_terms(cfg, cfg["tau"], o.delta)
    return cfg, o


def _grid_index(g, l):
    return [i for i in range(g.num_grids(SET_ACTIVE)) if g.grid_info(SET_ACTIVE, i)[:2] == l][0]


def test_apply_strip_operator_full_size():
    """configs[4] at its full size (L=8), launch configuration of bench.py: the balanced grid
    (4,4) (24 M DOF, moment/stencil pass 1 + TMA line-swept pass 2) element by element."""
    from paper_2204_05988_b200 import Problem
    g = Problem(get_config("c4_6d_stream"))
    cfg, o = _full_size_oracle("c4_6d_stream", (4, 4))
    rng = np.random.default_rng(9)
    gi = _grid_index(g, (4, 4))
    l1, l2, n1, n2 = g.grid_info(SET_ACTIVE, gi)
    X = rng.standard_normal((1, n1, n2))
    Yt = torch.empty(n1 * n2, dtype=torch.float64, device="cuda")
    g.sg_apply_strip_operator(SET_ACTIVE, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
    ref = o.apply_pair(o.terms, (4, 4), (4, 4), X)
    assert relmax(Yt.cpu().numpy().reshape(X.shape), ref) <= 1e-12


@pytest.mark.parametrize("chunk_mb", [None, "1"])
@pytest.mark.parametrize("name,L", [("c2_4d_stream", 8), ("c4_6d_stream", 5)])
def test_apply_strip_operator_fused_sizes(name, L, chunk_mb, monkeypatch):
    """Every active and coarse grid at a level where the fused whole-x kernel engages on many
    column blocks with a ragged tail (configs[2] L = 8: level-1/2 x-lattices (1,7), (2,6), ...;
    configs[4] L = 5: (1,4), (1,3)) next to the two-pass kernels of the other grids, element by
    element against the oracle (factors assembled on each grid's own levels).  chunk_mb: the
    opt-in L2-resident column-chunk pipeline with 1 MB chunks, i.e. 5-8
    chunks with a ragged last one on grids such as (4,4) / (2,3)."""
    from oracle.problem import delta_hmin, strip_terms
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    if chunk_mb:
        monkeypatch.setenv("SG_L2_MB", chunk_mb)
        monkeypatch.setenv("SG_L2_MINCOLS", "32")
    cfg = get_config(name, L=L)
    g, o = Problem(cfg), SGProblem(cfg, galerkin="direct")
    rng = np.random.default_rng(31)
    for set_, grids in ((SET_ACTIVE, o.active), (SET_COARSE, o.coarse)):
        for gi, l in enumerate(grids):
            X = rng.standard_normal(o.shape(l))
            Yt = torch.empty(X.size, dtype=torch.float64, device="cuda")
            g.sg_apply_strip_operator(set_, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
            assert relmax(Yt.cpu().numpy().reshape(X.shape), o.apply_diag(l, X)) <= 1e-12, (set_, l)


def _sample_nodes(m, d, n_random, rng):
    """Sampled lattice nodes of an m^d box lattice: all 3^d boundary-class corners/edge/face
    representatives plus n_random uniform nodes (node id = sum z_k m^k)."""
    reps = []
    for cls in np.ndindex(*([3] * d)):
        z = [0 if c == 0 else (m - 1 if c == 2 else int(rng.integers(1, m - 1))) for c in cls]
        reps.append(sum(zk * m ** k for k, zk in enumerate(z)))
    rnd = rng.choice(m ** d, size=n_random, replace=False)
    return np.unique(np.concatenate([np.asarray(reps), rnd]))


@pytest.mark.parametrize("l", [(1, 7), (7, 1)])
def test_apply_strip_operator_full_size_extreme_grids(l):
    """configs[4] (L=8): the extreme grids (1,7) and (7,1) (58 M DOF each: moment pass 1 +
    whole-x pass 2, stencil pass 1 + TMA pass 2) element by element on >= 10^4 sampled
    outputs (every x-row x ~400 v-rows, resp. ~400 x-rows x every v-row, all 3^d boundary
    classes included); the oracle assembles the level-7 rows on the patches of the sampled
    nodes (oracle/rows.py, pinned against whole assembly)."""
    from oracle.rows import sampled_apply
    from paper_2204_05988_b200 import Problem
    g = Problem(get_config("c4_6d_stream"))
    cfg, o = _full_size_oracle("c4_6d_stream", (1, 1))
    rng = np.random.default_rng(17)
    gi = _grid_index(g, l)
    _, _, n1, n2 = g.grid_info(SET_ACTIVE, gi)
    X = rng.standard_normal((1, n1, n2))
    Yt = torch.empty(n1 * n2, dtype=torch.float64, device="cuda")
    g.sg_apply_strip_operator(SET_ACTIVE, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
    Y = Yt.cpu().numpy().reshape(X.shape)
    m_big = 2 * 2 ** 6 + 1
    if l == (1, 7):
        xr, vr = np.arange(n1), _sample_nodes(m_big, 3, 400, rng)
    else:
        xr, vr = _sample_nodes(m_big, 3, 400, rng), np.arange(n2)
    assert len(xr) * len(vr) >= 10 ** 4
    ref = sampled_apply(cfg, o.terms, l, X, xr, vr)
    got = Y[:, xr][:, :, vr]
    assert relmax(got, ref) <= 1e-12


def test_apply_strip_operator_full_size_c3():
    """configs[3] at its full size (L=11, dG(1), L-shaped x factor): the balanced grids (5,6)
    and (6,5) (7.4 M and 6.9 M DOF) element by element."""
    from paper_2204_05988_b200 import Problem
    g = Problem(get_config("c3_4d_lshape"))
    rng = np.random.default_rng(21)
    for l in [(5, 6), (6, 5)]:
        cfg, o = _full_size_oracle("c3_4d_lshape", l)
        gi = _grid_index(g, l)
        _, _, n1, n2 = g.grid_info(SET_ACTIVE, gi)
        X = rng.standard_normal((2, n1, n2))
        Yt = torch.empty(2 * n1 * n2, dtype=torch.float64, device="cuda")
        g.sg_apply_strip_operator(SET_ACTIVE, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
        ref = o.apply_pair(o.terms, l, l, X)
        assert relmax(Yt.cpu().numpy().reshape(X.shape), ref) <= 1e-12, l


def test_full_size_c1_every_grid_and_one_strip():
    """configs[1] at its full size (L=14, 491 K active DOF, dG(1)): the strip operator on every
    active and coarse grid element by element; the first strip's right-hand side (interpolated
    u0, jump load) element by element; and the GPU strip solution (rtol 1e-13) checked by a
    property that holds at any size: it solves the Galerkin system A^(delta) U = b of the strip
    (PAPER.md l.424-438), its residual evaluated with the ORACLE's cross-grid operator
    E^T A_F E (one oracle apply, ~1.5 min; the oracle's own direct-LU Richardson needs hours)."""
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    cfg = get_config("c1_2d_rot")
    g, o = Problem(cfg), SGProblem(cfg)
    rng = np.random.default_rng(23)
    for set_, grids in ((SET_ACTIVE, o.active), (SET_COARSE, o.coarse)):
        for gi, l in enumerate(grids):
            X = rng.standard_normal(o.shape(l))
            Yt = torch.empty(X.size, dtype=torch.float64, device="cuda")
            g.sg_apply_strip_operator(set_, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
            assert relmax(Yt.cpu().numpy().reshape(X.shape), o.apply_diag(l, X)) <= 1e-12, (set_, l)
    tr0 = o.interp_u0()
    b_ref = o.rhs(1, tr0)
    u0 = torch.zeros(g.set_size(SET_ACTIVE, 1), dtype=torch.float64, device="cuda")
    g.sg_interp_u0(u0)
    bt = torch.zeros(g.set_size(SET_ACTIVE, o.S), dtype=torch.float64, device="cuda")
    g.sg_rhs(1, u0, bt)
    gb = to_blocks(g, bt)
    for l in o.active:
        assert relmax(gb[l], b_ref[l]) <= 1e-12, l
    ut = torch.zeros_like(bt)
    g.sg_solve_strip(bt, ut, rtol=1e-13, inner_rtol=1e-13, max_iter=200)
    U = to_blocks(g, ut)
    AU = o.apply_full(o.terms, U)
    nb = max(np.abs(b_ref[l]).max() for l in o.active)
    res = max(np.abs(AU[l] - b_ref[l]).max() for l in o.active)
    assert res <= 1e-9 * nb, res / nb


def test_apply_strip_operator_full_size_4d():
    """configs[2] at its full size (L=12, bench launch configuration): the balanced grid (6,6)
    (17.9 M DOF, TMA pass 2 + moment pass 1) element by element against the oracle's exact
    factor matrices on its own level-6 meshes."""
    from paper_2204_05988_b200 import Problem
    g = Problem(get_config("c2_4d_stream"))
    gi = _grid_index(g, (6, 6))
    l1, l2, n1, n2 = g.grid_info(SET_ACTIVE, gi)
    cfg, o = _full_size_oracle("c2_4d_stream", (6, 6))
    rng = np.random.default_rng(12)
    X = rng.standard_normal((1, n1, n2))
    Yt = torch.empty(n1 * n2, dtype=torch.float64, device="cuda")
    g.sg_apply_strip_operator(SET_ACTIVE, gi, torch.from_numpy(X.ravel()).cuda(), Yt)
    ref = o.apply_pair(o.terms, (6, 6), (6, 6), X)
    assert relmax(Yt.cpu().numpy().reshape(X.shape), ref) <= 1e-12


@pytest.mark.parametrize("name", CONFIG_ORDER)
def test_step_at_bench_settings(name):
    """sg_step at the settings bench.py times (outer rtol 1e-10, inner block solves to 1e-2)
    against the oracle's direct-LU Richardson at rtol 1e-13: 3 strips, the 1e-9 bar."""
    g, o = pair(name)
    nst = 3
    tr_ref, _, _ = o.run(nsteps=nst, rtol=1e-13)
    u0 = torch.zeros(g.set_size(SET_ACTIVE, 1), dtype=torch.float64, device="cuda")
    g.sg_interp_u0(u0)
    g.reset_stats()
    g.sg_step(1, nst, u0, rtol=1e-10, inner_rtol=1e-2)
    assert relmax(_full(o, to_blocks(g, u0, S=1)), _full(o, tr_ref)) <= 1e-9
    h = g.health()
    assert h["outer_unconverged"] == 0 and h["outer_nonfinite"] == 0 and h["inner_maxit"] == 0, h


@pytest.mark.parametrize("name,L", [("c0_2d_const", 6), ("c1_2d_rot", 5)])
def test_final_time(name, L):
    """All N = round(T/tau) strips to the final time T (configs[0]: 32 strips at its full
    L = 6; configs[1]: 402 strips at L = 5) against the oracle's solution at T
    (tests/golden/final_*.npz, written by tools/make_golden_final.py, which calls only
    oracle/): relative L2-on-the-full-grid bar 1e-9 (north_star)."""
    import os
    from oracle.sgrid import SGProblem
    from paper_2204_05988_b200 import Problem
    cfg = get_config(name, L=L)
    path = os.path.join(os.path.dirname(__file__), "golden", f"final_{name}_L{L}.npz")
    ref = np.load(path)
    o = SGProblem(cfg)
    N = int(round(cfg["T"] / cfg["tau"]))
    assert int(ref["nsteps"]) == N
    g = Problem(cfg)
    u = torch.zeros(g.set_size(SET_ACTIVE, 1), dtype=torch.float64, device="cuda")
    g.sg_interp_u0(u)
    g.sg_step(1, N, u, rtol=1e-13, inner_rtol=1e-13)
    got = to_blocks(g, u, S=1)
    blocks = {l: ref[f"block_{l[0]}_{l[1]}"] for l in o.active}
    diff = {l: got[l] - blocks[l] for l in o.active}
    # L2(Omega) norm of the function difference (representation independent, sec. 4.1)
    err = o.spatial_l2(diff) / o.spatial_l2(blocks)
    assert err <= 1e-9, err
    assert relmax(_full(o, got), ref["full"]) <= 1e-9
