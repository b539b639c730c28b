"""Pins of oracle/rows.py (patch-assembled factor rows, sampled strip-operator apply)
against whole assembly (oracle/fem.py, itself pinned in test_oracle_fem.py) and the
factored apply SGProblem.apply_pair (pinned against dense np.kron)."""
import numpy as np

from oracle.fem import assemble
from oracle.mesh import build_mesh
from oracle.problem import delta_hmin, strip_terms
from oracle.rows import factor_rows, sampled_apply
from sginputs import get_config


def _all_specs(cfg):
    terms = strip_terms(cfg, cfg["tau"], delta_hmin(cfg))
    return sorted({t[1] for t in terms}, key=repr), sorted({t[2] for t in terms}, key=repr), terms


def test_patch_rows_equal_whole_assembly():
    """Every factor matrix of configs[2] / configs[4] (x and v factors), level 3: the rows
    of every node (interior, face, edge, corner classes) from patches == whole assembly."""
    for name in ("c2_4d_stream", "c4_6d_stream"):
        cfg = get_config(name, L=4)
        xs, vs, _ = _all_specs(cfg)
        for which, specs in (("xmesh", xs), ("vmesh", vs)):
            mesh = build_mesh(cfg[which], cfg["nc"], 3)
            rows = np.arange(mesh.n)
            for ms in specs:
                ref = assemble(mesh, ms).tocsr()
                got = factor_rows(cfg[which], cfg["nc"], 3, rows, ms)
                diff = abs(ref - got).max()
                assert diff <= 1e-15 * max(abs(ref).max(), 1e-300), (name, which, ms)


def test_sampled_apply_equals_factored_apply():
    from oracle.sgrid import SGProblem
    cfg = get_config("c4_6d_stream", L=5)
    o = SGProblem(cfg, galerkin="direct")
    rng = np.random.default_rng(3)
    for l in [(1, 4), (4, 1), (2, 3)]:
        X = rng.standard_normal(o.shape(l))
        ref = o.apply_pair(o.terms, l, l, X)
        xr = rng.choice(X.shape[1], size=min(7, X.shape[1]), replace=False)
        vr = rng.choice(X.shape[2], size=min(9, X.shape[2]), replace=False)
        y = sampled_apply(cfg, o.terms, l, X, xr, vr)
        sub = ref[:, xr][:, :, vr]
        assert np.abs(y - sub).max() <= 1e-13 * np.abs(ref).max(), l
