"""Helpers shared by the GPU parity tests (host-side marshalling only)."""
import numpy as np

from oracle.fem import MatSpec, poly_key

SET_ACTIVE, SET_COARSE = 0, 1


def to_blocks(prob, vec, set_=SET_ACTIVE, S=None):
    """torch set vector -> {(l1,l2): numpy (S,n1,n2)}."""
    S = prob.S if S is None else S
    out = {}
    host = vec.detach().cpu().numpy()
    for g in range(prob.num_grids(set_)):
        l1, l2, n1, n2 = prob.grid_info(set_, g)
        o = prob.grid_offset(set_, g, S)
        out[(l1, l2)] = host[o:o + S * n1 * n2].reshape(S, n1, n2).copy()
    return out


def from_blocks(prob, blocks, set_=SET_ACTIVE, S=None):
    import torch
    S = prob.S if S is None else S
    n = prob.set_size(set_, S)
    host = np.zeros(n)
    for g in range(prob.num_grids(set_)):
        l1, l2, n1, n2 = prob.grid_info(set_, g)
        o = prob.grid_offset(set_, g, S)
        host[o:o + S * n1 * n2] = blocks[(l1, l2)].ravel()
    return torch.from_numpy(host).cuda()


_MONO = [(), (0,), (1,), (2,), (0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def oracle_spec(info, d):
    """GPU spec description -> oracle MatSpec (same mathematical definition)."""
    if info["kind"] == 1:
        return MatSpec("face", axis=info["face_axis"], sign=info["face_sign"])
    w = {}
    for c, axes in zip(info["weight"], _MONO):
        if c == 0.0:
            continue
        if any(a >= d for a in axes):
            raise AssertionError("weight uses an axis beyond d")
        e = [0] * d
        for a in axes:
            e[a] += 1
        w[tuple(e)] = w.get(tuple(e), 0.0) + c
    chi = None if info["chi_axis"] < 0 else (info["chi_axis"], info["chi_sign"])
    return MatSpec("vol", poly_key(w), info["trial_d"], info["test_d"], chi)


def relmax(a, b):
    a = np.asarray(a); b = np.asarray(b)
    den = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() / den
