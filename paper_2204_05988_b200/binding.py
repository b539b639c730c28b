"""ctypes binding of libsg.so with the same names as the C ABI (include/sg.h)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SG_SET_ACTIVE, SG_SET_COARSE = 0, 1
SG_FACTOR_X, SG_FACTOR_V = 0, 1
SG_MESH_BOX, SG_MESH_LSHAPE = 0, 1


class SGError(RuntimeError):
    pass


class SGNoConvergence(SGError):
    """SG_ERR_NOCONV: an iteration limit was reached before the tolerance (results are written)."""


SG_ERR_NOCONV = 5


def lib_path() -> str:
    return os.path.join(_HERE, "libsg.so")


class sg_beta_term(C.Structure):
    _fields_ = [("axis", C.c_int), ("a", C.c_double * 4), ("b", C.c_double * 4)]


class sg_gauss_term(C.Structure):
    _fields_ = [("coef", C.c_double), ("xc", C.c_double * 3), ("xw", C.c_double), ("xs", C.c_double),
                ("vc", C.c_double * 3), ("vw", C.c_double), ("vs", C.c_double)]


class sg_config(C.Structure):
    _fields_ = [("d", C.c_int), ("nc", C.c_int), ("L", C.c_int), ("q", C.c_int),
                ("xkind", C.c_int), ("vkind", C.c_int),
                ("xlo", C.c_double * 3), ("xhi", C.c_double * 3), ("vlo", C.c_double * 3), ("vhi", C.c_double * 3),
                ("tau", C.c_double), ("delta", C.c_double), ("sigma", C.c_double),
                ("nbeta", C.c_int), ("beta", sg_beta_term * 6),
                ("nu0", C.c_int), ("u0", sg_gauss_term * 4),
                ("inflow", C.c_int)]


def load_library():
    """Load libsg.so (raises SGError if it was not built: no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = lib_path()
    if not os.path.exists(p):
        raise SGError(f"{p} not found: run paper_2204_05988_b200/build.sh (there is no CPU fallback)")
    lib = C.CDLL(p)
    P, I, D, I64 = C.c_void_p, C.c_int, C.c_double, C.c_int64
    pD, pI, pI64, pI32 = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    sigs = {
        "sg_create": (I, [C.POINTER(sg_config), P, C.POINTER(P)]),
        "sg_build_meshes": (I, [P]),
        "sg_assemble_factors": (I, [P]),
        "sg_destroy": (None, [P]),
        "sg_last_error": (C.c_char_p, []),
        "sg_S": (I, [P]),
        "sg_delta": (D, [P]),
        "sg_num_grids": (I, [P, I]),
        "sg_grid_info": (I, [P, I, I, pI, pI, pI64, pI64]),
        "sg_grid_offset": (I64, [P, I, I, I]),
        "sg_set_size": (I64, [P, I, I]),
        "sg_mesh_info": (I, [P, I, I, pI64, pI, pI]),
        "sg_mesh_export": (I, [P, I, I, P, P]),
        "sg_transfer_export": (I, [P, I, I, P, P, P, P]),
        "sg_num_terms": (I, [P]),
        "sg_term_info": (I, [P, I, pD, pI, pI]),
        "sg_num_specs": (I, [P, I]),
        "sg_spec_info": (I, [P, I, I, pI, pD, pI, pI, pI, pI, pI, pI]),
        "sg_factor_export": (I, [P, I, I, I, P]),
        "sg_apply_strip_operator": (I, [P, I, I, P, P]),
        "sg_apply_full": (I, [P, P, P]),
        "sg_apply_mass_full": (I, [P, pD, I, I, P, P]),
        "sg_prolongate": (I, [P, I, I, I, I, I, P, P, D]),
        "sg_restrict": (I, [P, I, I, I, I, I, P, P, D]),
        "sg_combine": (I, [P, P, P, P]),
        "sg_interp_u0": (I, [P, P]),
        "sg_rhs": (I, [P, I, P, P]),
        "sg_solve_strip": (I, [P, P, P, D, D, I, pI, pD]),
        "sg_step": (I, [P, I, I, P, D, D]),
        "sg_stats": (I, [P, pI64, pI64, pI64, pI64, pI64]),
        "sg_solver_health": (I, [P, pI64, pI64, pI64, pI64]),
        "sg_outer_switches": (I, [P, pI64]),
        "sg_solve_history": (I, [P, I, pD, pD, pI]),
        "sg_reset_stats": (I, [P]),
        "sg_set_timing": (I, [P, I]),
        "sg_kernel_time": (I, [P, pD, pI64, pD, pD]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib


def _check(rc):
    if rc == SG_ERR_NOCONV:
        raise SGNoConvergence(f"libsg: {_LIB.sg_last_error().decode()}")
    if rc != 0:
        raise SGError(f"libsg error {rc}: {_LIB.sg_last_error().decode()}")


def _affine(poly: dict, d: int):
    """dict {expo: coef} of degree <= 1 -> [c0, c1..cd]."""
    out = [0.0] * 4
    for e, c in poly.items():
        e = tuple(e)
        s = sum(e)
        if s == 0:
            out[0] += c
        elif s == 1:
            out[1 + e.index(1)] += c
        else:
            raise ValueError("beta coefficients must be affine")
    return out


def config_from_dict(cfg: dict) -> sg_config:
    """Marshal an sginputs config dict into sg_config."""
    c = sg_config()
    d = cfg["d"]
    c.d, c.nc, c.L, c.q = d, cfg["nc"], cfg["L"], cfg["q"]
    kinds = {"box": SG_MESH_BOX, "lshape": SG_MESH_LSHAPE}
    c.xkind, c.vkind = kinds[cfg["xmesh"]["kind"]], kinds[cfg["vmesh"]["kind"]]
    for i in range(d):
        c.xlo[i], c.xhi[i] = cfg["xmesh"]["lo"][i], cfg["xmesh"]["hi"][i]
        c.vlo[i], c.vhi[i] = cfg["vmesh"]["lo"][i], cfg["vmesh"]["hi"][i]
    c.tau = cfg["tau"]
    c.delta = cfg.get("delta") or 0.0
    c.sigma = cfg["sigma"]
    c.nbeta = len(cfg["beta"])
    for k, (ax, a, b) in enumerate(cfg["beta"]):
        c.beta[k].axis = ax
        for i, v in enumerate(_affine(a, d)):
            c.beta[k].a[i] = v
        for i, v in enumerate(_affine(b, d)):
            c.beta[k].b[i] = v
    c.nu0 = len(cfg["u0"])
    for k, (coef, gx, gv) in enumerate(cfg["u0"]):
        t = c.u0[k]
        t.coef = coef
        for i in range(d):
            t.xc[i] = gx["center"][i]
            t.vc[i] = gv["center"][i]
        t.xw, t.xs, t.vw, t.vs = gx["w"], gx["scale"], gv["w"], gv["scale"]
    c.inflow = 1 if cfg.get("g") == "shifted_u0" else 0
    return c


def _ptr(t, n=None, name="buffer"):
    """Device pointer of a torch CUDA tensor (fp64, contiguous, at least n elements)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise SGError(f"{name}: expected a torch CUDA tensor")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise SGError(f"{name}: expected a contiguous float64 tensor")
    if n is not None and t.numel() < n:
        raise SGError(f"{name}: {t.numel()} elements, the call needs {n}")
    return C.c_void_p(t.data_ptr())


class Problem:
    """Owning wrapper of sg_problem*.  Methods mirror the C ABI names."""

    def __init__(self, cfg: dict, stream=None, build=True):
        import torch
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise SGError("no CUDA device: libsg has no CPU fallback")
        self.cfg_dict = cfg
        self.cfg = config_from_dict(cfg)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = C.c_void_p()
        _check(self.lib.sg_create(C.byref(self.cfg), C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h
        self.S = self.lib.sg_S(h)
        if build:
            self.sg_build_meshes()
            self.sg_assemble_factors()

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h:
            self.lib.sg_destroy(self.h)
            self.h = None

    # lifecycle
    def sg_build_meshes(self):
        _check(self.lib.sg_build_meshes(self.h))

    def sg_assemble_factors(self):
        _check(self.lib.sg_assemble_factors(self.h))

    # queries
    @property
    def delta(self):
        return self.lib.sg_delta(self.h)

    def num_grids(self, set_=SG_SET_ACTIVE):
        return self.lib.sg_num_grids(self.h, set_)

    def grid_info(self, set_, g):
        l1, l2 = C.c_int(), C.c_int()
        n1, n2 = C.c_int64(), C.c_int64()
        _check(self.lib.sg_grid_info(self.h, set_, g, C.byref(l1), C.byref(l2), C.byref(n1), C.byref(n2)))
        return l1.value, l2.value, n1.value, n2.value

    def grid_offset(self, set_, g, S):
        return self.lib.sg_grid_offset(self.h, set_, g, S)

    def set_size(self, set_, S):
        return self.lib.sg_set_size(self.h, set_, S)

    def mesh_info(self, factor, level):
        n, w, m = C.c_int64(), C.c_int(), C.c_int()
        _check(self.lib.sg_mesh_info(self.h, factor, level, C.byref(n), C.byref(w), C.byref(m)))
        return n.value, w.value, m.value

    def mesh_export(self, factor, level):
        n, W, m = self.mesh_info(factor, level)
        d = self.cfg.d
        lat = np.zeros((n, d), np.int32)
        cols = np.zeros((n, W), np.int32)
        _check(self.lib.sg_mesh_export(self.h, factor, level, lat.ctypes.data_as(C.c_void_p),
                                       cols.ctypes.data_as(C.c_void_p)))
        return lat, cols

    def transfer_export(self, factor, level):
        n, W, _ = self.mesh_info(factor, level)
        nc, _, _ = self.mesh_info(factor, level - 1)
        pc = np.zeros((n, 2), np.int32); pv = np.zeros((n, 2))
        rc = np.zeros((nc, W), np.int32); rv = np.zeros((nc, W))
        _check(self.lib.sg_transfer_export(self.h, factor, level, *[a.ctypes.data_as(C.c_void_p) for a in (pc, pv, rc, rv)]))
        return pc, pv, rc, rv

    def terms(self):
        out = []
        for t in range(self.lib.sg_num_terms(self.h)):
            T = (C.c_double * 4)()
            xs, vs = C.c_int(), C.c_int()
            _check(self.lib.sg_term_info(self.h, t, T, C.byref(xs), C.byref(vs)))
            out.append((np.array(T[:self.S * self.S]).reshape(self.S, self.S), xs.value, vs.value))
        return out

    def spec_info(self, factor, spec):
        kind = C.c_int(); w = (C.c_double * 10)()
        vals = [C.c_int() for _ in range(6)]
        _check(self.lib.sg_spec_info(self.h, factor, spec, C.byref(kind), w, *[C.byref(v) for v in vals]))
        tr, te, ca, cs, fa, fs = [v.value for v in vals]
        return dict(kind=kind.value, weight=list(w), trial_d=tr, test_d=te, chi_axis=ca, chi_sign=cs,
                    face_axis=fa, face_sign=fs)

    def num_specs(self, factor):
        return self.lib.sg_num_specs(self.h, factor)

    def factor_export(self, factor, spec, level):
        n, W, _ = self.mesh_info(factor, level)
        vals = np.zeros((n, W))
        _check(self.lib.sg_factor_export(self.h, factor, spec, level, vals.ctypes.data_as(C.c_void_p)))
        return vals

    # hot path (buffer sizes are checked against the handle's layout before any call)
    def _na(self, S=None):
        return self.set_size(SG_SET_ACTIVE, self.S if S is None else S)

    def sg_apply_strip_operator(self, set_, g, X, Y):
        _, _, n1, n2 = self.grid_info(set_, g)
        n = self.S * n1 * n2
        _check(self.lib.sg_apply_strip_operator(self.h, set_, g, _ptr(X, n, "X"), _ptr(Y, n, "Y")))

    def sg_apply_full(self, X, Y):
        n = self._na()
        _check(self.lib.sg_apply_full(self.h, _ptr(X, n, "X"), _ptr(Y, n, "Y")))

    def sg_apply_mass_full(self, Tb, X, Y):
        Tb = np.ascontiguousarray(Tb, dtype=np.float64)
        if Tb.ndim != 2:
            raise SGError("Tb: expected a 2D (S_out x S_in) array")
        _check(self.lib.sg_apply_mass_full(self.h, Tb.ctypes.data_as(C.POINTER(C.c_double)), Tb.shape[0],
                                           Tb.shape[1], _ptr(X, self._na(Tb.shape[1]), "X"),
                                           _ptr(Y, self._na(Tb.shape[0]), "Y")))

    def _transfer_sizes(self, factor, lf, lc, level_other, S):
        nf, _, _ = self.mesh_info(factor, lf)
        nc, _, _ = self.mesh_info(factor, lc)
        no, _, _ = self.mesh_info(1 - factor, level_other)
        return S * nc * no, S * nf * no

    def sg_prolongate(self, factor, lf, lc, level_other, S, inp, out, beta=0.0):
        ncoarse, nfine = self._transfer_sizes(factor, lf, lc, level_other, S)
        _check(self.lib.sg_prolongate(self.h, factor, lf, lc, level_other, S, _ptr(inp, ncoarse, "in"),
                                      _ptr(out, nfine, "out"), beta))

    def sg_restrict(self, factor, lc, lf, level_other, S, inp, out, beta=0.0):
        ncoarse, nfine = self._transfer_sizes(factor, lf, lc, level_other, S)
        _check(self.lib.sg_restrict(self.h, factor, lc, lf, level_other, S, _ptr(inp, nfine, "in"),
                                    _ptr(out, ncoarse, "out"), beta))

    def sg_combine(self, dhat_active, dhat_coarse, du):
        nc = self.set_size(SG_SET_COARSE, self.S)
        _check(self.lib.sg_combine(self.h, _ptr(dhat_active, self._na(), "dhat_active"),
                                   _ptr(dhat_coarse, nc, "dhat_coarse") if dhat_coarse is not None
                                   else C.c_void_p(0), _ptr(du, self._na(), "du")))

    def sg_interp_u0(self, u):
        _check(self.lib.sg_interp_u0(self.h, _ptr(u, self._na(1), "u")))

    def sg_rhs(self, j, trace_prev, b):
        _check(self.lib.sg_rhs(self.h, j, _ptr(trace_prev, self._na(1), "trace_prev"), _ptr(b, self._na(), "b")))

    def sg_solve_strip(self, b, u, rtol=1e-12, inner_rtol=1e-12, max_iter=200):
        """Returns (iterations, last update norm); raises SGNoConvergence at max_iter."""
        it, last = C.c_int(), C.c_double()
        n = self._na()
        _check(self.lib.sg_solve_strip(self.h, _ptr(b, n, "b"), _ptr(u, n, "u"), rtol, inner_rtol, max_iter,
                                       C.byref(it), C.byref(last)))
        return it.value, last.value

    def sg_step(self, j0, nsteps, trace, rtol=1e-10, inner_rtol=1e-10):
        """trace: torch CUDA tensor or numpy array (host); updated in place."""
        n = self._na(1)
        if isinstance(trace, np.ndarray):
            if trace.dtype != np.float64 or not trace.flags["C_CONTIGUOUS"] or trace.size < n:
                raise SGError(f"trace: expected a contiguous float64 array of >= {n} elements")
            p = trace.ctypes.data_as(C.c_void_p)
        else:
            p = _ptr(trace, n, "trace")
        _check(self.lib.sg_step(self.h, j0, nsteps, p, rtol, inner_rtol))

    # instrumentation
    def stats(self):
        v = [C.c_int64() for _ in range(5)]
        _check(self.lib.sg_stats(self.h, *[C.byref(x) for x in v]))
        sw = C.c_int64()
        _check(self.lib.sg_outer_switches(self.h, C.byref(sw)))
        return dict(zip(["applies", "dof_applied", "launches", "outer_iters", "inner_iters", "outer_mr_switches"],
                        [x.value for x in v] + [sw.value]))

    def health(self):
        v = [C.c_int64() for _ in range(4)]
        _check(self.lib.sg_solver_health(self.h, *[C.byref(x) for x in v]))
        return dict(zip(["outer_unconverged", "outer_nonfinite", "inner_maxit", "inner_breakdowns"],
                        [x.value for x in v]))

    def solve_history(self):
        """(update norms, step lengths) of every outer iteration of the last strip solve."""
        nd = (C.c_double * 256)()
        om = (C.c_double * 256)()
        n = C.c_int()
        _check(self.lib.sg_solve_history(self.h, 256, nd, om, C.byref(n)))
        return list(nd[:n.value]), list(om[:n.value])

    def reset_stats(self):
        _check(self.lib.sg_reset_stats(self.h))

    def set_timing(self, on):
        _check(self.lib.sg_set_timing(self.h, 1 if on else 0))

    def kernel_time(self):
        ms, n, b, f = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(self.lib.sg_kernel_time(self.h, C.byref(ms), C.byref(n), C.byref(b), C.byref(f)))
        return dict(ms=ms.value, launches=n.value, bytes=b.value, flops=f.value)

    # layout helpers (host-side index arithmetic only)
    def split(self, vec, set_=SG_SET_ACTIVE, S=None):
        """Views of a set vector per grid, shaped (S, n1, n2)."""
        S = self.S if S is None else S
        out = []
        for g in range(self.num_grids(set_)):
            l1, l2, n1, n2 = self.grid_info(set_, g)
            o = self.grid_offset(set_, g, S)
            out.append(vec[o:o + S * n1 * n2].view(S, n1, n2))
        return out
