"""Thin ctypes binding of libst.so (include/st.h). Argument marshalling only: every step of
the path runs in the library's CUDA kernels. Tensors are passed by data pointer (device or
host memory; the library stages host memory itself). Fails loudly when libst.so is absent.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libst.so")

ST_OK = 0
ST_E_NOT_CONVERGED = -3
ST_TIME_CONSTANT, ST_SPACE_TIME = 0, 1
ST_SRC_UNIFORM, ST_SRC_SIN = 0, 1


class Grid(C.Structure):
    _fields_ = [("sdim", C.c_int32), ("n", C.c_int64), ("nt", C.c_int64), ("L", C.c_double), ("tau", C.c_double)]


class Materials(C.Structure):
    _fields_ = [("C_ins", C.c_double), ("C_con", C.c_double), ("p_c", C.c_double),
                ("k_ins", C.c_double), ("k_con", C.c_double), ("p_k", C.c_double)]


class BCs(C.Structure):
    _fields_ = [("T0", C.c_double), ("has_patch", C.c_int32), ("face", C.c_int32),
                ("center", C.c_double), ("halfwidth", C.c_double)]


class Source(C.Structure):
    _fields_ = [("kind", C.c_int32), ("Q0", C.c_double), ("a", C.c_double), ("w", C.c_double)]


class Options(C.Structure):
    _fields_ = [("design_mode", C.c_int32), ("rtol", C.c_double), ("maxit", C.c_int32), ("restart", C.c_int32),
                ("smoother", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("omega", C.c_double),
                ("lambda_crit", C.c_double), ("coarse_max_nodes", C.c_int64), ("max_levels", C.c_int32),
                ("full_coarsening", C.c_int32), ("use_graphs", C.c_int32), ("verbose", C.c_int32)]


class Dist(C.Structure):
    _fields_ = [("nccl_comm", C.c_void_p), ("rank", C.c_int32), ("size", C.c_int32),
                ("cuda_stream", C.c_void_p), ("device", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("restarts", C.c_int32), ("rel_residual", C.c_double),
                ("setup_ms", C.c_double), ("solve_ms", C.c_double), ("n_levels", C.c_int32),
                ("converged", C.c_int32)]


class Hierarchy(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n", C.c_int64 * 32), ("nt", C.c_int64 * 32),
                ("kind", C.c_int32 * 32), ("form", C.c_int32 * 32), ("nodes", C.c_int64 * 32)]


EXPORTS = ["st_abi_version", "st_default_options", "st_setup", "st_destroy", "st_solve", "st_adjoint",
           "st_sensitivity", "st_apply", "st_rhs", "st_level_apply", "st_bench_op", "st_get_stats", "st_get_hierarchy",
           "st_num_nodes", "st_num_design", "st_kernel_launches", "st_strerror", "st_last_error"]

_lib = None


class StError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libst error {code}: {msg}")
        self.code = code


def load_library(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built (run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    P = C.POINTER
    lib.st_default_options.argtypes = [P(Options)]
    lib.st_setup.argtypes = [P(Grid), P(Materials), P(BCs), P(Source), P(Options), P(Dist), P(C.c_void_p)]
    lib.st_setup.restype = C.c_int
    lib.st_destroy.argtypes = [C.c_void_p]
    for name in ("st_solve",):
        getattr(lib, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.st_adjoint.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.st_sensitivity.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.st_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    lib.st_rhs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.st_level_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    lib.st_bench_op.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.st_get_stats.argtypes = [C.c_void_p, P(Stats)]
    lib.st_get_hierarchy.argtypes = [C.c_void_p, P(Hierarchy)]
    for name in ("st_num_nodes", "st_num_design", "st_kernel_launches"):
        getattr(lib, name).argtypes = [C.c_void_p]
        getattr(lib, name).restype = C.c_int64
    lib.st_strerror.argtypes = [C.c_int]
    lib.st_strerror.restype = C.c_char_p
    lib.st_last_error.restype = C.c_char_p
    lib.st_abi_version.restype = C.c_int
    _lib = lib
    return lib


def _ptr(a):
    """Data pointer of a torch tensor / numpy array (must be contiguous fp64)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous() or str(a.dtype) != "torch.float64":
            raise ValueError("tensors must be contiguous float64")
        return a.data_ptr()
    import numpy as np
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise ValueError("arrays must be C-contiguous float64")
    return a.ctypes.data


class Solver:
    """One space-time problem on one GPU: st_setup at construction, st_destroy on close()."""

    def __init__(self, sdim, n, nt, mats=(1.0, 1.0, 1.0, 1e-3, 1.0, 3.0), T0=0.0, has_patch=True,
                 center=0.5, halfwidth=0.05, source=("uniform", 1.0, 0.0, 0.0), L=1.0, tau=1.0,
                 time_constant=False, stream=None, device=None, **opts):
        self.lib = load_library()
        self.grid = Grid(sdim, n, nt, L, tau)
        self.mats = Materials(*mats)
        self.bcs = BCs(T0, 1 if has_patch else 0, 0, center, halfwidth)
        kind = {"uniform": ST_SRC_UNIFORM, "sin": ST_SRC_SIN}[source[0]]
        self.src = Source(kind, *source[1:])
        o = Options()
        self.lib.st_default_options(C.byref(o))
        o.design_mode = ST_TIME_CONSTANT if time_constant else ST_SPACE_TIME
        for k, v in opts.items():
            if not hasattr(o, k):
                raise TypeError(f"unknown option {k}")
            setattr(o, k, v)
        self.opts = o
        d = Dist(None, 0, 1, stream if stream is not None else None, -1 if device is None else device)
        h = C.c_void_p()
        self._check(self.lib.st_setup(C.byref(self.grid), C.byref(self.mats), C.byref(self.bcs),
                                      C.byref(self.src), C.byref(o), C.byref(d), C.byref(h)))
        self.ctx = h

    def _check(self, rc, allow_nc=False):
        if rc == ST_OK or (allow_nc and rc == ST_E_NOT_CONVERGED):
            return rc
        msg = self.lib.st_last_error().decode() or self.lib.st_strerror(rc).decode()
        raise StError(rc, msg)

    @property
    def n_nodes(self):
        return self.lib.st_num_nodes(self.ctx)

    @property
    def n_design(self):
        return self.lib.st_num_design(self.ctx)

    def solve(self, rho, T, allow_nc=False):
        return self._check(self.lib.st_solve(self.ctx, _ptr(rho), _ptr(T)), allow_nc)

    def adjoint(self, rho, dJdT, lam, allow_nc=False):
        return self._check(self.lib.st_adjoint(self.ctx, _ptr(rho), _ptr(dJdT), _ptr(lam)), allow_nc)

    def sensitivity(self, rho, T, lam, dJ):
        return self._check(self.lib.st_sensitivity(self.ctx, _ptr(rho), _ptr(T), _ptr(lam), _ptr(dJ)))

    def apply(self, rho, x, y, transpose=False, bc=True):
        return self._check(self.lib.st_apply(self.ctx, _ptr(rho), _ptr(x), _ptr(y), int(transpose), int(bc)))

    def level_apply(self, rho, level, x, y, transpose=False):
        return self._check(self.lib.st_level_apply(self.ctx, _ptr(rho), level, _ptr(x), _ptr(y), int(transpose)))

    def bench_op(self, rho, level, mode, reps, transpose=False):
        """Enqueue `reps` launches of the level operator kernel (internal work vectors) without
        synchronising."""
        return self._check(self.lib.st_bench_op(self.ctx, _ptr(rho), level, mode, int(transpose), reps))

    def rhs(self, rho, f=None, b=None):
        return self._check(self.lib.st_rhs(self.ctx, _ptr(rho), _ptr(f), _ptr(b)))

    def stats(self):
        s = Stats()
        self.lib.st_get_stats(self.ctx, C.byref(s))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def hierarchy(self):
        h = Hierarchy()
        self.lib.st_get_hierarchy(self.ctx, C.byref(h))
        kinds = ["fine", "space", "time", "full"]
        forms = ["rho", "mk", "b4", "dense"]
        return [dict(n=h.n[i], nt=h.nt[i], kind=kinds[h.kind[i]], form=forms[h.form[i]], nodes=h.nodes[i])
                for i in range(h.n_levels)]

    def kernel_launches(self):
        return self.lib.st_kernel_launches(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.st_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
