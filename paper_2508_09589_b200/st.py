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
ST_SRC_UNIFORM, ST_SRC_SIN, ST_SRC_EX1, ST_SRC_EX2 = 0, 1, 2, 3
ST_SMOOTH_JACOBI, ST_SMOOTH_GMRES = 0, 2  # st.h: the GMRES(k)-Jacobi smoother of the paper (one GPU)
ST_KRYLOV_FGMRES, ST_KRYLOV_GMRES = 0, 1
ST_COARSE_DENSE, ST_COARSE_GMRES = 0, 1
ST_KERNELS_TMA, ST_KERNELS_CPASYNC, ST_KERNELS_GENERIC, ST_KERNELS_TMA2D = 0, 1, 2, 3


class Grid(C.Structure):
    _fields_ = [("sdim", C.c_int32), ("n", C.c_int64), ("nt", C.c_int64), ("L", C.c_double), ("tau", C.c_double)]


class Materials(C.Structure):
    _fields_ = [("C_ins", C.c_double), ("C_con", C.c_double), ("p_c", C.c_double),
                ("k_ins", C.c_double), ("k_con", C.c_double), ("p_k", C.c_double)]


class BCs(C.Structure):
    _fields_ = [("T0", C.c_double), ("has_patch", C.c_int32), ("face", C.c_int32),
                ("center", C.c_double), ("halfwidth", C.c_double), ("all_walls", C.c_int32)]


class Source(C.Structure):
    _fields_ = [("kind", C.c_int32), ("Q0", C.c_double), ("a", C.c_double), ("w", C.c_double),
                ("sigma", C.c_double), ("R", C.c_double)]


class Options(C.Structure):
    _fields_ = [("design_mode", C.c_int32), ("rtol", C.c_double), ("maxit", C.c_int32), ("restart", C.c_int32),
                ("smoother", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("omega", C.c_double),
                ("lambda_crit", C.c_double), ("coarse_max_nodes", C.c_int64), ("max_levels", C.c_int32),
                ("full_coarsening", C.c_int32), ("use_graphs", C.c_int32), ("verbose", C.c_int32),
                ("agg_nodes", C.c_int64), ("nu_coarse", C.c_int32),
                ("krylov", C.c_int32), ("coarse_solver", C.c_int32), ("coarse_rtol", C.c_double),
                ("coarse_maxit", C.c_int32), ("kernel_family", C.c_int32), ("chunk_planes", C.c_int32),
                ("max_ctas", C.c_int32), ("fuse_prolong", C.c_int32),
                ("omega_factor", C.c_double), ("dgks_eta", C.c_double), ("graph_max_nodes", C.c_int64),
                ("smoother_rtol", C.c_double), ("nu_fine_nodes", C.c_int64),
                ("pitch_align", C.c_int32)]


ST_COMM_NONE, ST_COMM_NCCL, ST_COMM_HOST = 0, 1, 2
ST_NCCL_ID_BYTES = 128
_DP = C.POINTER(C.c_double)
CB_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, _DP, _DP, C.c_int64)
CB_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, _DP, C.c_int64)
CB_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, _DP, _DP, C.c_int64)


class HostComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("sendrecv", CB_SENDRECV), ("allreduce_sum", CB_ALLREDUCE),
                ("allgather", CB_ALLGATHER)]


class Dist(C.Structure):
    _fields_ = [("nccl_comm", C.c_void_p), ("rank", C.c_int32), ("size", C.c_int32),
                ("cuda_stream", C.c_void_p), ("device", C.c_int32), ("transport", C.c_int32),
                ("host", HostComm)]


class Plan(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n_dist_levels", C.c_int32), ("n", C.c_int64 * 32), ("nt", C.c_int64 * 32),
                ("kind", C.c_int32 * 32), ("dist", C.c_int32 * 32), ("layer0", C.c_int64 * 32),
                ("n_layers", C.c_int64 * 32), ("local_layers", C.c_int64 * 32), ("plane0", C.c_int64),
                ("n_planes", C.c_int64)]


class Layout(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("plane0", C.c_int64), ("n_planes", C.c_int64),
                ("layer0", C.c_int64), ("n_layers", C.c_int64), ("rho_layers", C.c_int64),
                ("nodes_local", C.c_int64), ("design_local", C.c_int64), ("n_levels", C.c_int32),
                ("n_dist_levels", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("restarts", C.c_int32), ("rel_residual", C.c_double),
                ("setup_ms", C.c_double), ("solve_ms", C.c_double), ("n_levels", C.c_int32),
                ("converged", C.c_int32), ("vcycles", C.c_int32), ("setups", C.c_int64)]


class TsStats(C.Structure):
    _fields_ = [("steps", C.c_int32), ("max_step_iterations", C.c_int32), ("cg_iterations", C.c_int64),
                ("ms", C.c_double), ("launches", C.c_int64)]


class Hierarchy(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n", C.c_int64 * 32), ("nt", C.c_int64 * 32),
                ("kind", C.c_int32 * 32), ("form", C.c_int32 * 32), ("nodes", C.c_int64 * 32),
                ("omega", C.c_double * 32), ("lam_max", C.c_double * 32)]


EXPORTS = ["st_abi_version", "st_default_options", "st_setup", "st_destroy", "st_solve", "st_adjoint",
           "st_sensitivity", "st_apply", "st_vcycle", "st_rhs", "st_filter", "st_oc_update", "st_dot", "st_pnorm", "st_level_apply", "st_level_transfer", "st_bench_op", "st_get_stats", "st_get_hierarchy",
           "st_local_layout", "st_nccl_unique_id", "st_nccl_comm_init", "st_nccl_comm_destroy", "st_plan",
           "st_struct_sizes",
           "st_num_nodes", "st_num_design", "st_kernel_launches", "st_strerror", "st_last_error", "st_timestep", "st_nccl_selftest", "st_pde_filter", "st_pde_filter_grad"]

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
    lib.st_design_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   P(Stats)]
    lib.st_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
    lib.st_rhs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.st_vcycle.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    lib.st_filter.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double]
    lib.st_oc_update.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                 P(C.c_double)]
    lib.st_dot.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, P(C.c_double)]
    lib.st_pde_filter.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                  C.c_void_p]
    lib.st_pde_filter_grad.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_void_p]
    lib.st_pnorm.argtypes = [C.c_void_p, C.c_void_p, C.c_double, P(C.c_double), C.c_void_p]
    lib.st_level_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    lib.st_level_transfer.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    lib.st_bench_op.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.st_get_stats.argtypes = [C.c_void_p, P(Stats)]
    lib.st_timestep.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, P(TsStats)]
    lib.st_get_hierarchy.argtypes = [C.c_void_p, P(Hierarchy)]
    lib.st_local_layout.argtypes = [C.c_void_p, P(Layout)]
    lib.st_nccl_unique_id.argtypes = [C.c_char_p]
    lib.st_nccl_comm_init.argtypes = [C.c_char_p, C.c_int32, C.c_int32, P(C.c_void_p)]
    lib.st_nccl_comm_destroy.argtypes = [C.c_void_p]
    lib.st_nccl_selftest.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P(C.c_int32)]
    lib.st_plan.argtypes = [P(Grid), P(Materials), P(BCs), P(Options), C.c_int32, C.c_int32, P(Plan)]
    lib.st_struct_sizes.argtypes = [P(C.c_int64)]
    for name in ("st_num_nodes", "st_num_design", "st_kernel_launches"):
        getattr(lib, name).argtypes = [C.c_void_p]
        getattr(lib, name).restype = C.c_int64
    lib.st_strerror.argtypes = [C.c_int]
    lib.st_strerror.restype = C.c_char_p
    lib.st_last_error.restype = C.c_char_p
    lib.st_abi_version.restype = C.c_int
    _lib = lib
    return lib


def _ptr(a, n=None, what="vector"):
    """Data pointer of a torch tensor / numpy array (contiguous fp64). n: the element count the C ABI
    will read or write through the pointer; a different size is an error (no out-of-bounds access)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous() or str(a.dtype) != "torch.float64":
            raise ValueError("tensors must be contiguous float64")
        size, ptr = a.numel(), a.data_ptr()
    else:
        import numpy as np
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
            raise ValueError("arrays must be C-contiguous float64")
        size, ptr = a.size, a.ctypes.data
    if n is not None and size != n:
        raise ValueError(f"{what}: {size} elements, the library expects {n}")
    return ptr


class TorchHostComm:
    """ST_COMM_HOST transport implemented with torch.distributed on host tensors (e.g. a gloo
    group). Marshalling only: the library stages device planes through pinned host buffers and
    calls these functions; any number of ranks may share one GPU."""

    def __init__(self, group=None):
        import numpy as np
        import torch
        import torch.distributed as dist
        self.np, self.torch, self.dist, self.group = np, torch, dist, group
        self.size = dist.get_world_size(group)
        self._cbs = (CB_SENDRECV(self._sendrecv), CB_ALLREDUCE(self._allreduce), CB_ALLGATHER(self._allgather))
        self.struct = HostComm(None, *self._cbs)

    def _t(self, ptr, n):
        return self.torch.from_numpy(self.np.ctypeslib.as_array(ptr, (int(n),)))

    def _fail(self, what, e):
        import sys
        sys.stderr.write(f"TorchHostComm.{what} failed: {e!r}\n")
        self.last_error = repr(e)
        return 1

    def _sendrecv(self, user, peer, send, recv, count):
        try:
            s, r = self._t(send, count).clone(), self._t(recv, count)
            reqs = [self.dist.isend(s, int(peer), group=self.group), self.dist.irecv(r, int(peer), group=self.group)]
            for q in reqs:
                q.wait()
            return 0
        except Exception as e:  # noqa: BLE001
            return self._fail("sendrecv", e)

    def _allreduce(self, user, buf, count):
        try:
            self.dist.all_reduce(self._t(buf, count), group=self.group)
            return 0
        except Exception as e:  # noqa: BLE001
            return self._fail("allreduce", e)

    def _allgather(self, user, send, recv, count):
        try:
            parts = [self.torch.empty(int(count), dtype=self.torch.float64) for _ in range(self.size)]
            self.dist.all_gather(parts, self._t(send, count).clone(), group=self.group)
            self._t(recv, count * self.size).copy_(self.torch.cat(parts))
            return 0
        except Exception as e:  # noqa: BLE001
            return self._fail("allgather", e)


STRUCTS = [Grid, Materials, BCs, Source, Options, Dist, Stats, Hierarchy, Layout, Plan, TsStats]


def plan(sdim, n, nt, rank=0, size=1, mats=(1.0, 1.0, 1.0, 1e-3, 1.0, 3.0), tau=1.0, L=1.0, has_patch=True,
         **opts):
    """Host-only st_plan: the hierarchy and this rank's slab of every level (no GPU needed)."""
    lib = load_library()
    o = Options()
    lib.st_default_options(C.byref(o))
    for k, v in opts.items():
        setattr(o, k, v)
    p = Plan()
    rc = lib.st_plan(C.byref(Grid(sdim, n, nt, L, tau)), C.byref(Materials(*mats)),
                     C.byref(BCs(0.0, 1 if has_patch else 0, 0, 0.5, 0.05, 0)), C.byref(o), rank, size, C.byref(p))
    if rc != ST_OK:
        raise StError(rc, lib.st_last_error().decode())
    kinds = ["fine", "space", "time", "full"]
    levels = [dict(n=p.n[i], nt=p.nt[i], kind=kinds[p.kind[i]], dist=bool(p.dist[i]), layer0=p.layer0[i],
                   n_layers=p.n_layers[i], local_layers=p.local_layers[i]) for i in range(p.n_levels)]
    return dict(levels=levels, n_dist=p.n_dist_levels, plane0=p.plane0, n_planes=p.n_planes)


def nccl_unique_id():
    lib = load_library()
    buf = C.create_string_buffer(ST_NCCL_ID_BYTES)
    if lib.st_nccl_unique_id(buf) != ST_OK:
        raise StError(-7, lib.st_last_error().decode())
    return buf.raw


def nccl_selftest(comm, rank: int, size: int) -> int:
    """st_nccl_selftest: checks the communicator's rank count and runs allreduce / allgather / grouped
    send-recv through the library's NCCL entry points; returns ncclCommCount."""
    lib = load_library()
    n = C.c_int32(-1)
    if lib.st_nccl_selftest(comm, rank, size, C.byref(n)) != ST_OK:
        raise StError(-7, lib.st_last_error().decode())
    return n.value


def nccl_comm_init(uid: bytes, rank: int, size: int):
    lib = load_library()
    comm = C.c_void_p()
    if lib.st_nccl_comm_init(uid, rank, size, C.byref(comm)) != ST_OK:
        raise StError(-7, lib.st_last_error().decode())
    return comm


class Solver:
    """One space-time problem: st_setup at construction, st_destroy on close().

    Time slabs: pass rank/size and either host_comm (a TorchHostComm; ranks may share a GPU)
    or nccl_comm (from nccl_unique_id / nccl_comm_init; one GPU per rank). Vectors are then
    this rank's owned planes (see layout())."""

    def __init__(self, sdim, n, nt, mats=(1.0, 1.0, 1.0, 1e-3, 1.0, 3.0), T0=0.0, has_patch=True,
                 center=0.5, halfwidth=0.05, source=("uniform", 1.0, 0.0, 0.0), L=1.0, tau=1.0,
                 time_constant=False, stream=None, device=None, rank=0, size=1, host_comm=None,
                 nccl_comm=None, all_walls=False, **opts):
        """source: (kind, Q0, a, w[, sigma, R]) with kind 'uniform' | 'sin' | 'ex1' | 'ex2' (st.h)."""
        self.lib = load_library()
        self.grid = Grid(sdim, n, nt, L, tau)
        self.mats = Materials(*mats)
        self.bcs = BCs(T0, 1 if has_patch else 0, 0, center, halfwidth, 1 if all_walls else 0)
        kind = {"uniform": ST_SRC_UNIFORM, "sin": ST_SRC_SIN, "ex1": ST_SRC_EX1, "ex2": ST_SRC_EX2}[source[0]]
        vals = list(source[1:]) + [0.0] * (5 - len(source[1:]))
        self.src = Source(kind, *vals[:5])
        o = Options()
        self.lib.st_default_options(C.byref(o))
        o.design_mode = ST_TIME_CONSTANT if time_constant else ST_SPACE_TIME
        for k, v in opts.items():
            if not hasattr(o, k):
                raise TypeError(f"unknown option {k}")
            setattr(o, k, v)
        self.opts = o
        transport = ST_COMM_NONE
        if size > 1:
            transport = ST_COMM_NCCL if nccl_comm is not None else ST_COMM_HOST
            if transport == ST_COMM_HOST and host_comm is None:
                raise ValueError("size > 1 needs host_comm or nccl_comm")
        self._host_comm = host_comm  # keeps the callbacks alive
        d = Dist(nccl_comm, rank, size, stream if stream is not None else None, -1 if device is None else device,
                 transport, host_comm.struct if host_comm is not None else HostComm())
        h = C.c_void_p()
        self._check(self.lib.st_setup(C.byref(self.grid), C.byref(self.mats), C.byref(self.bcs),
                                      C.byref(self.src), C.byref(o), C.byref(d), C.byref(h)))
        self.ctx = h

    def options(self):
        """The st_options_t this context was set up with (library defaults + the caller's overrides)."""
        return {name: getattr(self.opts, name) for name, _ in Options._fields_}

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

    def _nodes(self, a, what):
        return _ptr(a, self.n_nodes, what)

    def _rho(self, rho):
        return _ptr(rho, self.n_design, "rho")

    def _owned_design(self):
        """Element count of this rank's owned design layers (st_filter / st_oc_update / dJ)."""
        lay = self.layout()
        nsp = int(self.grid.n) ** int(self.grid.sdim)
        return nsp * (lay["n_layers"] if lay["rho_layers"] else 1)

    def solve(self, rho, T, allow_nc=False):
        return self._check(self.lib.st_solve(self.ctx, self._rho(rho), self._nodes(T, "T")), allow_nc)

    def adjoint(self, rho, dJdT, lam, allow_nc=False):
        return self._check(self.lib.st_adjoint(self.ctx, self._rho(rho), self._nodes(dJdT, "dJdT"),
                                               self._nodes(lam, "lambda")), allow_nc)

    def sensitivity(self, rho, T, lam, dJ):
        return self._check(self.lib.st_sensitivity(self.ctx, self._rho(rho), self._nodes(T, "T"),
                                                   self._nodes(lam, "lambda"), _ptr(dJ, self._owned_design(), "dJ")))

    def design_step(self, rho, dJdT, T, lam, dJ, allow_nc=False):
        """st_design_step: forward solve, adjoint solve and sensitivities in one call (host vectors: result
        copies overlap the next phase). Returns (forward stats, adjoint stats)."""
        fs = Stats()
        self._check(self.lib.st_design_step(self.ctx, self._rho(rho), self._nodes(dJdT, "dJdT"), self._nodes(T, "T"),
                                            self._nodes(lam, "lambda"), _ptr(dJ, self._owned_design(), "dJ"),
                                            C.byref(fs)), allow_nc)
        return {k: getattr(fs, k) for k, _ in Stats._fields_}, self.stats()

    def apply(self, rho, x, y, transpose=False, bc=True):
        return self._check(self.lib.st_apply(self.ctx, self._rho(rho), self._nodes(x, "x"), self._nodes(y, "y"),
                                             int(transpose), int(bc)))

    def filter(self, x, out, transpose=False, radius=2.0):
        """Density filter F (transpose: F^T, the chain rule) of config 5 (R-13)."""
        nown = self._owned_design()
        nout = nown if transpose else self.n_design
        return self._check(self.lib.st_filter(self.ctx, _ptr(x, nown, "filter input"), _ptr(out, nout, "filter output"),
                                              int(transpose), radius))

    def oc_update(self, rho, dJ, rho_new, volfrac=0.4, move=0.2, rho_min=1e-3):
        """Optimality-criteria step with bisection on the volume multiplier; returns Lambda."""
        nown = self._owned_design()
        lam = C.c_double()
        self._check(self.lib.st_oc_update(self.ctx, _ptr(rho, nown, "rho"), _ptr(dJ, nown, "dJ"), volfrac, move,
                                          rho_min, _ptr(rho_new, nown, "rho_new"), C.byref(lam)))
        return lam.value

    def pde_filter(self, gamma, gamma_bar, gamma_e=None, rx=None, rt=None, beta=32.0, eta=0.5):
        """The paper's PDE filter + Heaviside projection; radii default to 2.4 dx / 2.4 dt
        (rescaled). Returns the filter's CG iterations."""
        n, nt = int(self.grid.n), int(self.grid.nt)
        rx = 2.4 / n if rx is None else rx
        rt = 2.4 / nt if rt is None else rt
        ne = self.n_design
        self._check(self.lib.st_pde_filter(self.ctx, _ptr(gamma, ne, "gamma"), rx, rt, beta, eta,
                                           _ptr(gamma_e, ne, "gamma_e"), _ptr(gamma_bar, ne, "gamma_bar")))
        return self.stats()["iterations"]

    def pde_filter_grad(self, gamma_e, dphi_dgbar, out, rx=None, rt=None, beta=32.0, eta=0.5):
        """Chain rule of the filter + projection."""
        n, nt = int(self.grid.n), int(self.grid.nt)
        rx = 2.4 / n if rx is None else rx
        rt = 2.4 / nt if rt is None else rt
        ne = self.n_design
        self._check(self.lib.st_pde_filter_grad(self.ctx, _ptr(gamma_e, ne, "gamma_e"), _ptr(dphi_dgbar, ne, "dphi"),
                                                rx, rt, beta, eta, _ptr(out, ne, "out")))
        return self.stats()["iterations"]

    def pnorm(self, T, P=20.0, grad=None):
        """phi = (sum_e Tavg_e^P)^(1/P); grad (optional) receives dphi/dT."""
        phi = C.c_double()
        self._check(self.lib.st_pnorm(self.ctx, self._nodes(T, "T"), P, C.byref(phi),
                                      None if grad is None else self._nodes(grad, "grad")))
        return phi.value

    def dot(self, x, y):
        out = C.c_double()
        self._check(self.lib.st_dot(self.ctx, self._nodes(x, "x"), self._nodes(y, "y"), C.byref(out)))
        return out.value

    def vcycle(self, rho, b, z, transpose=False):
        """z = one V-cycle applied to b (test hook)."""
        return self._check(self.lib.st_vcycle(self.ctx, self._rho(rho), self._nodes(b, "b"), self._nodes(z, "z"),
                                              int(transpose)))

    def level_apply(self, rho, level, x, y, transpose=False):
        h = self.hierarchy()
        if not 0 <= level < len(h):
            raise ValueError("level out of range")
        nd = h[level]["nodes"]
        return self._check(self.lib.st_level_apply(self.ctx, self._rho(rho), level, _ptr(x, nd, "x"), _ptr(y, nd, "y"),
                                                   int(transpose)))

    def level_transfer(self, rho, level, vin, vout, restrict=False):
        """st_level_transfer: vout = P^T vin (level -> level + 1) or vout = P vin (level + 1 -> level)."""
        h = self.hierarchy()
        if not 0 <= level < len(h) - 1:
            raise ValueError("level out of range")
        nf, nc = h[level]["nodes"], h[level + 1]["nodes"]
        a, b = (nf, nc) if restrict else (nc, nf)
        return self._check(self.lib.st_level_transfer(self.ctx, self._rho(rho), level, _ptr(vin, a, "in"),
                                                      _ptr(vout, b, "out"), int(bool(restrict))))

    def bench_op(self, rho, level, mode, reps, transpose=False):
        """Enqueue `reps` launches of the level operator kernel (internal work vectors) without
        synchronising."""
        return self._check(self.lib.st_bench_op(self.ctx, self._rho(rho), level, mode, int(transpose), reps))

    def rhs(self, rho, f=None, b=None):
        return self._check(self.lib.st_rhs(self.ctx, self._rho(rho), None if f is None else self._nodes(f, "f"),
                                           None if b is None else self._nodes(b, "b")))

    def timestep(self, rho, nsteps, T):
        """The GPU time-stepping baseline (st_timestep): backward Euler with nsteps steps; T receives the
        (nsteps + 1) x (n+1)^sdim nodal temperatures. Returns st_ts_stats_t as a dict."""
        st = TsStats()
        plane = (int(self.grid.n) + 1) ** int(self.grid.sdim)
        self._check(self.lib.st_timestep(self.ctx, self._rho(rho), int(nsteps), _ptr(T, plane * (nsteps + 1), "T"),
                                         C.byref(st)))
        return {k: getattr(st, k) for k, _ in TsStats._fields_}

    def stats(self):
        s = Stats()
        self.lib.st_get_stats(self.ctx, C.byref(s))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def hierarchy(self):
        h = Hierarchy()
        self.lib.st_get_hierarchy(self.ctx, C.byref(h))
        kinds = ["fine", "space", "time", "full"]
        forms = ["rho", "mk", "b4", "dense"]
        return [dict(n=h.n[i], nt=h.nt[i], kind=kinds[h.kind[i]], form=forms[h.form[i]], nodes=h.nodes[i],
                     omega=h.omega[i], lam_max=h.lam_max[i]) for i in range(h.n_levels)]

    def layout(self):
        lay = Layout()
        self.lib.st_local_layout(self.ctx, C.byref(lay))
        return {k: getattr(lay, k) for k, _ in Layout._fields_}

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
