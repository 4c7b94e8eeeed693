"""ORACLE (test infrastructure only — see oracle/__init__.py).

Assembled-matrix definition of the stabilised CG space-time FE method of
arxiv 2508.09589 and its direct solution. Every function cites the passage it follows.
fp64 throughout. Node numbering: x1 fastest, then x2 (then x3), then t (SPEC.md:49,
DESIGN.md reading R-10). Local element node a = b0 + 2 b1 + 4 b2 (+ 8 b3) with b_d the
0/1 position along direction d (x1, x2, [x3,] t).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import itertools
import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "Mesh", "Materials", "BCs", "Source", "Problem",
    "element_matrices", "element_parts", "connectivity", "simp",
    "assemble_K", "source_vector", "dirichlet", "apply_dirichlet",
    "pnorm_objective", "diffusion_timescale", "row_apply", "sensitivity_elements",
    "node_constraint", "source_rows",
]


# --------------------------------------------------------------------------------------
# Mesh, materials, conditions
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Mesh:
    """Regular n^sdim x nt space-time mesh of square(cubic)-in-space elements
    (sec. 3.1.2). Coordinates are the rescaled ones of PAPER.md:151-172:
    x* in [0,1]^sdim, t* in [0,1], so dx = 1/n, dt = 1/nt."""
    sdim: int
    n: int
    nt: int
    L: float = 1.0
    tau: float = 1.0

    def __post_init__(self):
        if self.sdim not in (2, 3):
            raise ValueError("sdim must be 2 or 3")
        if self.n < 2 or self.nt < 2:
            raise ValueError("element counts must be >= 2 (SPEC.md:50)")

    @property
    def dx(self) -> float:
        return 1.0 / self.n

    @property
    def dt(self) -> float:
        return 1.0 / self.nt

    @property
    def plane_nodes(self) -> int:
        return (self.n + 1) ** self.sdim

    @property
    def n_nodes(self) -> int:
        """N_n = (n_x1+1)(n_x2+1)(n_t+1)."""
        return self.plane_nodes * (self.nt + 1)

    @property
    def n_elems(self) -> int:
        """N_e = n_x1 n_x2 n_t."""
        return self.n ** self.sdim * self.nt

    @property
    def plane_elems(self) -> int:
        return self.n ** self.sdim


@dataclass(frozen=True)
class Materials:
    """Modified SIMP constants (eq. 'SIMP c' / 'SIMP k')."""
    C_ins: float = 1.0
    C_con: float = 1.0
    p_c: float = 1.0
    k_ins: float = 1e-3
    k_con: float = 1.0
    p_k: float = 3.0


@dataclass(frozen=True)
class BCs:
    """Dirichlet data (readings R-1..R-4): T = T0 on the t = 0 node plane
    (initial condition), T = 0 on a sink patch of the face x1 = 0 (all t): nodes whose
    transverse coordinates lie within `halfwidth` of `center` (width L/10 centred:
    PAPER.md:294 read on the left edge per BASELINE config 1). `all_walls` puts T = 0 on
    every spatial boundary node instead (Example 2)."""
    T0: float = 0.0
    has_patch: bool = True
    center: float = 0.5
    halfwidth: float = 0.05
    all_walls: bool = False


@dataclass(frozen=True)
class Source:
    """Heat source. kind:
      'uniform': Q = Q0;  'sin': Q = Q0 (1 + a sin(w t_phys))  (BASELINE configs)
      -> rescaled Q~ = Q tau / dT with dT = 1, t_phys = tau t*.
      'ex1': Q~ = 1/2 Q0 (1 - t)(1 + cos 50 t) with Q0 = 100 given already rescaled
             (tau = 1).
      'ex2': Q~ = Q0 exp(-|x - x0(t)|^2 / (2 sigma^2)), x0(t) = (L/2 + R cos(w t + pi/2),
             L/2 + R sin(w t + pi/2)), t physical.
    """
    kind: str = "uniform"
    Q0: float = 1.0
    a: float = 0.0
    w: float = 0.0
    sigma: float = 0.05
    R: float = 0.25


def simp(rho, mats: Materials, mesh: Mesh):
    """Element coefficients from the physical density:
    C = C_ins + (C_con - C_ins) rho^p_c,  k~ = (k_ins + (k_con - k_ins) rho^p_k) tau/L^2
    (rescaling k~ = k tau / L^2). Returns C, k~, dC/drho, dk~/drho."""
    rho = np.asarray(rho, dtype=np.float64)
    scale = mesh.tau / mesh.L ** 2
    C = mats.C_ins + (mats.C_con - mats.C_ins) * rho ** mats.p_c
    k = (mats.k_ins + (mats.k_con - mats.k_ins) * rho ** mats.p_k) * scale
    if mats.C_con == mats.C_ins:
        dC = np.zeros_like(rho)
    else:
        dC = mats.p_c * (mats.C_con - mats.C_ins) * rho ** (mats.p_c - 1.0)
    if mats.k_con == mats.k_ins:
        dk = np.zeros_like(rho)
    else:
        dk = mats.p_k * (mats.k_con - mats.k_ins) * rho ** (mats.p_k - 1.0) * scale
    return C, k, dC, dk


def diffusion_timescale(C: float, L: float, k: float) -> float:
    """tau_diff = C L^2 / k (eq. diffusionTimescale)."""
    return C * L * L / k


# --------------------------------------------------------------------------------------
# Element matrices by Gauss quadrature of the weak form
# --------------------------------------------------------------------------------------
_GP = np.array([-1.0 / math.sqrt(3.0), 1.0 / math.sqrt(3.0)])  # 2-point Gauss on [-1,1]
_GW = np.array([1.0, 1.0])


def _phi(b, s):
    return 0.5 * (1.0 - s) if b == 0 else 0.5 * (1.0 + s)


def _dphi(b):
    return -0.5 if b == 0 else 0.5


def element_parts(sdim: int, dx: float, dt: float):
    """The three element integrals of the weak form by
    2^(sdim+1)-point tensor Gauss quadrature, exact for these polynomial integrands
    (R-5):
        Gt[a,b] = int N_a dN_b/dt dV        (capacity / time-convection, C~_3 = C)
        Kt[a,b] = int dN_a/dt dN_b/dt dV    (time diffusion, multiplied by k_ad)
        Kx[a,b] = int grad_x N_a . grad_x N_b dV   (spatial conduction)
    Row index a is the test function v = N_a, column b the trial basis of T."""
    nd = sdim + 1
    nloc = 2 ** nd
    h = [dx] * sdim + [dt]
    detJ = float(np.prod([hh / 2.0 for hh in h]))
    Gt = np.zeros((nloc, nloc))
    Kt = np.zeros((nloc, nloc))
    Kx = np.zeros((nloc, nloc))
    bits = [[(a >> d) & 1 for d in range(nd)] for a in range(nloc)]
    for q in itertools.product(range(2), repeat=nd):
        s = [_GP[qq] for qq in q]
        w = float(np.prod([_GW[qq] for qq in q])) * detJ
        N = np.array([np.prod([_phi(bits[a][d], s[d]) for d in range(nd)]) for a in range(nloc)])
        dN = np.zeros((nloc, nd))
        for a in range(nloc):
            for d in range(nd):
                val = (2.0 / h[d]) * _dphi(bits[a][d])
                for d2 in range(nd):
                    if d2 != d:
                        val *= _phi(bits[a][d2], s[d2])
                dN[a, d] = val
        Gt += w * np.outer(N, dN[:, nd - 1])
        Kt += w * np.outer(dN[:, nd - 1], dN[:, nd - 1])
        Kx += w * dN[:, :sdim] @ dN[:, :sdim].T
    return Gt, Kt, Kx


def element_matrices(sdim: int, dx: float, dt: float):
    """Element matrix A_e = C_e G + k~_e Kx with the time-direction artificial diffusion
    k_ad = 1/2 C~ dt folded into G:
        G = Gt + (dt/2) Kt,   Kx as in element_parts.
    Returns (G, Kx)."""
    Gt, Kt, Kx = element_parts(sdim, dx, dt)
    return Gt + 0.5 * dt * Kt, Kx


# --------------------------------------------------------------------------------------
# Assembly
# --------------------------------------------------------------------------------------
def connectivity(mesh: Mesh) -> np.ndarray:
    """conn[e, a] = global node of local node a of element e; elements numbered
    e = e1 + n (e2 + n (... + n tau)), the C-order of rho[t][x2][x1] (R-10)."""
    n, nt, sd = mesh.n, mesh.nt, mesh.sdim
    nn = n + 1
    if sd == 2:
        t, e2, e1 = np.meshgrid(np.arange(nt), np.arange(n), np.arange(n), indexing="ij")
        coords = [e1.ravel(), e2.ravel(), t.ravel()]
        strides = [1, nn, nn * nn]
    else:
        t, e3, e2, e1 = np.meshgrid(np.arange(nt), np.arange(n), np.arange(n), np.arange(n),
                                    indexing="ij")
        coords = [e1.ravel(), e2.ravel(), e3.ravel(), t.ravel()]
        strides = [1, nn, nn * nn, nn ** 3]
    nd = sd + 1
    conn = np.zeros((coords[0].size, 2 ** nd), dtype=np.int64)
    for a in range(2 ** nd):
        idx = np.zeros(coords[0].size, dtype=np.int64)
        for d in range(nd):
            idx += (coords[d] + ((a >> d) & 1)) * strides[d]
        conn[:, a] = idx
    return conn


def _expand_rho(rho, mesh: Mesh):
    """rho per element: space-time ([nt] + [n]*sdim) or time-constant ([n]*sdim, extruded
    through time). Returns (flat per-element array, time_constant)."""
    rho = np.asarray(rho, dtype=np.float64)
    if rho.size == mesh.n_elems:
        return rho.reshape(-1), False
    if rho.size == mesh.plane_elems:
        return np.tile(rho.reshape(-1), mesh.nt), True
    raise ValueError(f"rho has {rho.size} entries; expected {mesh.n_elems} or {mesh.plane_elems}")


def assemble_K(mesh: Mesh, C_e, k_e):
    """Global all-at-once matrix J: sum of element matrices
    C_e G + k~_e Kx over the regular mesh, no boundary conditions. CSR, nonsymmetric."""
    G, Kx = element_matrices(mesh.sdim, mesh.dx, mesh.dt)
    conn = connectivity(mesh)
    vals = C_e[:, None, None] * G[None] + k_e[:, None, None] * Kx[None]
    nloc = conn.shape[1]
    rows = np.repeat(conn, nloc, axis=1).reshape(-1)
    cols = np.tile(conn, (1, nloc)).reshape(-1)
    K = sp.coo_matrix((vals.reshape(-1), (rows, cols)), shape=(mesh.n_nodes, mesh.n_nodes))
    return K.tocsr()


def _q_tilde(src: Source, mesh: Mesh, xs, ts):
    """Rescaled source Q~ at rescaled points (xs: list of coordinate arrays, ts: t*)."""
    if src.kind == "uniform":
        return np.full_like(ts, src.Q0 * mesh.tau)
    if src.kind == "sin":
        tp = mesh.tau * ts
        return src.Q0 * (1.0 + src.a * np.sin(src.w * tp)) * mesh.tau
    if src.kind == "ex1":
        return 0.5 * src.Q0 * (1.0 - ts) * (1.0 + np.cos(50.0 * ts))
    if src.kind == "ex2":
        tp = mesh.tau * ts
        x10 = 0.5 + src.R * np.cos(src.w * tp + 0.5 * np.pi)
        x20 = 0.5 + src.R * np.sin(src.w * tp + 0.5 * np.pi)
        r2 = (xs[0] - x10) ** 2 + (xs[1] - x20) ** 2
        return src.Q0 * np.exp(-r2 / (2.0 * src.sigma ** 2))
    raise ValueError(src.kind)


def source_vector(mesh: Mesh, src: Source):
    """f_a = sum_e int N_a Q~ dV, Q~ sampled at the 2^(sdim+1) Gauss
    points of every element (R-5)."""
    nd = mesh.sdim + 1
    nloc = 2 ** nd
    conn = connectivity(mesh)
    h = [mesh.dx] * mesh.sdim + [mesh.dt]
    detJ = float(np.prod([hh / 2.0 for hh in h]))
    n = mesh.n
    # element origin coordinates, in the element numbering of connectivity()
    e = np.arange(mesh.n_elems)
    org = []
    rem = e.copy()
    for d in range(mesh.sdim):
        org.append((rem % n) * mesh.dx)
        rem //= n
    org.append(rem * mesh.dt)
    fe = np.zeros((mesh.n_elems, nloc))
    bits = [[(a >> d) & 1 for d in range(nd)] for a in range(nloc)]
    for q in itertools.product(range(2), repeat=nd):
        s = [_GP[qq] for qq in q]
        pts = [org[d] + 0.5 * h[d] * (1.0 + s[d]) for d in range(nd)]
        Q = _q_tilde(src, mesh, pts[:-1], pts[-1])
        N = np.array([np.prod([_phi(bits[a][d], s[d]) for d in range(nd)]) for a in range(nloc)])
        fe += detJ * Q[:, None] * N[None, :]
    f = np.zeros(mesh.n_nodes)
    np.add.at(f, conn.reshape(-1), fe.reshape(-1))
    return f


def dirichlet(mesh: Mesh, bcs: BCs):
    """Constrained node set and prescribed values (R-1..R-4):
    the t = 0 node plane carries the initial condition T0; the sink patch
    (x1 = 0, transverse coordinates within halfwidth of center, all t) carries T = 0
    (PAPER.md:294). Returns (cons: bool[N_n], xD: float[N_n])."""
    nn = mesh.n + 1
    sd = mesh.sdim
    shape = (mesh.nt + 1,) + (nn,) * sd          # [t][x_sd]...[x1]
    cons = np.zeros(shape, dtype=bool)
    xD = np.zeros(shape)
    cons[0] = True
    xD[0] = bcs.T0
    if bcs.all_walls:
        wall = np.zeros((nn,) * sd, dtype=bool)
        for d in range(sd):
            sl0 = [slice(None)] * sd
            sl1 = [slice(None)] * sd
            sl0[d] = 0
            sl1[d] = nn - 1
            wall[tuple(sl0)] = True
            wall[tuple(sl1)] = True
        cons[:, wall] = True
        xD[:, wall] = 0.0
    elif bcs.has_patch:
        j = np.arange(nn)
        inside = np.abs(j / mesh.n - bcs.center) <= bcs.halfwidth * (1.0 + 1e-12)
        if sd == 2:
            # array axes [t][x2][x1]; face x1 = 0
            m = np.zeros((nn, nn), dtype=bool)
            m[inside, 0] = True
        else:
            m = np.zeros((nn, nn, nn), dtype=bool)
            m[np.ix_(inside, inside, np.array([0]))] = True
        cons[:, m] = True
        xD[:, m] = 0.0
    return cons.reshape(-1), xD.reshape(-1)


def apply_dirichlet(K, f, cons, xD):
    """Symmetric elimination with unit diagonal (R-1):
    b = f - K xD on free rows, b = xD on constrained rows; constrained rows and columns
    of K zeroed and the diagonal set to 1."""
    free = (~cons).astype(np.float64)
    b = f - K @ xD
    b = np.where(cons, xD, b)
    Mf = sp.diags(free)
    Kbc = (Mf @ K @ Mf + sp.diags(cons.astype(np.float64))).tocsr()
    return Kbc, b


# --------------------------------------------------------------------------------------
# Objective functionals
# --------------------------------------------------------------------------------------
def pnorm_objective(mesh: Mesh, T, P: float = 20.0):
    """phi = (sum_e T_avg,e^P)^(1/P), T_avg,e = mean of the element's 2^(sdim+1) nodal
    temperatures, and its gradient assembled per PAPER.md:593-595."""
    conn = connectivity(mesh)
    nloc = conn.shape[1]
    Tavg = T[conn].mean(axis=1)
    theta = np.sum(Tavg ** P)
    phi = theta ** (1.0 / P)
    ge = theta ** ((1.0 - P) / P) * Tavg ** (P - 1.0) / nloc
    g = np.zeros(mesh.n_nodes)
    np.add.at(g, conn.reshape(-1), np.repeat(ge, nloc))
    return phi, g


# --------------------------------------------------------------------------------------
# Problem: forward, adjoint, sensitivities
# --------------------------------------------------------------------------------------
@dataclass
class Problem:
    """One space-time problem: mesh, materials, conditions and source. Methods follow
    PAPER.md sec. 3.1 (system), 3.3.3 (adjoint and sensitivities)."""
    mesh: Mesh
    mats: Materials = field(default_factory=Materials)
    bcs: BCs = field(default_factory=BCs)
    src: Source = field(default_factory=Source)

    def coefficients(self, rho):
        r, tc = _expand_rho(rho, self.mesh)
        C, k, dC, dk = simp(r, self.mats, self.mesh)
        return C, k, dC, dk, tc

    def K(self, rho):
        """Unconstrained all-at-once matrix J(rho)."""
        C, k, _, _, _ = self.coefficients(rho)
        return assemble_K(self.mesh, C, k)

    def f(self):
        """Source vector f."""
        return source_vector(self.mesh, self.src)

    def constraints(self):
        return dirichlet(self.mesh, self.bcs)

    def system(self, rho):
        """(K_bc, b, cons, xD) after Dirichlet elimination."""
        cons, xD = self.constraints()
        Kbc, b = apply_dirichlet(self.K(rho), self.f(), cons, xD)
        return Kbc, b, cons, xD

    def forward(self, rho):
        """Direct solution of K_bc T = b (SuperLU); exact up to rounding (R-17)."""
        Kbc, b, _, _ = self.system(rho)
        lu = spla.splu(Kbc.tocsc())
        return lu.solve(b)

    def adjoint(self, rho, g):
        """lambda from J^T lambda = (dphi/ds)^T; constrained entries of
        g are ignored and lambda = 0 there (elimination, R-1)."""
        Kbc, _, cons, _ = self.system(rho)
        rhs = np.where(cons, 0.0, np.asarray(g, dtype=np.float64))
        lu = spla.splu(Kbc.tocsc())
        return lu.solve(rhs, trans="T")

    def solve_both(self, rho, g=None):
        """Forward and adjoint with one factorisation; g defaults to the compliance RHS f."""
        Kbc, b, cons, _ = self.system(rho)
        lu = spla.splu(Kbc.tocsc())
        T = lu.solve(b)
        if g is None:
            g = self.f()
        lam = lu.solve(np.where(cons, 0.0, g), trans="T")
        return T, lam

    def compliance(self, T):
        """Time-integrated thermal compliance phi = f^T T (R-8)."""
        return float(self.f() @ T)

    def compliance_rhs(self):
        """dphi/dT for phi = f^T T: f with constrained entries zeroed."""
        cons, _ = self.constraints()
        return np.where(cons, 0.0, self.f())

    def sensitivity(self, rho, T, lam):
        """dphi/drho_e = -lambda_e^T (dC/drho G + dk~/drho Kx) T_e with the
        k_ad(C(rho)) term inside G (R-9); full T incl. prescribed values,
        lambda = 0 on constrained nodes. Time-constant rho: summed through time
        (transposed extrusion)."""
        _, _, dC, dk, tc = self.coefficients(rho)
        G, Kx = element_matrices(self.mesh.sdim, self.mesh.dx, self.mesh.dt)
        conn = connectivity(self.mesh)
        Te = np.asarray(T)[conn]
        Le = np.asarray(lam)[conn]
        gG = np.einsum("ea,ab,eb->e", Le, G, Te)
        gK = np.einsum("ea,ab,eb->e", Le, Kx, Te)
        dJ = -(dC * gG + dk * gK)
        if tc:
            dJ = dJ.reshape(self.mesh.nt, -1).sum(axis=0)
            return dJ.reshape((self.mesh.n,) * self.mesh.sdim)
        return dJ.reshape((self.mesh.nt,) + (self.mesh.n,) * self.mesh.sdim)


# --------------------------------------------------------------------------------------
# Sampled evaluation for full-size certification (R-21): the same element matrices,
# summed element by element for a few rows / elements only (no global assembly).
# --------------------------------------------------------------------------------------
def _node_coords(mesh: Mesh, node):
    nn = mesh.n + 1
    c = []
    for _ in range(mesh.sdim):
        c.append(node % nn)
        node //= nn
    c.append(node)  # time plane
    return c


def node_constraint(mesh: Mesh, bcs: BCs, node):
    """(constrained, prescribed value) of ONE node, the rule of dirichlet() (R-1..R-4)
    evaluated at the node's coordinates: the t = 0 plane carries T0; the sink patch
    (x1 = 0, transverse indices j with |j/n - center| <= halfwidth, all t) or, with all_walls, every
    spatial boundary node carries 0. Sampled certification only (R-21)."""
    c = _node_coords(mesh, int(node))
    sp_c, t = c[:-1], c[-1]
    if bcs.all_walls:
        wall = any(x == 0 or x == mesh.n for x in sp_c)
        if wall:
            return True, 0.0
    elif bcs.has_patch and sp_c[0] == 0:
        if all(abs(j / mesh.n - bcs.center) <= bcs.halfwidth * (1.0 + 1e-12) for j in sp_c[1:]):
            return True, 0.0
    if t == 0:
        return True, bcs.T0
    return False, 0.0


def _elem_index(mesh: Mesh, e):
    """Flat element index e1 + n (e2 + ... + n tau) of element coordinates e (R-10)."""
    eidx, mul = 0, 1
    for d in range(mesh.sdim + 1):
        eidx += e[d] * mul
        mul *= mesh.n
    return eidx


def _rho_of(prob: "Problem", rho, eidx):
    """Density of space-time element eidx: rho is per space-time element or time-constant
    (extruded through time)."""
    mesh = prob.mesh
    r = np.asarray(rho).reshape(-1)
    if r.size == mesh.n_elems:
        return float(r[eidx])
    if r.size == mesh.plane_elems:
        return float(r[eidx % mesh.plane_elems])
    raise ValueError("rho size")


def row_apply(prob: "Problem", rho, x, nodes, transpose=False):
    """(K_bc x)[nodes] (or (K_bc^T x)[nodes]) for the eliminated all-at-once matrix
    (R-1), summing A_e = C_e G + k~_e Kx (element_matrices, quadrature; SIMP
    coefficients by simp()) over the elements adjacent to each node. Purely
    local: x only needs to support x[node] for the nodes of the rows' stencils (a numpy array or a
    mapping), the coefficients are evaluated for the touched elements only, and constraints by
    node_constraint() — so it scales to the full BASELINE sizes (R-21)."""
    mesh = prob.mesh
    G, Kx = element_matrices(mesh.sdim, mesh.dx, mesh.dt)
    nd = mesh.sdim + 1
    nloc = 2 ** nd
    nn = mesh.n + 1
    strides = [nn ** d for d in range(mesh.sdim)] + [nn ** mesh.sdim]
    ecount = [mesh.n] * mesh.sdim + [mesh.nt]
    out = np.zeros(len(nodes))
    for s, node in enumerate(nodes):
        node = int(node)
        cons, _ = node_constraint(mesh, prob.bcs, node)
        if cons:
            out[s] = x[node]
            continue
        cc = _node_coords(mesh, node)
        acc = 0.0
        for a in range(nloc):  # the node is local corner a of the element at cc - bits(a)
            e = [cc[d] - ((a >> d) & 1) for d in range(nd)]
            if any(e[d] < 0 or e[d] >= ecount[d] for d in range(nd)):
                continue
            C, k, _, _ = simp(_rho_of(prob, rho, _elem_index(mesh, e)), prob.mats, mesh)
            Ae = C * G + k * Kx
            for b in range(nloc):
                gb = sum((e[d] + ((b >> d) & 1)) * strides[d] for d in range(nd))
                if node_constraint(mesh, prob.bcs, gb)[0]:
                    continue
                acc += (Ae[b, a] if transpose else Ae[a, b]) * x[gb]
        out[s] = acc
    return out


def source_rows(mesh: Mesh, src: Source, nodes):
    """f[nodes] of source_vector() (R-5): per node, the sum over its adjacent
    elements of the 2^(sdim+1)-point Gauss quadrature of N_a Q~ (sampled certification, R-21)."""
    nd = mesh.sdim + 1
    nloc = 2 ** nd
    h = [mesh.dx] * mesh.sdim + [mesh.dt]
    detJ = float(np.prod([hh / 2.0 for hh in h]))
    ecount = [mesh.n] * mesh.sdim + [mesh.nt]
    bits = [[(a >> d) & 1 for d in range(nd)] for a in range(nloc)]
    out = np.zeros(len(nodes))
    for s, node in enumerate(nodes):
        cc = _node_coords(mesh, int(node))
        acc = 0.0
        for a in range(nloc):
            e = [cc[d] - bits[a][d] for d in range(nd)]
            if any(e[d] < 0 or e[d] >= ecount[d] for d in range(nd)):
                continue
            org = [e[d] * h[d] for d in range(nd)]
            for q in itertools.product(range(2), repeat=nd):
                sq = [_GP[qq] for qq in q]
                pts = [np.array([org[d] + 0.5 * h[d] * (1.0 + sq[d])]) for d in range(nd)]
                Q = float(_q_tilde(src, mesh, pts[:-1], pts[-1])[0])
                N = np.prod([_phi(bits[a][d], sq[d]) for d in range(nd)])
                acc += detJ * Q * N
        out[s] = acc
    return out


def sensitivity_elements(prob: "Problem", rho, T, lam, elems):
    """dphi/drho_e (R-9) of the space-time elements `elems` (index
    e1 + n (e2 + ... + n tau)), full T and lambda = 0 on constrained nodes. Purely local like
    row_apply: T and lam only need T[node] / lam[node] at the elements' nodes."""
    mesh = prob.mesh
    G, Kx = element_matrices(mesh.sdim, mesh.dx, mesh.dt)
    nd = mesh.sdim + 1
    nloc = 2 ** nd
    nn = mesh.n + 1
    strides = [nn ** d for d in range(mesh.sdim)] + [nn ** mesh.sdim]
    out = np.zeros(len(elems))
    for s, e in enumerate(elems):
        e = int(e)
        ec = []
        r = e
        for d in range(mesh.sdim):
            ec.append(r % mesh.n)
            r //= mesh.n
        ec.append(r)
        idx = [sum((ec[d] + ((a >> d) & 1)) * strides[d] for d in range(nd)) for a in range(nloc)]
        Te = np.array([T[i] for i in idx], dtype=np.float64)
        Le = np.array([0.0 if node_constraint(mesh, prob.bcs, i)[0] else lam[i] for i in idx], dtype=np.float64)
        _, _, dC, dk = simp(_rho_of(prob, rho, e), prob.mats, mesh)
        out[s] = -(dC * (Le @ G @ Te) + dk * (Le @ Kx @ Te))
    return out
