"""ORACLE (test infrastructure only — see oracle/__init__.py).

First-order backward-difference time stepping on the spatial Q1 mesh — the comparison
method of PAPER.md:620 (sec. 4) and the limit the space-time solution must converge to
under time refinement (first order). Spatial element matrices are built
here by their own 2D/3D Gauss quadrature, independent of stfem.element_parts.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _spatial_elements(sdim: int, dx: float):
    """Q1 mass and stiffness on a dx^sdim element by 2^sdim-point Gauss quadrature."""
    gp = [-1.0 / math.sqrt(3.0), 1.0 / math.sqrt(3.0)]
    nloc = 2 ** sdim
    M = np.zeros((nloc, nloc))
    S = np.zeros((nloc, nloc))
    det = (dx / 2.0) ** sdim
    for q in itertools.product(gp, repeat=sdim):
        N = np.zeros(nloc)
        dN = np.zeros((nloc, sdim))
        for a in range(nloc):
            b = [(a >> d) & 1 for d in range(sdim)]
            ph = [0.5 * (1 - q[d]) if b[d] == 0 else 0.5 * (1 + q[d]) for d in range(sdim)]
            dph = [(-0.5 if b[d] == 0 else 0.5) * 2.0 / dx for d in range(sdim)]
            N[a] = np.prod(ph)
            for d in range(sdim):
                dN[a, d] = dph[d] * np.prod([ph[e] for e in range(sdim) if e != d])
        M += det * np.outer(N, N)
        S += det * dN @ dN.T
    return M, S


def backward_euler(n: int, sdim: int, C_e, k_e, q_of_t, nsteps: int, T0: float,
                   cons_plane, t_end: float = 1.0):
    """(M_C/dt + K_k) T^{m+1} = (M_C/dt) T^m + F(t_{m+1}) with T^0 = T0, constrained nodes
    of one spatial plane held at 0 (sink patch); spatially uniform source q_of_t(t)
    (rescaled units). C_e, k_e: per spatial element, x1 fastest.
    Returns the list of T^m, m = 0..nsteps."""
    nn = n + 1
    dx = 1.0 / n
    Me, Se = _spatial_elements(sdim, dx)
    if sdim == 2:
        e2, e1 = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        org = [e1.ravel(), e2.ravel()]
        strides = [1, nn]
    else:
        e3, e2, e1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        org = [e1.ravel(), e2.ravel(), e3.ravel()]
        strides = [1, nn, nn * nn]
    nloc = 2 ** sdim
    conn = np.zeros((org[0].size, nloc), dtype=np.int64)
    for a in range(nloc):
        for d in range(sdim):
            conn[:, a] += (org[d] + ((a >> d) & 1)) * strides[d]
    N = nn ** sdim
    rows = np.repeat(conn, nloc, axis=1).reshape(-1)
    cols = np.tile(conn, (1, nloc)).reshape(-1)
    C_e = np.asarray(C_e, dtype=np.float64).reshape(-1)
    k_e = np.asarray(k_e, dtype=np.float64).reshape(-1)
    M = sp.coo_matrix(((C_e[:, None, None] * Me).reshape(-1), (rows, cols)), shape=(N, N)).tocsr()
    K = sp.coo_matrix(((k_e[:, None, None] * Se).reshape(-1), (rows, cols)), shape=(N, N)).tocsr()
    load = np.zeros(N)
    np.add.at(load, conn.reshape(-1), np.repeat(np.full(conn.shape[0], dx ** sdim / nloc), nloc))
    dt = t_end / nsteps
    cons = np.asarray(cons_plane, dtype=bool)
    free = (~cons).astype(np.float64)
    Mf = sp.diags(free)
    A = (Mf @ (M / dt + K) @ Mf + sp.diags(cons.astype(np.float64))).tocsc()
    lu = spla.splu(A)
    T = np.full(N, float(T0))  # T^0 = T0 (IC) except on the sink, which holds 0 (R-2)
    T[cons] = 0.0
    out = [T.copy()]
    for m in range(nsteps):
        t1 = (m + 1) * dt
        rhs = (M / dt) @ T + q_of_t(t1) * load
        rhs = np.where(cons, 0.0, rhs)
        T = lu.solve(rhs)
        out.append(T.copy())
    return out
