"""ORACLE (test infrastructure only — see oracle/__init__.py).

The paper's design regularisation (sec. 2.4.2 "Filtering and projection"), the
space-time PDE filter and Heaviside projection, and their chain rule:

  filter      -d/dxi_i (d_ij d g~/dxi_j) + g~ = g on the space-time domain Pi, natural (Neumann)
              boundaries, d = diag(r_x^2/12, ..., r_t^2/12), discretised with the
              Q1 space-time elements of the state mesh (Lazarov & Sigmund 2011, cited there):
                  (K_f + M_f) g~_nodal = T_f g,   K_f, M_f by tensor Gauss quadrature,
                  (T_f g)_a = sum_e g_e int_e N_a dV,
              and the element value of the filtered field as the mean of its nodal values
              (R-25; the paper does not print the node -> element map);
  projection  g_bar = (tanh(beta eta) + tanh(beta (g~ - eta))) / (tanh(beta eta) + tanh(beta (1 - eta)))
              (eta = 0.5, beta = 32);
  chain rule  dphi/dg = T_f^T (K_f + M_f)^-1 A^T (dg_bar/dg~ .* dphi/dg_bar)  (the
              sensitivities pass through another reaction-diffusion solve), A the node -> element mean.

The radii are in the rescaled coordinates of the mesh (x in [0, 1]^d, t in [0, 1]); the paper's
defaults are r_x = 2.4 dx and r_t = 2.4 dt. Direct SuperLU solves; plain assembly.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .stfem import Mesh, connectivity

_GP = np.array([-1.0 / math.sqrt(3.0), 1.0 / math.sqrt(3.0)])


def _phi(b, s):
    return 0.5 * (1.0 - s) if b == 0 else 0.5 * (1.0 + s)


def _dphi(b):
    return -0.5 if b == 0 else 0.5


def filter_element_matrix(sdim: int, dx: float, dt: float, rx: float, rt: float):
    """F_e = int (grad N . d grad N + N N) dV over one space-time element, d = diag(rx^2/12 (x sdim),
    rt^2/12), by 2^(sdim+1)-point Gauss quadrature (exact for these polynomials)."""
    nd = sdim + 1
    nloc = 2 ** nd
    h = [dx] * sdim + [dt]
    dcoef = [rx * rx / 12.0] * sdim + [rt * rt / 12.0]
    detJ = float(np.prod([hh / 2.0 for hh in h]))
    F = np.zeros((nloc, nloc))
    bits = [[(a >> d) & 1 for d in range(nd)] for a in range(nloc)]
    for q in itertools.product(range(2), repeat=nd):
        s = [_GP[qq] for qq in q]
        N = np.array([np.prod([_phi(bits[a][d], s[d]) for d in range(nd)]) for a in range(nloc)])
        dN = np.zeros((nloc, nd))
        for a in range(nloc):
            for d in range(nd):
                v = (2.0 / h[d]) * _dphi(bits[a][d])
                for d2 in range(nd):
                    if d2 != d:
                        v *= _phi(bits[a][d2], s[d2])
                dN[a, d] = v
        F += detJ * (np.outer(N, N) + (dN * np.array(dcoef)[None, :]) @ dN.T)
    return F


def filter_matrices(mesh: Mesh, rx: float, rt: float):
    """(K_f + M_f) assembled (CSR, SPD) and T_f (nodes x elements), A (elements x nodes, the mean)."""
    Fe = filter_element_matrix(mesh.sdim, mesh.dx, mesh.dt, rx, rt)
    conn = connectivity(mesh)
    nloc = conn.shape[1]
    rows = np.repeat(conn, nloc, axis=1).reshape(-1)
    cols = np.tile(conn, (1, nloc)).reshape(-1)
    F = sp.coo_matrix((np.tile(Fe.reshape(-1), mesh.n_elems), (rows, cols)),
                      shape=(mesh.n_nodes, mesh.n_nodes)).tocsr()
    vol = mesh.dx ** mesh.sdim * mesh.dt
    e = np.repeat(np.arange(mesh.n_elems), nloc)
    Tf = sp.coo_matrix((np.full(e.size, vol / nloc), (conn.reshape(-1), e)),
                       shape=(mesh.n_nodes, mesh.n_elems)).tocsr()
    A = sp.coo_matrix((np.full(e.size, 1.0 / nloc), (e, conn.reshape(-1))),
                      shape=(mesh.n_elems, mesh.n_nodes)).tocsr()
    return F, Tf, A


def projection(g, beta: float = 32.0, eta: float = 0.5):
    """Heaviside projection of PAPER.md:549-551 and its derivative."""
    g = np.asarray(g, dtype=np.float64)
    den = math.tanh(beta * eta) + math.tanh(beta * (1.0 - eta))
    gb = (math.tanh(beta * eta) + np.tanh(beta * (g - eta))) / den
    dg = beta * (1.0 - np.tanh(beta * (g - eta)) ** 2) / den
    return gb, dg


def pde_filter(mesh: Mesh, gamma, rx: float, rt: float, beta: float = 32.0, eta: float = 0.5):
    """Element design g -> (filtered nodal field, filtered element field g~_e, projected g_bar)."""
    F, Tf, A = filter_matrices(mesh, rx, rt)
    gn = spla.splu(F.tocsc()).solve(Tf @ np.asarray(gamma, dtype=np.float64).reshape(-1))
    ge = A @ gn
    gb, _ = projection(ge, beta, eta)
    return gn, ge, gb


def pde_filter_grad(mesh: Mesh, ge, dphi_dgb, rx: float, rt: float, beta: float = 32.0, eta: float = 0.5):
    """Chain rule: dphi/dg = T_f^T F^-1 A^T (dg_bar/dg~ .* dphi/dg_bar) (F symmetric)."""
    F, Tf, A = filter_matrices(mesh, rx, rt)
    _, dg = projection(ge, beta, eta)
    w = spla.splu(F.tocsc()).solve(A.T @ (dg * np.asarray(dphi_dgb, dtype=np.float64).reshape(-1)))
    return Tf.T @ w
