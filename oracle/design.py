"""ORACLE (test infrastructure only — see oracle/__init__.py).

The design loop of BASELINE config 5 as SURVEY.md 8(c) c-13 / DESIGN.md R-13 read it (the
BASELINE names "optimality criteria, volume fraction 0.4, density filter radius 2 elements" but
fixes no formula; this is NOT the paper's method, which uses a PDE filter, projection and MMA,
PAPER.md:531-559):

  density filter  rho~_i = sum_j w_ij rho_j / sum_j w_ij,  w_ij = max(0, r - |idx_i - idx_j|)
                  over the element grid (x1, x2[, x3], t) (space only for a time-constant design);
  chain rule      dphi/drho_j = sum_i w_ij (dphi/drho~_i) / W_i;
  OC              rho_new = clip(rho sqrt(max(0, -dphi/drho) / Lambda),
                             [max(rho_min, rho - move), min(1, rho + move)])
                  with Lambda by bisection on mean(rho_new) = volfrac (l1 = 0, l2 = 1e9, midpoint,
                  until (l2 - l1) / (l1 + l2) <= 1e-12, at most 200 halvings).

Plain loops over the neighbourhood offsets; no code shared with the CUDA path.
"""
from __future__ import annotations

import itertools

import numpy as np


def _weights(ndim: int, r: float):
    """(offset, weight) pairs of the hat filter over an ndim-dimensional element grid."""
    out = []
    for off in itertools.product((-1, 0, 1), repeat=ndim):
        w = max(0.0, r - float(np.sqrt(sum(o * o for o in off))))
        if w > 0.0:
            out.append((off, w))
    return out


def _shift(a, off):
    """b[i] = a[i + off] where i + off is inside the array, else NaN-marker via a mask."""
    res = np.zeros_like(a)
    mask = np.zeros(a.shape, dtype=bool)
    src = []
    dst = []
    for d, o in enumerate(off):
        n = a.shape[d]
        if o >= 0:
            src.append(slice(o, n))
            dst.append(slice(0, n - o))
        else:
            src.append(slice(0, n + o))
            dst.append(slice(-o, n))
    res[tuple(dst)] = a[tuple(src)]
    mask[tuple(dst)] = True
    return res, mask


def density_filter(rho, r: float = 2.0, transpose: bool = False):
    """F rho (or F^T g) on the element array `rho` (all axes filtered: [t][x2][x1] for a space-time
    design, [x2][x1] for a time-constant one)."""
    rho = np.asarray(rho, dtype=np.float64)
    W = np.zeros_like(rho)
    for off, w in _weights(rho.ndim, r):
        _, m = _shift(rho, off)
        W += w * m
    src = rho / W if transpose else rho
    acc = np.zeros_like(rho)
    for off, w in _weights(rho.ndim, r):
        v, m = _shift(src, off)
        acc += w * v * m
    return acc if transpose else acc / W


def oc_update(rho, dJ, volfrac: float = 0.4, move: float = 0.2, rho_min: float = 1e-3):
    """Optimality-criteria step; returns (rho_new, Lambda)."""
    rho = np.asarray(rho, dtype=np.float64)
    B = np.maximum(0.0, -np.asarray(dJ, dtype=np.float64))
    lo = np.maximum(rho_min, rho - move)
    hi = np.minimum(1.0, rho + move)

    def new(lam):
        return np.minimum(hi, np.maximum(lo, rho * np.sqrt(B / lam)))

    l1, l2 = 0.0, 1e9
    it = 0
    while it < 200 and (l2 - l1) / (l1 + l2) > 1e-12:
        lm = 0.5 * (l1 + l2)
        if new(lm).sum() / rho.size > volfrac:
            l1 = lm
        else:
            l2 = lm
        it += 1
    lam = 0.5 * (l1 + l2)
    return new(lam), lam


def design_loop(prob, rho0, iterations: int, volfrac: float = 0.4, r: float = 2.0, move: float = 0.2,
                rho_min: float = 1e-3):
    """Config-5 loop: filter -> forward -> compliance adjoint -> sensitivities -> F^T -> OC.
    Returns the designs after every iteration and the compliance history phi = f^T T."""
    rho = np.asarray(rho0, dtype=np.float64).copy()
    hist, designs = [], []
    for _ in range(iterations):
        rt = density_filter(rho, r)
        T, lam = prob.solve_both(rt)
        hist.append(prob.compliance(T))
        dJt = prob.sensitivity(rt, T, lam)
        dJ = density_filter(dJt, r, transpose=True)
        rho, _ = oc_update(rho, dJ, volfrac, move, rho_min)
        designs.append(rho.copy())
    return designs, hist
