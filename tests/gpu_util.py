"""Shared helpers of the -m gpu parity tests: build matching oracle / CUDA problems from
one description. Holds no method arithmetic."""
import numpy as np

import oracle as O

CFG1_MATS = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)       # k = 1e-3 + rho^3 (1 - 1e-3), c = 1
CFG4_MATS = (0.1, 1.0, 1.0, 1e-4, 1.0, 3.0)       # k_min = 1e-4, c = 0.1 + 0.9 rho


def make_pair(sdim, n, nt, mats=CFG1_MATS, T0=0.0, has_patch=True, source=("uniform", 1.0, 0.0, 0.0),
              tau=1.0, time_constant=False, all_walls=False, **opts):
    """source: (kind, Q0, a, w[, sigma, R]) — the same tuple drives both sides."""
    import paper_2508_09589_b200 as S
    solver = S.Solver(sdim, n, nt, mats=mats, T0=T0, has_patch=has_patch, source=source, tau=tau,
                      time_constant=time_constant, all_walls=all_walls, **opts)
    src = O.Source(*source)
    prob = O.Problem(O.Mesh(sdim, n, nt, tau=tau), O.Materials(*mats),
                     O.BCs(T0=T0, has_patch=has_patch, all_walls=all_walls), src)
    return solver, prob


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
