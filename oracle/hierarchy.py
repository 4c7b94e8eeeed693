"""ORACLE (test infrastructure only — see oracle/__init__.py).

Algorithm 1 of arxiv 2508.09589 (alg:coarstrat): the semi-coarsening
schedule of the space-time multigrid hierarchy.
"""
from __future__ import annotations

import math


def d_eff(k_con: float, k_ins: float, C_con: float, C_ins: float, tau: float = 1.0,
          L: float = 1.0) -> float:
    """D_eff = sqrt(k~_con k~_ins / (C_con C_ins)) (Algorithm 1 line 2) with the rescaled
    conductivities k~ = k tau / L^2."""
    kc = k_con * tau / L ** 2
    ki = k_ins * tau / L ** 2
    return math.sqrt(kc * ki / (C_con * C_ins))

def algorithm1(n: int, nt: int, D: float, n_levels: int | None = None,
               lambda_crit: float = 0.5, sdim: int = 2, max_nodes: int | None = None,
               full: bool = False):
    """Level list [(n_l, nt_l, kind)] with kind in {'fine', 'space', 'time', 'full'}.

    For l = 1..N_l-1: lambda_eff = D dt_{l-1} / dx_{l-1}^2 with dx = 1/n, dt = 1/nt in
    rescaled units; coarsen in time if lambda_eff < lambda_crit (strict, R-18),
    else in space. With n_levels given, an odd count in the chosen
    direction raises. With n_levels None, coarsening stops when the level has
    <= max_nodes nodes or the chosen direction cannot be halved (R-19).
    full=True coarsens space and time together (the 'full space-time coarsening'
    comparison)."""
    levels = [(n, nt, "fine")]
    cur_n, cur_nt = n, nt
    l = 1
    while True:
        if n_levels is not None and l >= n_levels:
            break
        if n_levels is None and max_nodes is not None:
            if (cur_n + 1) ** sdim * (cur_nt + 1) <= max_nodes:
                break
        lam = D * (1.0 / cur_nt) / (1.0 / cur_n) ** 2
        if full:
            kind = "full"
            ok = cur_n % 2 == 0 and cur_nt % 2 == 0 and cur_n >= 2 and cur_nt >= 2
        elif lam < lambda_crit:
            kind = "time"
            ok = cur_nt % 2 == 0 and cur_nt >= 2
        else:
            kind = "space"
            ok = cur_n % 2 == 0 and cur_n >= 2
        if not ok:
            if n_levels is not None:
                raise ValueError(f"level {l}: cannot coarsen in {kind} ({cur_n}x{cur_nt})")
            break
        if kind in ("space", "full"):
            cur_n //= 2
        if kind in ("time", "full"):
            cur_nt //= 2
        levels.append((cur_n, cur_nt, kind))
        l += 1
    return levels
