"""Seeded synthetic input generators shared by the oracle-side tests and the CUDA-side
tests/bench (reading R-11).

This module holds NONE of the method's arithmetic: it only draws design densities and
test vectors. Both sides consume the same arrays, so the generator never affects parity.
"""
from __future__ import annotations

import numpy as np


def rho_uniform(shape, seed: int = 0, lo: float = 0.1, hi: float = 1.0) -> np.ndarray:
    """i.i.d. U[lo, hi] element densities (config 1: U[0.1, 1], BASELINE configs[0])."""
    return np.random.default_rng(seed).uniform(lo, hi, size=shape)


def _minmax(a: np.ndarray, lo: float, hi: float) -> np.ndarray:
    amin, amax = a.min(), a.max()
    if amax - amin <= 0:
        return np.full_like(a, 0.5 * (lo + hi))
    return lo + (hi - lo) * (a - amin) / (amax - amin)


def smooth_layer(spatial_shape, seed: int, t: int, sigma: float = 3.0, lo: float = 0.01,
                 hi: float = 1.0) -> np.ndarray:
    """Layer t of the per-layer smooth field: its own generator default_rng((seed, t)), so any
    slab of layers can be drawn without the others (time slabs)."""
    from scipy.ndimage import gaussian_filter
    g = gaussian_filter(np.random.default_rng((seed, t)).standard_normal(spatial_shape), sigma=sigma,
                        mode="reflect")
    return _minmax(g, lo, hi)


def rho_smooth(shape, seed: int = 0, sigma: float = 3.0, lo: float = 0.01, hi: float = 1.0,
               per_layer: bool = False, layers=None, threads: int = 16) -> np.ndarray:
    """Smooth random field: standard normal -> Gaussian filter (sigma = 3 elements, the
    'radius 3 elements' of BASELINE configs 2-4, reflect mode) -> min-max affine onto
    [lo, hi]. per_layer=True: shape = (nt, *spatial), an independent field per time
    layer (smooth_layer), each min-max scaled (config 3); layers = (a, b) draws layers
    [a, b) only (a rank's slab)."""
    from scipy.ndimage import gaussian_filter
    if per_layer:
        a, b = layers if layers is not None else (0, shape[0])
        out = np.empty((b - a,) + tuple(shape[1:]))

        def one(t):
            out[t - a] = smooth_layer(tuple(shape[1:]), seed, t, sigma, lo, hi)

        if b - a >= 64 and threads > 1:  # scipy.ndimage releases the GIL: draw layers in parallel
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(a, b)))
        else:
            for t in range(a, b):
                one(t)
        return out
    rng = np.random.default_rng(seed)
    g = gaussian_filter(rng.standard_normal(shape), sigma=sigma, mode="reflect")
    return _minmax(g, lo, hi)


def rand_vector(n: int, seed: int = 1, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Random test vector x ~ U[lo, hi] (operator parity, R-15)."""
    return np.random.default_rng(seed).uniform(lo, hi, size=n)


# BASELINE.json configs, as (sdim, n, nt, design) — design: 'uniform' | 'smooth_tc' |
# 'smooth_layers' | 'const'.
CONFIGS = {
    1: dict(sdim=2, n=16, nt=16, design="uniform", tau=1.0),
    2: dict(sdim=2, n=256, nt=256, design="smooth_tc", tau=1.0),
    3: dict(sdim=2, n=1024, nt=1024, design="smooth_layers", tau=1.0),
    4: dict(sdim=3, n=64, nt=128, design="smooth_tc", tau=1.0),
    5: dict(sdim=2, n=512, nt=512, design="const", tau=1.0),
}


def design_for(sdim: int, n: int, nt: int, design: str, seed: int = 0, layers=None) -> np.ndarray:
    """Element densities for a config-shaped grid (shape [nt][x..] or [x..]); layers = (a, b):
    only layers [a, b) of a per-layer design (a time slab)."""
    sp_shape = (n,) * sdim
    if design == "uniform":
        return rho_uniform((nt,) + sp_shape, seed=seed)
    if design == "smooth_tc":
        return rho_smooth(sp_shape, seed=seed)
    if design == "smooth_layers":
        return rho_smooth((nt,) + sp_shape, seed=seed, per_layer=True, layers=layers)
    if design == "const":
        return np.full((nt,) + sp_shape, 0.4)
    raise ValueError(design)
