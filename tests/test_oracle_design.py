"""Pins of the oracle's config-5 design update (oracle/design.py; R-13): brute force,
invariants and closed forms. CPU only."""
import itertools

import numpy as np
import pytest

import oracle as O


def _brute_filter(a, r):
    out = np.zeros_like(a)
    idx = list(itertools.product(*[range(s) for s in a.shape]))
    for i in idx:
        num = den = 0.0
        for j in idx:
            w = max(0.0, r - np.sqrt(sum((p - q) ** 2 for p, q in zip(i, j))))
            num += w * a[j]
            den += w
        out[i] = num / den
    return out


@pytest.mark.parametrize("shape", [(3, 4, 5), (4, 4), (2, 3, 3, 3)])
def test_filter_equals_brute_force(shape):
    a = np.random.default_rng(1).uniform(0, 1, shape)
    assert np.allclose(O.density_filter(a, 2.0), _brute_filter(a, 2.0), rtol=1e-14, atol=1e-15)


def test_filter_invariants():
    rng = np.random.default_rng(2)
    a, b = rng.uniform(-1, 1, (5, 6, 7)), rng.uniform(-1, 1, (5, 6, 7))
    assert np.allclose(O.density_filter(np.full((5, 6, 7), 0.37)), 0.37, rtol=1e-15)   # constants kept
    lhs = np.sum(O.density_filter(a) * b)
    rhs = np.sum(a * O.density_filter(b, transpose=True))
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)                                            # F^T is the adjoint


def test_oc_volume_and_move_limits():
    rng = np.random.default_rng(3)
    rho = rng.uniform(0.2, 0.8, (4, 6, 6))
    dJ = -rng.uniform(1e-6, 1e-3, rho.shape)
    new, lam = O.oc_update(rho, dJ, volfrac=0.4, move=0.2)
    assert abs(new.mean() - 0.4) <= 1e-9
    assert np.all(new <= np.minimum(1.0, rho + 0.2) + 1e-15) and np.all(new >= np.maximum(1e-3, rho - 0.2) - 1e-15)


def test_oc_closed_form_uniform_sensitivity():
    """dJ = -B uniform, no active limit: rho_new = rho sqrt(B / Lambda) with mean volfrac =>
    Lambda = B (mean(rho) / volfrac)^2."""
    rho = np.full((3, 5, 5), 0.42)
    rho[0, 0, 0] = 0.40
    B = 2.5e-4
    new, lam = O.oc_update(rho, np.full(rho.shape, -B), volfrac=0.41, move=0.2)
    assert abs(lam - B * (rho.mean() / 0.41) ** 2) <= 1e-9 * lam
    assert np.allclose(new, rho * np.sqrt(B / lam), rtol=1e-12)
