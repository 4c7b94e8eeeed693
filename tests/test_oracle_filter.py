"""Pins of the oracle's PDE filter, Heaviside projection and chain rule (oracle/pdefilter.py;
PAPER.md:531-554), -m "not gpu": closed-form element matrices, exact reproduction of a constant
design (natural boundaries), projection closed values, and the chain rule against central finite
differences."""
import numpy as np
import pytest

import oracle as O


def _m1(h):
    return h / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])


def _k1(h):
    return 1.0 / h * np.array([[1.0, -1.0], [-1.0, 1.0]])


def _kron(mats):
    """Kronecker product in the element's local node order a = b0 + 2 b1 + ... (x1 fastest)."""
    out = np.array([[1.0]])
    for m in mats:
        out = np.kron(m, out)
    return out


@pytest.mark.parametrize("sdim", [2, 3])
def test_filter_element_matrix_closed_form(sdim):
    """F_e = M_t (x) M_s + rx^2/12 M_t (x) K_s + rt^2/12 K_t (x) M_s from the 1D factors
    m = h/6 [[2,1],[1,2]], k = 1/h [[1,-1],[-1,1]] (tensor-product Q1)."""
    dx, dt, rx, rt = 0.125, 0.0625, 0.3, 0.15
    F = O.filter_element_matrix(sdim, dx, dt, rx, rt)
    ms = [_m1(dx)] * sdim
    M = _kron(ms + [_m1(dt)])
    Ks = sum(_kron([(_k1(dx) if e == d else _m1(dx)) for e in range(sdim)] + [_m1(dt)]) for d in range(sdim))
    Kt = _kron(ms + [_k1(dt)])
    ref = M + rx * rx / 12.0 * Ks + rt * rt / 12.0 * Kt
    assert np.abs(F - ref).max() <= 1e-15 * np.abs(ref).max()
    assert np.allclose(F, F.T)


@pytest.mark.parametrize("sdim,n,nt", [(2, 6, 5), (3, 3, 4)])
def test_constant_design_is_reproduced(sdim, n, nt):
    """Natural boundaries: the constant function solves -div(d grad g~) + g~ = c exactly, so a
    constant design is returned unchanged by the filter (and its element mean)."""
    mesh = O.Mesh(sdim, n, nt)
    g = np.full(mesh.n_elems, 0.37)
    gn, ge, gb = O.pde_filter(mesh, g, 2.4 / n, 2.4 / nt)
    assert np.abs(gn - 0.37).max() <= 1e-13 and np.abs(ge - 0.37).max() <= 1e-13


def test_projection_closed_values():
    gb, dg = O.projection(np.array([0.0, 0.5, 1.0]), 32.0, 0.5)
    assert gb[0] == pytest.approx(0.0, abs=1e-15) and gb[1] == pytest.approx(0.5, abs=1e-15)
    assert gb[2] == pytest.approx(1.0, abs=1e-15)
    x = np.linspace(0.05, 0.95, 7)
    h = 1e-6
    fd = (O.projection(x + h)[0] - O.projection(x - h)[0]) / (2 * h)
    assert np.allclose(O.projection(x)[1], fd, rtol=1e-7)


def test_filter_smooths_a_checkerboard():
    mesh = O.Mesh(2, 8, 8)
    e = np.arange(mesh.n_elems)
    g = ((e % 8 + (e // 8) % 8 + e // 64) % 2).astype(float)
    _, ge, _ = O.pde_filter(mesh, g, 2.4 / 8, 2.4 / 8)
    assert np.std(ge) < 0.25 * np.std(g)
    assert ge.mean() == pytest.approx(g.mean(), rel=1e-2)


@pytest.mark.parametrize("sdim,n,nt", [(2, 5, 4), (3, 3, 3)])
def test_chain_rule_matches_central_fd(sdim, n, nt):
    """phi(g) = sum_e w_e g_bar_e(g): the chain rule equals central differences."""
    mesh = O.Mesh(sdim, n, nt)
    rng = np.random.default_rng(2)
    g = rng.uniform(0.3, 0.7, mesh.n_elems)
    w = rng.uniform(-1, 1, mesh.n_elems)
    rx, rt, beta = 2.4 / n, 2.4 / nt, 8.0

    def phi(gg):
        return float(w @ O.pde_filter(mesh, gg, rx, rt, beta)[2])
    _, ge, _ = O.pde_filter(mesh, g, rx, rt, beta)
    grad = O.pde_filter_grad(mesh, ge, w, rx, rt, beta)
    h = 1e-6
    for j in rng.choice(mesh.n_elems, 6, replace=False):
        gp, gm = g.copy(), g.copy()
        gp[j] += h
        gm[j] -= h
        fd = (phi(gp) - phi(gm)) / (2 * h)
        assert grad[j] == pytest.approx(fd, rel=1e-6, abs=1e-12)
