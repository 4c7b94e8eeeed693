"""Pins of the oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage or closed form it pins. A plausible mistake in the oracle
(dropped term, wrong sign/index, transposed operand) fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import st_inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CFG1_MATS = O.Materials(C_ins=1.0, C_con=1.0, p_c=1.0, k_ins=1e-3, k_con=1.0, p_k=3.0)
CFG4_MATS = O.Materials(C_ins=0.1, C_con=1.0, p_c=1.0, k_ins=1e-4, k_con=1.0, p_k=3.0)


# ---------------------------------------------------------------- element matrices
def _1d(h):
    m = h / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])          # int phi_a phi_b
    s = 1.0 / h * np.array([[1.0, -1.0], [-1.0, 1.0]])        # int phi_a' phi_b'
    c = 0.5 * np.array([[-1.0, 1.0], [-1.0, 1.0]])            # int phi_a phi_b'
    return m, s, c


@pytest.mark.parametrize("sdim", [2, 3])
@pytest.mark.parametrize("dx,dt", [(1 / 16, 1 / 16), (0.25, 0.1), (1 / 64, 1 / 128)])
def test_element_matrix_equals_kronecker_closed_form(sdim, dx, dt):
    """Quadrature of the weak form equals the tensor-product closed form
    built by hand from 1D linear-element integrals: G = (c_t + dt/2 s_t) (x) M_x,
    Kx = m_t (x) sum_d (s on dim d, m elsewhere). Local index a = x1 + 2 x2 (+4 x3) + 2^sdim t
    => kron(t, ..., x2, x1)."""
    mx, sx, _ = _1d(dx)
    mt, st, ct = _1d(dt)
    Mx = mx
    for _ in range(sdim - 1):
        Mx = np.kron(Mx, mx)
    Kspace = np.zeros_like(Mx)
    for d in range(sdim):
        term = np.array([[1.0]])
        for e in reversed(range(sdim)):
            term = np.kron(term, sx if e == d else mx)
        Kspace += term
    G_ref = np.kron(ct + 0.5 * dt * st, Mx)
    K_ref = np.kron(mt, Kspace)
    G, Kx = O.element_matrices(sdim, dx, dt)
    assert np.max(np.abs(G - G_ref)) <= 1e-15 * max(1.0, np.abs(G_ref).max())
    assert np.max(np.abs(Kx - K_ref)) <= 1e-14 * np.abs(K_ref).max()
    # the stabilisation cancels the downwind half of the time convection: U = [[0,0],[-1,1]]
    assert np.allclose(ct + 0.5 * dt * st, [[0.0, 0.0], [-1.0, 1.0]], atol=1e-15)


@pytest.mark.parametrize("sdim", [2, 3])
def test_element_parts_identities(sdim):
    """Row sums vanish (constant field in the kernel); Gt + Gt^T = top-face mass
    minus bottom-face mass (integration by parts in t); Kx, Kt symmetric."""
    dx, dt = 0.2, 0.05
    Gt, Kt, Kx = O.element_parts(sdim, dx, dt)
    for A in (Gt, Kt, Kx):
        assert np.abs(A.sum(axis=1)).max() < 1e-14
    assert np.allclose(Kt, Kt.T) and np.allclose(Kx, Kx.T)
    nloc = 2 ** (sdim + 1)
    half = nloc // 2
    mx, _, _ = _1d(dx)
    Mface = mx
    for _ in range(sdim - 1):
        Mface = np.kron(Mface, mx)
    D = np.zeros((nloc, nloc))
    D[half:, half:] = Mface
    D[:half, :half] = -Mface
    assert np.max(np.abs(Gt + Gt.T - D)) < 1e-16


def test_time_peclet_number_is_one():
    """k_ad = C dt / 2 gives element Peclet number C dt / (2 k_ad) = 1."""
    gold = json.load(open(os.path.join(GOLD, "paper_counts.json")))["peclet_time"]["value"]
    dx, dt = 0.1, 0.03
    Gt, Kt, _ = O.element_parts(2, dx, dt)
    G, _ = O.element_matrices(2, dx, dt)
    mask = np.abs(Kt) > 1e-12
    k_ad_over_C = ((G - Gt)[mask] / Kt[mask])
    assert np.allclose(k_ad_over_C, dt / 2.0, rtol=1e-13)
    assert dt / (2.0 * k_ad_over_C.mean()) == pytest.approx(gold, rel=1e-12)


# ---------------------------------------------------------------- assembly
def test_assembly_matches_bruteforce_loop():
    """CSR assembly equals a plain triple loop over elements and local nodes (3x3x3 mesh,
    random coefficients) — checks connectivity and element numbering."""
    mesh = O.Mesh(2, 3, 3)
    rng = np.random.default_rng(5)
    C = rng.uniform(0.5, 2, mesh.n_elems)
    k = rng.uniform(0.03, 3, mesh.n_elems)
    K = O.assemble_K(mesh, C, k).toarray()
    G, Kx = O.element_matrices(2, mesh.dx, mesh.dt)
    nn = mesh.n + 1
    Kb = np.zeros_like(K)
    e = 0
    for t in range(mesh.nt):
        for y in range(mesh.n):
            for x in range(mesh.n):
                nodes = [(x + (a & 1)) + nn * ((y + ((a >> 1) & 1)) + nn * (t + ((a >> 2) & 1)))
                         for a in range(8)]
                for a in range(8):
                    for b in range(8):
                        Kb[nodes[a], nodes[b]] += C[e] * G[a, b] + k[e] * Kx[a, b]
                e += 1
    assert np.max(np.abs(K - Kb)) < 1e-15


def test_assembled_rowsum_zero_and_dims():
    mesh = O.Mesh(2, 4, 5)
    P = O.Problem(mesh, CFG1_MATS)
    K = P.K(I.rho_uniform((5, 4, 4), 3))
    assert K.shape == (mesh.n_nodes, mesh.n_nodes)
    assert np.abs(K @ np.ones(mesh.n_nodes)).max() < 1e-15
    # 27-point stencil: interior row has 27 nonzeros
    nn = 5
    row = 2 + nn * (2 + nn * 2)
    assert K[row].nnz == 27


def test_paper_dof_counts():
    gold = json.load(open(os.path.join(GOLD, "paper_counts.json")))
    for c in gold["dofs"]:
        m = O.Mesh(2, c["n"], c["nt"])
        assert m.n_nodes == c["N_n"], c["cite"]
        if "N_e" in c:
            assert m.n_elems == c["N_e"], c["cite"]
    for c in gold["spatial_dofs"]:
        assert (c["n"] + 1) ** 2 == c["N"]


def test_tau_diff_values():
    gold = json.load(open(os.path.join(GOLD, "paper_counts.json")))["tau_diff"]
    for c in gold:
        assert round(O.diffusion_timescale(c["C"], c["L"], c["k"]), 2) == pytest.approx(c["value"])


@pytest.mark.parametrize("n,count", [(16, 1), (256, 25), (512, 51), (1024, 103)])
def test_patch_nodes_per_plane(n, count):
    """Sink of width L/10 centred on the face: node counts per plane."""
    mesh = O.Mesh(2, n, 2)
    cons, _ = O.dirichlet(mesh, O.BCs())
    plane1 = cons.reshape(3, n + 1, n + 1)[1]
    assert plane1.sum() == count and plane1[:, 0].sum() == count
    assert cons.reshape(3, -1)[0].all()


def test_patch_nodes_3d():
    mesh = O.Mesh(3, 64, 2)
    cons, _ = O.dirichlet(mesh, O.BCs())
    assert cons.reshape(3, -1)[1].sum() == 49


def test_source_sums():
    """Partition of unity: sum f = int Q~ over the space-time domain."""
    m = O.Mesh(2, 8, 16)
    f = O.source_vector(m, O.Source("uniform", 1.0))
    assert f.sum() == pytest.approx(1.0, abs=1e-14)
    f = O.source_vector(m, O.Source("sin", 1.0, 1.0, 2 * np.pi))
    assert f.sum() == pytest.approx(1.0, abs=1e-10)   # int_0^1 (1 + sin 2 pi t) dt = 1
    m5 = O.Mesh(2, 4, 8, tau=2.0)
    assert O.source_vector(m5, O.Source("uniform", 1.0)).sum() == pytest.approx(2.0)  # Q~ = Q tau
    m3 = O.Mesh(3, 3, 4)
    assert O.source_vector(m3, O.Source()).sum() == pytest.approx(1.0, abs=1e-14)
    f1 = O.source_vector(O.Mesh(2, 2, 64), O.Source("ex1", 100.0))
    t = np.linspace(0, 1, 200001)
    ex = np.trapezoid(50.0 * (1 - t) * (1 + np.cos(50 * t)), t)
    assert f1.sum() == pytest.approx(ex, rel=2e-4)


# ---------------------------------------------------------------- solves: closed forms
@pytest.mark.parametrize("mats,sdim", [(CFG1_MATS, 2), (CFG4_MATS, 2), (CFG1_MATS, 3)])
def test_uniform_stays_uniform(mats, sdim):
    """Q = 0, insulated walls, T0 = c, uniform C: T == c for ANY k(rho) (north_star pin 1)."""
    n, nt = (6, 8) if sdim == 2 else (3, 4)
    mesh = O.Mesh(sdim, n, nt)
    rng = np.random.default_rng(2)
    if mats.C_con == mats.C_ins:
        rho = rng.uniform(0.05, 1, (nt,) + (n,) * sdim)
    else:
        # capacity must be uniform: vary k only through a material with C independent of rho
        mats = O.Materials(0.55, 0.55, 1.0, 1e-4, 1.0, 3.0)
        rho = rng.uniform(0.05, 1, (nt,) + (n,) * sdim)
    P = O.Problem(mesh, mats, O.BCs(T0=0.7, has_patch=False), O.Source("uniform", 0.0))
    T = P.forward(rho)
    assert np.abs(T - 0.7).max() < 1e-13


def test_zero_source_zero_ic_gives_zero():
    mesh = O.Mesh(2, 6, 6)
    P = O.Problem(mesh, CFG1_MATS, O.BCs(T0=0.0), O.Source("uniform", 0.0))
    assert np.abs(P.forward(I.rho_uniform((6, 6, 6), 1))).max() == 0.0


@pytest.mark.parametrize("mats", [CFG1_MATS, CFG4_MATS])
def test_uniform_closed_form_with_source(mats):
    """Uniform C and Q, no patch, T0: T_n = T0 + n Q dt / C for n < nt and
    T_nt = T0 + (nt - 1/2) Q dt / C, independent of k (derivation in DESIGN.md, F5)."""
    n, nt, Q, T0 = 6, 10, 1.7, 0.3
    mesh = O.Mesh(2, n, nt)
    rho0 = 0.37
    rho = np.full((n, n), rho0)   # time-constant uniform => uniform C, uniform k
    P = O.Problem(mesh, mats, O.BCs(T0=T0, has_patch=False), O.Source("uniform", Q))
    T = P.forward(rho).reshape(nt + 1, -1)
    C = mats.C_ins + (mats.C_con - mats.C_ins) * rho0 ** mats.p_c
    dt = 1.0 / nt
    for p in range(nt):
        assert np.abs(T[p] - (T0 + p * Q * dt / C)).max() < 1e-13
    assert np.abs(T[nt] - (T0 + (nt - 0.5) * Q * dt / C)).max() < 1e-13


def test_uniform_closed_form_time_varying_source():
    """Uniform space, Q(t) = 1 + sin(2 pi t): at interior spatial nodes
    T_p - T_{p-1} = f_p / (C dx^2) (mass row sum = C dx^2, stiffness row sum = 0)."""
    n, nt = 4, 12
    mesh = O.Mesh(2, n, nt)
    P = O.Problem(mesh, CFG1_MATS, O.BCs(T0=0.0, has_patch=False),
                  O.Source("sin", 1.0, 1.0, 2 * np.pi))
    T = P.forward(np.full((n, n), 0.5)).reshape(nt + 1, n + 1, n + 1)
    f = P.f().reshape(nt + 1, n + 1, n + 1)
    for p in range(1, nt + 1):
        assert T[p, 2, 2] - T[p - 1, 2, 2] == pytest.approx(f[p, 2, 2] / (1.0 * mesh.dx ** 2), abs=1e-13)


def test_uniform_adjoint_and_sensitivity_closed_forms():
    """Uniform case, g = f: lambda_0 = 0, lambda_p = (nt - p + 1/2) Q dt / C; the sensitivity
    reduces to -C' dx^d lambda_{tau+1} (T_{tau+1} - T_tau) (spatial stiffness terms vanish)."""
    n, nt, Q = 5, 8, 1.0
    mesh = O.Mesh(2, n, nt)
    rho0 = 0.37
    rho = np.full((nt, n, n), rho0)
    P = O.Problem(mesh, CFG4_MATS, O.BCs(T0=0.0, has_patch=False), O.Source("uniform", Q))
    T, lam = P.solve_both(rho)
    C = 0.1 + 0.9 * rho0
    dt = 1.0 / nt
    lp = lam.reshape(nt + 1, -1)
    Tp = T.reshape(nt + 1, -1)
    assert np.abs(lp[0]).max() == 0.0
    for p in range(1, nt + 1):
        assert np.abs(lp[p] - (nt - p + 0.5) * Q * dt / C).max() < 1e-13
    dJ = P.sensitivity(rho, T, lam)
    dC = 0.9
    for tau in range(nt):
        ref = -dC * mesh.dx ** 2 * lp[tau + 1, 0] * (Tp[tau + 1, 0] - Tp[tau, 0])
        assert np.abs(dJ[tau] - ref).max() < 1e-15


def test_direct_solve_matches_dense():
    mesh = O.Mesh(2, 4, 4)
    P = O.Problem(mesh, CFG1_MATS)
    rho = I.rho_uniform((4, 4, 4), 7)
    Kbc, b, cons, _ = P.system(rho)
    T_dense = np.linalg.solve(Kbc.toarray(), b)
    assert np.abs(P.forward(rho) - T_dense).max() < 1e-13
    g = P.compliance_rhs()
    lam_dense = np.linalg.solve(Kbc.toarray().T, g)
    assert np.abs(P.adjoint(rho, g) - lam_dense).max() < 1e-13


# ---------------------------------------------------------------- convergence to time stepping
def test_converges_to_backward_euler_first_order():
    """The stabilised space-time solution converges to fine-step implicit time stepping at
    first order in dt (north_star pin 2): error ratio ~2 per halving."""
    n = 8
    rng = np.random.default_rng(11)
    rho_sp = rng.uniform(0.1, 1.0, (n, n))
    C_e, k_e, _, _ = O.simp(rho_sp.reshape(-1), CFG1_MATS, O.Mesh(2, n, 2))
    src = O.Source("sin", 1.0, 1.0, 2 * np.pi)
    cons_full, _ = O.dirichlet(O.Mesh(2, n, 2), O.BCs())
    cons_plane = cons_full.reshape(3, -1)[1]
    nref = 4096
    ref = O.backward_euler(n, 2, C_e, k_e, lambda t: 1.0 + np.sin(2 * np.pi * t), nref, 0.0, cons_plane)
    errs = []
    for nt in (8, 16, 32, 64):
        mesh = O.Mesh(2, n, nt)
        T = O.Problem(mesh, CFG1_MATS, O.BCs(), src).forward(rho_sp).reshape(nt + 1, -1)
        R = np.stack([ref[p * (nref // nt)] for p in range(nt + 1)])
        errs.append(np.linalg.norm(T - R) / np.linalg.norm(R))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(1.8 < r < 2.4 for r in ratios), (errs, ratios)


# ---------------------------------------------------------------- sensitivities vs FD
def _fd_check(P, rho, idx_list, h=1e-6):
    T, lam = P.solve_both(rho)
    dJ = P.sensitivity(rho, T, lam)
    for idx in idx_list:
        rp = rho.copy(); rp[idx] += h
        rm = rho.copy(); rm[idx] -= h
        fd = (P.compliance(P.forward(rp)) - P.compliance(P.forward(rm))) / (2 * h)
        # FD round-off ~ eps * phi / h ~ 1e-10 absolute
        assert dJ[idx] == pytest.approx(fd, rel=2e-6, abs=2e-9), idx


@pytest.mark.parametrize("T0", [0.0, 0.7])
def test_sensitivity_vs_central_fd_spacetime(T0):
    """dphi/drho_e = -lambda^T dK/drho_e T equals central finite differences of phi = f^T T
    (north_star pin 3), incl. the k_ad(C(rho)) term and non-homogeneous T0."""
    mesh = O.Mesh(2, 4, 6)
    P = O.Problem(mesh, CFG4_MATS, O.BCs(T0=T0), O.Source("sin", 1.0, 1.0, 2 * np.pi))
    rho = I.rho_uniform((6, 4, 4), 4)
    rng = np.random.default_rng(0)
    idx = [tuple(rng.integers(0, s) for s in rho.shape) for _ in range(8)]
    _fd_check(P, rho, idx)


def test_sensitivity_vs_central_fd_time_constant():
    mesh = O.Mesh(2, 4, 6)
    P = O.Problem(mesh, CFG4_MATS, O.BCs(), O.Source())
    rho = I.rho_uniform((4, 4), 9)
    _fd_check(P, rho, [(0, 0), (1, 2), (3, 3), (2, 0)])


def test_sensitivity_vs_central_fd_3d():
    mesh = O.Mesh(3, 2, 4)
    P = O.Problem(mesh, CFG4_MATS, O.BCs(T0=0.2), O.Source())
    rho = I.rho_uniform((4, 2, 2, 2), 6)
    _fd_check(P, rho, [(0, 0, 0, 0), (1, 1, 0, 1), (3, 1, 1, 1), (2, 0, 1, 0)])


def test_pnorm_gradient_vs_fd():
    """p-norm objective gradient vs central FD in T."""
    mesh = O.Mesh(2, 3, 3)
    T = np.random.default_rng(3).uniform(0.2, 1.0, mesh.n_nodes)
    phi, g = O.pnorm_objective(mesh, T, P=20.0)
    for i in (0, 7, 31, 60):
        Tp = T.copy(); Tp[i] += 1e-6
        Tm = T.copy(); Tm[i] -= 1e-6
        fd = (O.pnorm_objective(mesh, Tp)[0] - O.pnorm_objective(mesh, Tm)[0]) / 2e-6
        assert g[i] == pytest.approx(fd, rel=1e-6, abs=1e-12)
    # uniform T_avg = c over N_e elements => phi = c N_e^(1/P) (closed form of the p-norm)
    phi_u, _ = O.pnorm_objective(mesh, np.full(mesh.n_nodes, 0.5), P=20.0)
    assert phi_u == pytest.approx(0.5 * mesh.n_elems ** (1 / 20.0), rel=1e-13)


# ---------------------------------------------------------------- Algorithm 1
def test_algorithm1_reproduces_paper_tables():
    gold = json.load(open(os.path.join(GOLD, "hierarchies.json")))
    for c in gold["cases"]:
        D = O.d_eff(c["k_con"], c["k_ins"], c["C_con"], c["C_ins"], c["tau"])
        lv = O.algorithm1(c["n"], c["nt"], D, n_levels=c["n_levels"])
        assert [[a, b] for a, b, _ in lv] == c["levels"], c["cite"]


def test_algorithm1_d_eff_values():
    assert O.d_eff(3.0, 0.03, 1.0, 0.5) == pytest.approx(0.424264, rel=1e-6)
    assert O.d_eff(1.0, 1e-3, 1.0, 1.0) == pytest.approx(np.sqrt(1e-3))


def test_algorithm1_odd_raises_and_stop_rule():
    with pytest.raises(ValueError):
        O.algorithm1(6, 6, 10.0, n_levels=4)   # space: 6 -> 3 -> odd
    lv = O.algorithm1(256, 256, np.sqrt(1e-3), max_nodes=25000)
    assert (lv[-1][0] + 1) ** 2 * (lv[-1][1] + 1) <= 25000
    assert [k for *_, k in lv][:4] == ["fine", "space", "space", "space"]


@pytest.mark.parametrize("sdim,n,nt,tc", [(2, 5, 6, False), (3, 3, 4, True), (2, 6, 4, True)])
def test_sampled_rows_and_elements_equal_assembled(sdim, n, nt, tc):
    """row_apply / sensitivity_elements (used to certify full-size GPU results, R-21)
    equal the assembled K_bc, K_bc^T and the vectorised sensitivities on every row / element."""
    rng = np.random.default_rng(3)
    mesh = O.Mesh(sdim, n, nt)
    prob = O.Problem(mesh, O.Materials(0.1, 1.0, 1.0, 1e-4, 1.0, 3.0), O.BCs(T0=0.4), O.Source("sin", 1.0, 1.0, 6.0))
    rho = rng.uniform(0.1, 1.0, (n,) * sdim if tc else (nt,) + (n,) * sdim)
    Kbc, _, _, _ = prob.system(rho)
    x = rng.uniform(-1, 1, mesh.n_nodes)
    allrows = np.arange(mesh.n_nodes)
    assert np.allclose(O.row_apply(prob, rho, x, allrows), Kbc @ x, rtol=0, atol=1e-14)
    assert np.allclose(O.row_apply(prob, rho, x, allrows, transpose=True), Kbc.T @ x, rtol=0, atol=1e-14)
    T, lam = prob.solve_both(rho)
    dJ = prob.sensitivity(rho, T, lam)
    # space-time elements; a time-constant design sums them through time
    per = O.sensitivity_elements(prob, np.broadcast_to(rho, (nt,) + (n,) * sdim).copy() if tc else rho, T, lam,
                                 np.arange(mesh.n_elems))
    ref = per.reshape(nt, -1).sum(axis=0).reshape(dJ.shape) if tc else per.reshape(dJ.shape)
    assert np.allclose(ref, dJ, rtol=1e-12, atol=1e-15)
