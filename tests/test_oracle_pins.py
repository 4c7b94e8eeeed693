"""Round-2 pins of the oracle (-m "not gpu"; VERDICT r01 'pin the oracle fully'):

* the rescaling k~ = k tau / L^2, Q~ = Q tau of simp() / source_vector() (sec. 2.1)
  against the system assembled in PHYSICAL coordinates (element integrals with the physical
  steps L/n, tau/nt, physical k and Q, source by the closed form int N_a dV = |e| / 2^(d+1));
* the sampled, purely local certification helpers (node_constraint, source_rows, row_apply,
  sensitivity_elements; R-21) against the global definitions on every node / element;
* the library's host-only hierarchy plan (st_plan) against oracle.algorithm1 on
  BASELINE configs 1-5 and the paper's printed hierarchies;
* the config-1 regression values, read from tests/golden/config1_regression.json (written by the
  committed scripts/gen_golden.py, which calls oracle/ only)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle as O
import st_inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CFG1_MATS = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)
CFG4_MATS = (0.1, 1.0, 1.0, 1e-4, 1.0, 3.0)


# ------------------------------------------------------------------ rescaling identity
def _physical_solution(sdim, n, nt, L, tau, mats, Q, T0, rho):
    """K_phys T = f_phys in physical coordinates (x in [0, L]^d, t in [0, tau]): per element
    A_e = C_e G(dx_p, dt_p) + k_e Kx(dx_p, dt_p) with the PHYSICAL conductivity (no rescaling) and
    the stabilisation k_ad = dt_p C / 2 inside G (element_matrices takes the steps as arguments);
    f_a = Q sum_e |e| / 2^(d+1) (uniform Q: the trilinear basis integrates to |e| / 2^(d+1))."""
    mesh = O.Mesh(sdim, n, nt)            # numbering / connectivity only
    dxp, dtp = L / n, tau / nt
    G, Kx = O.element_matrices(sdim, dxp, dtp)
    r = np.asarray(rho, dtype=np.float64).reshape(-1)
    if r.size == mesh.plane_elems:
        r = np.tile(r, nt)
    C = mats.C_ins + (mats.C_con - mats.C_ins) * r ** mats.p_c
    k = mats.k_ins + (mats.k_con - mats.k_ins) * r ** mats.p_k     # physical: no tau / L^2
    conn = O.connectivity(mesh)
    nloc = conn.shape[1]
    vals = C[:, None, None] * G[None] + k[:, None, None] * Kx[None]
    K = sp.coo_matrix((vals.reshape(-1), (np.repeat(conn, nloc, axis=1).reshape(-1), np.tile(conn, (1, nloc)).reshape(-1))),
                      shape=(mesh.n_nodes, mesh.n_nodes)).tocsr()
    f = np.zeros(mesh.n_nodes)
    np.add.at(f, conn.reshape(-1), Q * dxp ** sdim * dtp / nloc)
    cons, xD = O.dirichlet(mesh, O.BCs(T0=T0))
    Kbc, b = O.apply_dirichlet(K, f, cons, xD)
    return spla.splu(Kbc.tocsc()).solve(b)


@pytest.mark.parametrize("sdim,L,tau", [(2, 1.0, 2.0), (2, 2.0, 1.0), (2, 0.5, 3.0), (3, 2.0, 0.5)])
def test_rescaling_identity_pins_ktilde_and_qtilde(sdim, L, tau):
    """The rescaled oracle problem (k~ = k tau / L^2, Q~ = Q tau) has the same
    nodal temperatures as the physical problem: A_phys = L^d A*(k~), f_phys = L^d f*(Q~). A wrong
    exponent or a dropped factor in simp() or source_vector() breaks the equality (tau != 1 is what
    config 5 runs, R-7)."""
    n, nt = (6, 8) if sdim == 2 else (3, 4)
    mats = O.Materials(*CFG4_MATS)
    rho = I.rho_uniform((nt,) + (n,) * sdim, 3)
    Q, T0 = 1.7, 0.25
    Tp = _physical_solution(sdim, n, nt, L, tau, mats, Q, T0, rho)
    prob = O.Problem(O.Mesh(sdim, n, nt, L=L, tau=tau), mats, O.BCs(T0=T0), O.Source("uniform", Q))
    Ts = prob.forward(rho)
    assert np.linalg.norm(Ts - Tp) <= 1e-11 * np.linalg.norm(Tp)
    # and the identity is not vacuous: without the rescaling the solution differs
    prob1 = O.Problem(O.Mesh(sdim, n, nt), mats, O.BCs(T0=T0), O.Source("uniform", Q))
    assert np.linalg.norm(prob1.forward(rho) - Tp) > 1e-3 * np.linalg.norm(Tp)


# ------------------------------------------------------------------ sampled helpers
@pytest.mark.parametrize("sdim,n,nt,bcs", [(2, 8, 6, O.BCs(T0=0.3)), (2, 20, 4, O.BCs(T0=0.0, halfwidth=0.15)),
                                         (3, 6, 3, O.BCs(T0=0.7)), (2, 5, 3, O.BCs(T0=0.2, all_walls=True)),
                                         (3, 4, 2, O.BCs(all_walls=True)), (2, 6, 4, O.BCs(has_patch=False))])
def test_node_constraint_equals_dirichlet(sdim, n, nt, bcs):
    mesh = O.Mesh(sdim, n, nt)
    cons, xD = O.dirichlet(mesh, bcs)
    for node in range(mesh.n_nodes):
        c, v = O.node_constraint(mesh, bcs, node)
        assert c == bool(cons[node]) and (not c or v == xD[node]), node


@pytest.mark.parametrize("src", [O.Source("uniform", 1.3), O.Source("sin", 1.0, 1.0, 2 * np.pi), O.Source("ex1", 100.0),
                                 O.Source("ex2", 2.0, w=1.1, sigma=0.1, R=0.25)])
@pytest.mark.parametrize("sdim", [2, 3])
def test_source_rows_equal_source_vector(src, sdim):
    if src.kind == "ex2" and sdim == 3:
        pytest.skip("Example 2 is a 2D source (PAPER.md:309-320)")
    mesh = O.Mesh(sdim, 5 if sdim == 2 else 3, 6, tau=1.5)
    f = O.source_vector(mesh, src)
    rows = O.source_rows(mesh, src, np.arange(mesh.n_nodes))
    assert np.abs(rows - f).max() <= 1e-15 * max(1.0, np.abs(f).max())


def test_row_apply_accepts_a_node_mapping():
    """The full-size certification passes the GPU vector as a mapping of the stencil nodes only."""
    mesh = O.Mesh(2, 6, 5)
    prob = O.Problem(mesh, O.Materials(*CFG1_MATS), O.BCs(T0=0.2))
    rho = I.rho_uniform((5, 6, 6), 4)
    x = I.rand_vector(mesh.n_nodes, 2)
    rows = np.array([0, 7, 30, 100, mesh.n_nodes - 1])
    m = {i: x[i] for i in range(mesh.n_nodes)}
    assert np.array_equal(O.row_apply(prob, rho, m, rows), O.row_apply(prob, rho, x, rows))


# ------------------------------------------------------------------ st_plan vs Algorithm 1
def _plan_levels(sdim, n, nt, mats, tau=1.0, **opts):
    from paper_2508_09589_b200 import st
    p = st.plan(sdim, n, nt, mats=mats, tau=tau, **opts)
    return [(l["n"], l["nt"], l["kind"]) for l in p["levels"]]


@pytest.mark.parametrize("cfg", [
    (2, 16, 16, CFG1_MATS, 1.0), (2, 256, 256, CFG1_MATS, 1.0), (2, 1024, 1024, CFG1_MATS, 1.0),
    (3, 64, 128, CFG4_MATS, 1.0), (2, 512, 512, CFG1_MATS, 1.0), (2, 512, 1024, CFG1_MATS, 2.0),
    (2, 512, 2048, CFG1_MATS, 4.0), (2, 512, 4096, CFG1_MATS, 8.0)],
    ids=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5-G1", "cfg5-G2", "cfg5-G4", "cfg5-G8"])
def test_st_plan_equals_algorithm1_on_baseline_configs(cfg):
    """The library's host-side Algorithm 1 (csrc/api.cu build_hierarchy) gives the oracle's level
    list on every BASELINE config, stopping at <= coarse_max_nodes (R-19)."""
    sdim, n, nt, m, tau = cfg
    mats = O.Materials(*m)
    D = O.d_eff(mats.k_con, mats.k_ins, mats.C_con, mats.C_ins, tau=tau)
    ref = O.algorithm1(n, nt, D, sdim=sdim, max_nodes=400)
    got = _plan_levels(sdim, n, nt, m, tau=tau, coarse_max_nodes=400)
    assert got == [(a, b, c) for a, b, c in ref]


def test_st_plan_reproduces_the_paper_hierarchies():
    """With the paper's level counts N_l the plan equals every printed hierarchy
    (tests/golden/hierarchies.json: PAPER.md:628-643, 790-804, 995-1010). The coarsest levels there
    (up to 21^2 x 321 = 141,561 nodes) need the paper's GMRES coarsest solve (ST_COARSE_GMRES)."""
    from paper_2508_09589_b200 import st
    cases = json.load(open(os.path.join(GOLD, "hierarchies.json")))["cases"]
    for cs in cases:
        m = (cs["C_ins"], cs["C_con"], 1.0, cs["k_ins"], cs["k_con"], 3.0)
        got = _plan_levels(2, cs["n"], cs["nt"], m, tau=cs["tau"], max_levels=cs["n_levels"], coarse_max_nodes=8,
                           coarse_solver=st.ST_COARSE_GMRES)
        assert [[a, b] for a, b, _ in got] == cs["levels"], cs["name"]
    # the dense coarsest solve refuses them (more than 4096 stored nodes), with a clear error
    cs = cases[0]
    with pytest.raises(st.StError, match="ST_COARSE_GMRES"):
        _plan_levels(2, cs["n"], cs["nt"], (cs["C_ins"], cs["C_con"], 1.0, cs["k_ins"], cs["k_con"], 3.0), tau=cs["tau"],
                     max_levels=cs["n_levels"], coarse_max_nodes=8)


# ------------------------------------------------------------------ regression values
def test_config1_regression_values_from_committed_script():
    g = json.load(open(os.path.join(GOLD, "config1_regression.json")))
    mesh = O.Mesh(2, 16, 16)
    P = O.Problem(mesh, O.Materials(*CFG1_MATS))
    rho = I.rho_uniform((16, 16, 16), 0)
    T, lam = P.solve_both(rho)
    dJ = P.sensitivity(rho, T, lam)
    Kbc, _, _, _ = P.system(rho)
    x = np.random.default_rng(1).uniform(-1, 1, mesh.n_nodes)
    assert P.compliance(T) == pytest.approx(g["compliance_fT"], rel=1e-11)
    assert np.linalg.norm(T) == pytest.approx(g["norm_T"], rel=1e-11)
    assert T.max() == pytest.approx(g["max_T"], rel=1e-11)
    assert np.linalg.norm(lam) == pytest.approx(g["norm_lambda"], rel=1e-11)
    assert np.linalg.norm(dJ) == pytest.approx(g["norm_dJ"], rel=1e-9)
    assert dJ.sum() == pytest.approx(g["sum_dJ"], rel=1e-9)
    assert np.linalg.norm(Kbc @ x) == pytest.approx(g["norm_Kbc_x_seed1"], rel=1e-12)
