"""GPU parity of the persistent-kernel SCHEDULES the full-size runs use, and of
the round-2 solver options, against the oracle on oracle-scale grids.

At BASELINE sizes the persistent stencil kernels walk long (tile, plane) runs per CTA: tv2d switches
to sliced 16 / 32-plane time chunks once a CTA has >= 256 items (512^2 x 512 and config 3), and tc3d
gives each CTA ~650 items at config 4. The options chunk_planes and max_ctas (st_options_t, read per
launch) force those schedules on grids the oracle factorises in seconds: a cap of a few CTAs makes
every CTA sweep many tiles and planes (multi-plane runs, segment switches inside and across chunks,
cross-segment TMA prefetch), and a forced chunk length cuts time into slices (ragged last chunk
included). Every case compares K x and K^T x (with and without elimination) at <= 1e-12 and a full
solve (all modes of all levels) at <= 1e-8 (north_star tolerances, R-15)."""
import numpy as np
import pytest

import oracle as O
import paper_2508_09589_b200 as S
import st_inputs as I
from gpu_util import CFG1_MATS, CFG4_MATS, make_pair, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

DEV = torch.device("cuda:0")


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=DEV)


def host(t):
    return t.detach().cpu().numpy()


def _design(sdim, n, nt, tc, seed):
    return I.rho_smooth((n,) * sdim, seed=seed) if tc else I.rho_uniform((nt,) + (n,) * sdim, seed)


# (name, sdim, n, nt, time_constant, mats): tv2d = space-time design with uniform capacity (fine level
# from the k~ table, SRC 0; per-layer stored-stencil levels, SRC 1); tc2d / tc3d = time-constant
SCHED_CASES = [
    ("tv2d", 2, 48, 40, False, CFG1_MATS),
    ("tv2d-ragged", 2, 40, 36, False, CFG1_MATS),
    ("tc2d", 2, 48, 40, True, CFG1_MATS),
    ("tc3d", 3, 10, 12, True, CFG4_MATS),
    ("tc3d-ragged", 3, 10, 10, True, CFG1_MATS),
]
SCHEDULES = [(0, 1), (0, 3), (16, 0), (16, 2), (32, 5), (5, 3), (-1, 2)]  # (chunk_planes, max_ctas)


_ORACLE = {}


def _oracle_case(case):
    """Assembled operators and direct solutions of a case (computed once per case)."""
    if case[0] not in _ORACLE:
        name, sdim, n, nt, tc, mats = case
        prob = O.Problem(O.Mesh(sdim, n, nt), O.Materials(*mats), O.BCs(T0=0.2), O.Source())
        rho = _design(sdim, n, nt, tc, 3)
        K = prob.K(rho)
        Kbc, _, _, _ = prob.system(rho)
        T_ref, lam_ref = prob.solve_both(rho)
        _ORACLE[case[0]] = (prob, rho, K, Kbc, T_ref, lam_ref)
    return _ORACLE[case[0]]


SOLVE_SCHEDULES = {(0, 1), (16, 2), (32, 5), (5, 3)}


@pytest.mark.parametrize("sched", SCHEDULES, ids=lambda s: f"chunk{s[0]}-ctas{s[1]}")
@pytest.mark.parametrize("case", SCHED_CASES, ids=lambda c: c[0])
def test_forced_schedule_operator_and_solve_parity(case, sched):
    name, sdim, n, nt, tc, mats = case
    chunk, ctas = sched
    prob, rho, K, Kbc, T_ref, lam_ref = _oracle_case(case)
    solver, _ = make_pair(sdim, n, nt, mats=mats, T0=0.2, time_constant=tc, rtol=1e-11, maxit=600,
                          chunk_planes=chunk, max_ctas=ctas, coarse_max_nodes=64)
    x = I.rand_vector(prob.mesh.n_nodes, 17)
    xd, yd = dev(x), torch.empty(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    for trans in (False, True):
        for bc in (False, True):
            A = Kbc if bc else K
            ref = (A.T if trans else A) @ x
            solver.apply(dev(rho), xd, yd, transpose=trans, bc=bc)
            assert rel(host(yd), ref) <= 1e-12, (name, sched, trans, bc, rel(host(yd), ref))
    if sched in SOLVE_SCHEDULES:  # every mode of every level under the forced schedule
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(dev(rho), T)
        assert solver.stats()["converged"] == 1
        assert rel(host(T), T_ref) <= 1e-8
        lam = torch.zeros_like(T)
        solver.adjoint(dev(rho), None, lam)
        assert rel(host(lam), lam_ref) <= 1e-8
    solver.close()


@pytest.mark.parametrize("sched", [(0, 0), (16, 3), (32, 2)], ids=lambda s: f"chunk{s[0]}-ctas{s[1]}")
def test_forced_schedule_level_operators_equal_default(sched):
    """Every coarse level operator (stored-stencil SRC 1 tv2d levels, B4 levels below a time
    coarsening) under a forced schedule equals the default schedule's, forward and transposed."""
    n, nt = 64, 48
    rho = I.rho_uniform((nt, n, n), 5)
    ref_solver, _ = make_pair(2, n, nt, mats=CFG1_MATS, coarse_max_nodes=64)
    solver, _ = make_pair(2, n, nt, mats=CFG1_MATS, coarse_max_nodes=64, chunk_planes=sched[0], max_ctas=sched[1])
    h = solver.hierarchy()
    assert len(h) >= 4
    for l, lv in enumerate(h[:-1]):
        x = dev(I.rand_vector(lv["nodes"], 30 + l))
        for trans in (False, True):
            y0 = torch.empty_like(x)
            y1 = torch.empty_like(x)
            ref_solver.level_apply(dev(rho), l, x, y0, transpose=trans)
            solver.level_apply(dev(rho), l, x, y1, transpose=trans)
            assert rel(host(y1), host(y0)) <= 1e-13, (l, lv["kind"], trans)
    solver.close()
    ref_solver.close()


# ------------------------------------------------------------------ solver options (ABI 3)
@pytest.mark.parametrize("sdim,n,nt,tc,mats", [(2, 16, 16, False, CFG1_MATS), (2, 32, 32, True, CFG1_MATS),
                                               (3, 6, 12, True, CFG4_MATS), (2, 24, 20, False, CFG4_MATS)])
@pytest.mark.parametrize("restart", [3, 16])
def test_right_preconditioned_gmres_matches_oracle(sdim, n, nt, tc, mats, restart):
    """options krylov = ST_KRYLOV_GMRES (no Z vectors: x += M (V y) per restart; the memory plan of
    config 3 on one GPU) converges to the oracle's T and lambda; restart 3 forces
    several restart cycles."""
    solver, prob = make_pair(sdim, n, nt, mats=mats, time_constant=tc, rtol=1e-10, maxit=800,
                             krylov=S.st.ST_KRYLOV_GMRES, restart=restart)
    rho = _design(sdim, n, nt, tc, 1)
    T_ref, lam_ref = prob.solve_both(rho)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(rho), T)
    st = solver.stats()
    assert st["converged"] == 1 and st["vcycles"] == st["iterations"] + st["restarts"]
    assert rel(host(T), T_ref) <= 1e-8
    lam = torch.zeros_like(T)
    solver.adjoint(dev(rho), None, lam)  # null dJdT: the compliance RHS m_f f (R-8)
    assert rel(host(lam), lam_ref) <= 1e-8
    solver.close()


def test_gmres_and_fgmres_take_the_same_iterations():
    """With the fixed linear Jacobi V-cycle, GMRES(m) and FGMRES(m) build the same Krylov space:
    the same iteration counts and (to rounding) the same solution."""
    n, nt = 32, 32
    rho = dev(I.rho_smooth((n, n), seed=2))
    out = {}
    for k in (S.st.ST_KRYLOV_FGMRES, S.st.ST_KRYLOV_GMRES):
        solver, prob = make_pair(2, n, nt, time_constant=True, rtol=1e-10, krylov=k)
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(rho, T)
        out[k] = (host(T), solver.stats()["iterations"])
        solver.close()
    a, b = out[S.st.ST_KRYLOV_FGMRES], out[S.st.ST_KRYLOV_GMRES]
    assert a[1] == b[1]
    assert rel(b[0], a[0]) <= 1e-9


def test_null_adjoint_rhs_is_the_compliance_gradient():
    solver, prob = make_pair(2, 20, 12, rtol=1e-11)
    rho = dev(I.rho_uniform((12, 20, 20), 6))
    l1 = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    l2 = torch.zeros_like(l1)
    solver.adjoint(rho, dev(prob.compliance_rhs()), l1)
    solver.adjoint(rho, None, l2)
    assert rel(host(l2), host(l1)) <= 1e-13
    solver.close()


def test_design_fingerprint_detects_a_one_ulp_change():
    """a design change is detected exactly (128-bit hash of the bit patterns), so a
    one-ulp perturbation of ONE element rebuilds the rho-dependent operators and the same design
    passed again does not."""
    solver, prob = make_pair(2, 32, 16, rtol=1e-10)
    r = I.rho_uniform((16, 32, 32), 2)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(r), T)
    s0 = solver.stats()["setups"]
    solver.solve(dev(r), T)
    assert solver.stats()["setups"] == s0
    r2 = r.copy()
    r2.reshape(-1)[12345] = np.nextafter(r2.reshape(-1)[12345], 2.0)
    solver.solve(dev(r2), T)
    assert solver.stats()["setups"] == s0 + 1
    solver.close()


def test_fused_prolongation_option_equivalence_and_kernel_families_solve():
    """fuse_prolong = 0 / 1 give the same solution; the cp.async and generic kernel families solve
    the config-3-shaped space-time problem to the oracle's T."""
    n, nt = 32, 24
    rho = _design(2, n, nt, False, 4)
    outs = []
    for opts in (dict(), dict(fuse_prolong=0), dict(kernel_family=S.st.ST_KERNELS_CPASYNC),
                 dict(kernel_family=S.st.ST_KERNELS_GENERIC)):
        solver, prob = make_pair(2, n, nt, source=("sin", 1.0, 1.0, 2 * np.pi), rtol=1e-10, **opts)
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(dev(rho), T)
        outs.append(host(T))
        solver.close()
    T_ref = prob.forward(rho)
    for T in outs:
        assert rel(T, T_ref) <= 1e-8


# ------------------------------------------------------------------ the paper's coarsest solve
@pytest.mark.parametrize("sdim,n,nt,tc,mats", [(2, 32, 32, False, CFG1_MATS), (2, 32, 64, True, CFG1_MATS),
                                               (3, 8, 16, True, CFG4_MATS)])
def test_gmres_coarsest_solve_matches_oracle(sdim, n, nt, tc, mats):
    """coarse_solver = ST_COARSE_GMRES (GMRES(<= 200)-Jacobi to rtol 1e-6 on the
    coarsest level, here a level of several thousand nodes, larger than the dense solve takes) inside
    FGMRES: T and lambda equal the oracle's."""
    solver, prob = make_pair(sdim, n, nt, mats=mats, time_constant=tc, rtol=1e-10, maxit=800,
                             coarse_solver=S.st.ST_COARSE_GMRES, coarse_max_nodes=6000)
    h = solver.hierarchy()
    assert h[-1]["nodes"] > 1000 and h[-1]["form"] != "dense"
    rho = _design(sdim, n, nt, tc, 2)
    T_ref, lam_ref = prob.solve_both(rho)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(rho), T)
    assert solver.stats()["converged"] == 1
    assert rel(host(T), T_ref) <= 1e-8
    lam = torch.zeros_like(T)
    solver.adjoint(dev(rho), None, lam)
    assert rel(host(lam), lam_ref) <= 1e-8
    solver.close()


def test_paper_solver_variant_with_inner_tolerances():
    """The paper's full preconditioner: GMRES(10)-Jacobi smoother with inner rtol
    1e-6, GMRES(200) coarsest solve with rtol 1e-6, on the semi-coarsened hierarchy; converges to the
    oracle's solution, and semi-coarsening needs fewer outer iterations than full space-time coarsening
    (5.6 / 9.4 vs 9.7 / 55.6)."""
    n, nt = 32, 32
    rho = _design(2, n, nt, False, 7)
    its = {}
    for full in (0, 1):
        solver, prob = make_pair(2, n, nt, rtol=1e-10, maxit=800, smoother=S.st.ST_SMOOTH_GMRES, nu_pre=10,
                                 nu_post=10, smoother_rtol=1e-6, coarse_solver=S.st.ST_COARSE_GMRES,
                                 coarse_max_nodes=2000, full_coarsening=full)
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(dev(rho), T)
        assert solver.stats()["converged"] == 1
        f_its = solver.stats()["iterations"]
        lam = torch.zeros_like(T)
        solver.adjoint(dev(rho), None, lam)
        its[full] = (f_its, solver.stats()["iterations"])
        T_ref, lam_ref = prob.solve_both(rho)
        assert rel(host(T), T_ref) <= 1e-8 and rel(host(lam), lam_ref) <= 1e-8
        solver.close()
    assert its[0][0] <= its[1][0] and its[0][1] <= its[1][1], its


# ------------------------------------------------------------------ the GPU time-stepping baseline
@pytest.mark.parametrize("sdim,n,nsteps,mats,T0,src", [
    (2, 16, 16, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0)),
    (2, 32, 24, CFG4_MATS, 0.4, ("sin", 1.0, 1.0, 2 * np.pi)),
    (2, 20, 12, (0.5, 1.0, 2.0, 0.03, 3.0, 3.0), 0.0, ("ex1", 100.0, 0.0, 0.0)),
    (3, 8, 8, CFG4_MATS, 0.2, ("uniform", 1.0, 0.0, 0.0)),
])
def test_timestepping_baseline_matches_oracle_backward_euler(sdim, n, nsteps, mats, T0, src):
    """st_timestep: the GPU backward-difference stepper with a
    spatial-MG-preconditioned CG per step equals the oracle's direct backward Euler (oracle/timestep.py,
    its own quadrature) at every time plane, to the solver tolerance."""
    solver, prob = make_pair(sdim, n, nsteps, mats=mats, T0=T0, source=src, time_constant=True, rtol=1e-12,
                             maxit=500)
    rho = I.rho_smooth((n,) * sdim, seed=4)
    T = torch.empty((nsteps + 1) * (n + 1) ** sdim, dtype=torch.float64, device=DEV)
    st = solver.timestep(dev(rho), nsteps, T)
    assert st["steps"] == nsteps and st["cg_iterations"] >= nsteps
    C, k, _, _ = O.simp(rho.reshape(-1), prob.mats, prob.mesh)
    cons, _ = O.dirichlet(prob.mesh, prob.bcs)
    plane = (n + 1) ** sdim
    qsrc = prob.src

    def q_of_t(t):  # the oracle's rescaled source at time t (spatially uniform kinds)
        return float(O.stfem._q_tilde(qsrc, prob.mesh, [np.zeros(1)] * sdim, np.array([t]))[0])
    ref = O.backward_euler(n, sdim, C, k, q_of_t, nsteps, T0, cons[plane:2 * plane])
    got = host(T).reshape(nsteps + 1, plane)
    for m in range(nsteps + 1):
        assert rel(got[m], ref[m]) <= 1e-9, (m, rel(got[m], ref[m]))
    # host output buffer (library staging) gives the same result
    Th = np.zeros((nsteps + 1) * plane)
    solver.timestep(rho, nsteps, Th)
    assert rel(Th, host(T)) <= 1e-14
    solver.close()


def test_timestepping_converges_to_the_space_time_solution():
    """Both discretisations approach the same continuous solution: with nsteps = nt they differ by
    O(dt) (first-order backward difference vs the stabilised space-time element), and the
    gap shrinks under time refinement."""
    n = 16
    rho = I.rho_smooth((n, n), seed=1)
    gaps = []
    for nt in (16, 32, 64):
        solver, prob = make_pair(2, n, nt, time_constant=True, rtol=1e-12, maxit=500)
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(dev(rho), T)
        Tts = torch.empty_like(T)
        solver.timestep(dev(rho), nt, Tts)
        gaps.append(rel(host(Tts), host(T)))
        solver.close()
    assert gaps[1] < gaps[0] and gaps[2] < gaps[1], gaps


# ------------------------------------------------------------------ the paper's PDE filter + projection
@pytest.mark.parametrize("sdim,n,nt,rfac", [(2, 16, 16, 2.4), (2, 40, 24, 2.4), (3, 6, 10, 2.4), (2, 12, 20, 6.0)])
def test_pde_filter_projection_and_chain_rule_match_oracle(sdim, n, nt, rfac):
    """st_pde_filter / st_pde_filter_grad: the filtered element
    field, its projection and the chain-rule sensitivities equal the oracle's direct solves (CG to 1e-12);
    the filter then feeds the state solve (the physical design of PAPER.md:552)."""
    solver, prob = make_pair(sdim, n, nt, rtol=1e-11, maxit=500)
    rng = np.random.default_rng(5)
    g = rng.uniform(0.0, 1.0, (nt,) + (n,) * sdim)
    rx, rt = rfac / n, rfac / nt
    gb = torch.empty(g.size, dtype=torch.float64, device=DEV)
    ge = torch.empty_like(gb)
    its = solver.pde_filter(dev(g), gb, ge, rx=rx, rt=rt)
    assert 0 < its <= 200
    _, ge_ref, gb_ref = O.pde_filter(prob.mesh, g.reshape(-1), rx, rt)
    assert rel(host(ge), ge_ref) <= 1e-10
    assert rel(host(gb), gb_ref) <= 1e-9
    w = rng.uniform(-1, 1, g.size)
    out = torch.empty_like(gb)
    solver.pde_filter_grad(ge, dev(w), out, rx=rx, rt=rt)
    ref = O.pde_filter_grad(prob.mesh, ge_ref, w, rx, rt)
    assert rel(host(out), ref) <= 1e-9
    # the projected field is a valid design for the state solve
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(gb.clamp(1e-3, 1.0), T)
    assert solver.stats()["converged"] == 1
    solver.close()
