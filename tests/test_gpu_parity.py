"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on
the same seeded inputs (north_star tolerances: operator <= 1e-12, solution <= 1e-8 at
rtol 1e-10, sensitivities <= 1e-7, all fp64, normwise relative; R-15, R-16)."""
import numpy as np
import pytest
import scipy.sparse as sp

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


OP_CASES = [
    # (sdim, n, nt, mats, T0, design, seed, tc)
    (2, 16, 16, CFG1_MATS, 0.0, "uniform", 0, False),
    (2, 16, 16, CFG1_MATS, 0.0, "uniform", 3, False),
    (2, 12, 20, CFG4_MATS, 0.3, "uniform", 1, False),
    (2, 32, 32, CFG1_MATS, 0.0, "smooth_tc", 0, True),
    (2, 2, 2, CFG1_MATS, 0.5, "uniform", 2, False),
    (2, 7, 5, CFG4_MATS, 0.0, "uniform", 4, False),
    (3, 4, 6, CFG4_MATS, 0.2, "uniform", 0, False),
    (3, 6, 12, CFG4_MATS, 0.0, "smooth_tc", 0, True),
    (3, 10, 8, CFG4_MATS, 0.2, "smooth_tc", 1, True),     # (3+1)D TMA kernel: several 32x4x2 tiles, ragged
]


def _rho(sdim, n, nt, design, seed, tc):
    if design == "uniform":
        shape = (n,) * sdim if tc else (nt,) + (n,) * sdim
        return I.rho_uniform(shape, seed)
    return I.design_for(sdim, n, nt, design, seed)


@pytest.mark.parametrize("case", OP_CASES, ids=lambda c: f"{c[0]}d-{c[1]}x{c[2]}-s{c[6]}-{'tc' if c[7] else 'st'}")
def test_operator_parity(case):
    sdim, n, nt, mats, T0, design, seed, tc = case
    solver, prob = make_pair(sdim, n, nt, mats=mats, T0=T0, time_constant=tc)
    rho = _rho(sdim, n, nt, design, seed, tc)
    K = prob.K(rho)
    Kbc, _, _, _ = prob.system(rho)
    x = I.rand_vector(prob.mesh.n_nodes, seed + 1)
    xd, yd = dev(x), torch.empty(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    rd = dev(rho)
    for trans in (False, True):
        for bc in (False, True):
            A = (Kbc if bc else K)
            ref = (A.T if trans else A) @ x
            solver.apply(rd, xd, yd, transpose=trans, bc=bc)
            assert rel(host(yd), ref) <= 1e-12, (trans, bc, rel(host(yd), ref))
    solver.close()


@pytest.mark.parametrize("src,T0", [(("uniform", 1.0, 0.0, 0.0), 0.0), (("sin", 1.0, 1.0, 2 * np.pi), 0.4)])
def test_rhs_parity(src, T0):
    solver, prob = make_pair(2, 12, 10, mats=CFG4_MATS, T0=T0, source=src)
    rho = I.rho_uniform((10, 12, 12), 5)
    _, b_ref, _, _ = prob.system(rho)
    f = torch.empty(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    b = torch.empty_like(f)
    solver.rhs(dev(rho), f, b)
    assert rel(host(f), prob.f()) <= 1e-13
    assert rel(host(b), b_ref) <= 1e-12


SOLVE_CASES = [
    # name, sdim, n, nt, mats, T0, source, tau, design, tc
    ("cfg1", 2, 16, 16, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "uniform", False),
    ("cfg2-replica", 2, 32, 32, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "smooth_tc", True),
    ("cfg3-replica", 2, 32, 32, CFG1_MATS, 0.0, ("sin", 1.0, 1.0, 2 * np.pi), 1.0, "smooth_layers", False),
    ("cfg4-replica", 3, 6, 12, CFG4_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "smooth_tc", True),
    ("cfg5-replica-G2", 2, 16, 32, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 2.0, "const", False),
    ("nonzero-T0", 2, 12, 20, CFG4_MATS, 0.7, ("sin", 1.0, 1.0, 2 * np.pi), 1.0, "uniform", False),
    # the paper's default materials: C 0.5 / 1, k 0.03 / 3, p_c = 2, p_k = 3
    ("paper-materials", 2, 16, 16, (0.5, 1.0, 2.0, 0.03, 3.0, 3.0), 0.0, ("sin", 1.0, 1.0, 2 * np.pi), 1.0,
     "uniform", False),
    ("paper-materials-tc", 2, 24, 16, (0.5, 1.0, 2.0, 0.03, 3.0, 3.0), 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0,
     "smooth_tc", True),
]


@pytest.mark.parametrize("case", SOLVE_CASES, ids=lambda c: c[0])
def test_solve_adjoint_sensitivity_parity(case):
    name, sdim, n, nt, mats, T0, src, tau, design, tc = case
    solver, prob = make_pair(sdim, n, nt, mats=mats, T0=T0, source=src, tau=tau, time_constant=tc,
                             rtol=1e-10, maxit=400)
    if design == "uniform":
        rho = _rho(sdim, n, nt, "uniform", 0, tc)
    else:
        rho = I.design_for(sdim, n, nt, design, 0)
    T_ref, lam_ref = prob.solve_both(rho)
    dJ_ref = prob.sensitivity(rho, T_ref, lam_ref)
    rd = dev(rho)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(rd, T)
    st = solver.stats()
    assert st["converged"] == 1 and st["rel_residual"] <= 1e-10
    assert rel(host(T), T_ref) <= 1e-8, rel(host(T), T_ref)
    g = dev(prob.compliance_rhs())
    lam = torch.zeros_like(T)
    solver.adjoint(rd, g, lam)
    assert solver.stats()["converged"] == 1
    assert rel(host(lam), lam_ref) <= 1e-8, rel(host(lam), lam_ref)
    dJ = torch.empty(rho.size, dtype=torch.float64, device=DEV)
    solver.sensitivity(rd, T, lam, dJ)
    assert rel(host(dJ).reshape(dJ_ref.shape), dJ_ref) <= 1e-7, rel(host(dJ).reshape(dJ_ref.shape), dJ_ref)
    solver.close()


@pytest.mark.parametrize("case", [("cfg3-replica", 2, 32, 32, CFG1_MATS, ("sin", 1.0, 1.0, 2 * np.pi), "smooth_layers", False),
                                  ("cfg2-replica", 2, 32, 32, CFG1_MATS, ("uniform", 1.0, 0.0, 0.0), "smooth_tc", True),
                                  ("cfg4-replica", 3, 8, 16, CFG4_MATS, ("uniform", 1.0, 0.0, 0.0), "smooth_tc", True)],
                         ids=lambda c: c[0])
@pytest.mark.parametrize("smoother", [(0, 3), (2, 10)], ids=["jacobi3", "gmres10"])
def test_full_coarsening_solves_and_semi_coarsening_needs_fewer_iterations(case, smoother):
    """Full space-time coarsening (option full_coarsening) gives the oracle's T and
    lambda, and Algorithm 1's semi-coarsening needs no more FGMRES iterations than it (PAPER.md:781,
    Example 1B: 9.7 / 55.6 state / adjoint iterations with full coarsening vs 5.6 / 9.4 with
    semi-coarsening; the paper's counts are for its GMRES-Jacobi smoother and grids, so only the
    ordering is asserted). Run with the damped-Jacobi smoother of this build and with the paper's
    GMRES(10)-Jacobi smoother (ST_SMOOTH_GMRES)."""
    name, sdim, n, nt, mats, src, design, tc = case
    rho = I.design_for(sdim, n, nt, design, 0)
    its = {}
    for full in (0, 1):
        solver, prob = make_pair(sdim, n, nt, mats=mats, source=src, time_constant=tc, rtol=1e-10, maxit=400,
                                 full_coarsening=full, smoother=smoother[0], nu_pre=smoother[1],
                                 nu_post=smoother[1])
        if full:
            assert all(h["kind"] == "full" for h in solver.hierarchy()[1:])
        T_ref, lam_ref = prob.solve_both(rho)
        rd = dev(rho)
        T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
        solver.solve(rd, T)
        a = solver.stats()
        assert a["converged"] == 1 and rel(host(T), T_ref) <= 1e-8, (full, rel(host(T), T_ref))
        lam = torch.zeros_like(T)
        solver.adjoint(rd, dev(prob.compliance_rhs()), lam)
        b = solver.stats()
        assert b["converged"] == 1 and rel(host(lam), lam_ref) <= 1e-8, (full, rel(host(lam), lam_ref))
        its[full] = (a["iterations"], b["iterations"])
        solver.close()
    print(name, smoother, "semi", its[0], "full", its[1])
    assert its[0][0] <= its[1][0] and its[0][1] <= its[1][1], its


def test_host_pointer_path_and_warm_start():
    """C ABI with HOST buffers (library stages them) gives the same result; a warm start
    from the solution converges in zero iterations."""
    solver, prob = make_pair(2, 16, 16, rtol=1e-10)
    rho = I.rho_uniform((16, 16, 16), 0)
    T_ref = prob.forward(rho)
    T = np.zeros(prob.mesh.n_nodes)
    solver.solve(rho, T)
    assert rel(T, T_ref) <= 1e-8
    solver.solve(rho, T)
    assert solver.stats()["iterations"] == 0
    lam = np.zeros_like(T)
    solver.adjoint(rho, prob.compliance_rhs(), lam)
    dJ = np.zeros(rho.size)
    solver.sensitivity(rho, T, lam, dJ)
    _, lam_ref = prob.solve_both(rho)
    assert rel(dJ.reshape(rho.shape), prob.sensitivity(rho, T_ref, lam_ref)) <= 1e-7
    solver.close()


def _P1(nf, kind):
    """1D linear interpolation coarse(n/2) -> fine(n) nodes."""
    nc = nf // 2
    P = np.zeros((nf + 1, nc + 1))
    for i in range(nf + 1):
        if i % 2 == 0:
            P[i, i // 2] = 1.0
        else:
            P[i, i // 2] = P[i, i // 2 + 1] = 0.5
    return P


@pytest.mark.parametrize("sdim,n,nt,tc,mats", [(2, 16, 16, False, CFG4_MATS), (2, 32, 32, True, CFG4_MATS),
                                                 (3, 4, 8, False, CFG4_MATS), (2, 8, 32, False, CFG4_MATS),
                                                 (3, 8, 8, True, CFG4_MATS),
                                                 # uniform capacity, space-time design: the stored-stencil
                                                 # TMA kernel (tv2d SRC 1) on levels of several ragged tiles
                                                 (2, 80, 12, False, CFG1_MATS),
                                                 # full space-time coarsening
                                                 (2, 16, 16, False, "full4"), (2, 32, 32, True, "full4"),
                                                 (2, 32, 16, False, "full1"), (3, 4, 8, False, "full4"),
                                                 (3, 8, 8, True, "full4")])
def test_coarse_operators(sdim, n, nt, tc, mats):
    """Each coarse level equals, with the Dirichlet masks of its own grid, the operator built
    here independently from assembled matrices: conduction part
    by Galerkin P^T A P with the space/time linear interpolation P; capacity
    part by Galerkin under space coarsening and re-stabilised (upwind U, layer-mean capacity)
    under time coarsening."""
    opts = {}
    if isinstance(mats, str):  # "full<mats>": the full-coarsening hierarchy
        opts = {"full_coarsening": 1}
        mats = CFG4_MATS if mats == "full4" else CFG1_MATS
    solver, prob = make_pair(sdim, n, nt, mats=mats, time_constant=tc, **opts)
    rho = I.rho_uniform((n,) * sdim if tc else (nt,) + (n,) * sdim, 3)
    H = solver.hierarchy()
    if opts:
        assert all(h["kind"] == "full" for h in H[1:]), H
    C, k, _, _, _ = prob.coefficients(rho)
    Kcap = O.assemble_K(prob.mesh, C, np.zeros_like(k)).tocsr()
    Kcon = O.assemble_K(prob.mesh, np.zeros_like(C), k).tocsr()
    nf, ntf = H[0]["n"], H[0]["nt"]
    def space_step(Kcap, Kcon, nf, ntf):
        Px = sp.csr_matrix(_P1(nf, "s"))
        Ps = Px
        for _ in range(sdim - 1):
            Ps = sp.kron(Px, Ps)
        P = sp.kron(sp.identity(ntf + 1), Ps).tocsr()
        return (P.T @ Kcap @ P).tocsr(), (P.T @ Kcon @ P).tocsr()

    for l in range(1, len(H)):
        Psp = (nf + 1) ** sdim
        if H[l]["kind"] in ("space", "full"):
            Kcap, Kcon = space_step(Kcap, Kcon, nf, ntf)
            P = None
            if H[l]["kind"] == "full":  # P_t (x) P_s = the time step applied to the space-coarsened operator
                nf = H[l]["n"]
                Psp = (nf + 1) ** sdim
        if H[l]["kind"] in ("time", "full"):
            P = sp.kron(sp.csr_matrix(_P1(ntf, "t")), sp.identity(Psp)).tocsr()
            # layer masses M_tau = -block(tau+1, tau) of the capacity part (U[1][0] = -1)
            ntc = ntf // 2
            U = np.array([[0.0, 0.0], [-1.0, 1.0]])
            blocks = []
            for T in range(ntc):
                M0 = -Kcap[(2 * T + 1) * Psp:(2 * T + 2) * Psp, (2 * T) * Psp:(2 * T + 1) * Psp]
                M1 = -Kcap[(2 * T + 2) * Psp:(2 * T + 3) * Psp, (2 * T + 1) * Psp:(2 * T + 2) * Psp]
                Mb = 0.5 * (M0 + M1)
                E = sp.lil_matrix((ntc + 1, ntc + 1))
                for a in range(2):
                    for b in range(2):
                        E[T + a, T + b] = U[a, b]
                blocks.append(sp.kron(E.tocsr(), Mb))
            Kcap = sum(blocks).tocsr()
        if P is not None:
            Kcon = (P.T @ Kcon @ P).tocsr()
        nf, ntf = H[l]["n"], H[l]["nt"]
        mesh_l = O.Mesh(sdim, nf, max(ntf, 2))
        cons, _ = O.dirichlet(mesh_l, O.BCs())
        cons = cons[:(nf + 1) ** sdim * (ntf + 1)]
        free = (~cons).astype(float)
        Kl = Kcap + Kcon
        Aref = sp.diags(free) @ Kl @ sp.diags(free) + sp.diags(cons.astype(float))
        x = I.rand_vector(Aref.shape[0], 7 + l)
        y = torch.empty(Aref.shape[0], dtype=torch.float64, device=DEV)
        for trans in (False, True):
            solver.level_apply(dev(rho), l, dev(x), y, transpose=trans)
            ref = (Aref.T if trans else Aref) @ x
            assert rel(host(y), ref) <= 1e-12, (l, H[l], trans, rel(host(y), ref))
    solver.close()


@pytest.mark.parametrize("sdim,n,nt,tc,opts", [(2, 16, 16, False, {}), (2, 40, 24, True, {}), (2, 8, 32, False, {}),
                                                  (3, 4, 8, False, {}), (3, 8, 16, True, {}), (3, 10, 8, True, {}),
                                                  (2, 16, 16, False, {"full_coarsening": 1}),
                                                  (3, 8, 8, True, {"full_coarsening": 1}),
                                                  (2, 16, 8, False, {"all_walls": True})])
def test_transfer_parity(sdim, n, nt, tc, opts):
    """Every level transfer equals the textbook linear interpolation P between the two node grids
    (1 at coincident nodes, 1/2 to each neighbour along every coarsened direction,
    Kronecker product over the directions) with the Dirichlet masks of DESIGN.md 'Coarse operators':
    restriction m_c P^T r, prolongation m_f P e. Covers the space, time and full coarsening kernels of
    both dimensions (the paired (2+1)D space kernels, the paired time kernels, the generic kernels)."""
    opts = dict(opts)
    walls = bool(opts.pop("all_walls", False))
    solver, prob = make_pair(sdim, n, nt, mats=CFG4_MATS, time_constant=tc, all_walls=walls, **opts)
    rho = dev(I.rho_uniform((n,) * sdim if tc else (nt,) + (n,) * sdim, 3))
    H = solver.hierarchy()
    kinds = set()
    for l in range(len(H) - 1):
        nf, ntf, nc, ntc, kind = H[l]["n"], H[l]["nt"], H[l + 1]["n"], H[l + 1]["nt"], H[l + 1]["kind"]
        kinds.add(kind)
        Ps = sp.identity((nf + 1) ** sdim, format="csr")
        if kind in ("space", "full"):
            Px = sp.csr_matrix(_P1(nf, "s"))
            Ps = Px
            for _ in range(sdim - 1):
                Ps = sp.kron(Px, Ps)
        Pt = sp.csr_matrix(_P1(ntf, "t")) if kind in ("time", "full") else sp.identity(ntf + 1)
        P = sp.kron(Pt, Ps).tocsr()
        assert P.shape == ((nf + 1) ** sdim * (ntf + 1), (nc + 1) ** sdim * (ntc + 1))
        free = []
        for (m, mt) in ((nf, ntf), (nc, ntc)):
            cons, _ = O.dirichlet(O.Mesh(sdim, m, max(mt, 2)), O.BCs(all_walls=walls))
            free.append((~cons[:(m + 1) ** sdim * (mt + 1)]).astype(float))
        r = I.rand_vector(P.shape[0], 11 + l)
        e = I.rand_vector(P.shape[1], 31 + l)
        rc = torch.empty(P.shape[1], dtype=torch.float64, device=DEV)
        xf = torch.empty(P.shape[0], dtype=torch.float64, device=DEV)
        solver.level_transfer(rho, l, dev(r), rc, restrict=True)
        solver.level_transfer(rho, l, dev(e), xf, restrict=False)
        assert rel(host(rc), free[1] * (P.T @ r)) <= 1e-14, (l, H[l + 1], rel(host(rc), free[1] * (P.T @ r)))
        assert rel(host(xf), free[0] * (P @ e)) <= 1e-14, (l, H[l + 1], rel(host(xf), free[0] * (P @ e)))
    if not opts and n >= 8:
        assert {"space", "time"} <= kinds, kinds
    solver.close()


def test_iteration_counts_reasonable():
    """Config-1 forward/adjoint converge in a modest number of outer iterations."""
    solver, prob = make_pair(2, 16, 16)
    rho = dev(I.rho_uniform((16, 16, 16), 0))
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(rho, T)
    assert solver.stats()["iterations"] <= 40
    solver.close()


KERNEL_VARIANTS = {"tma": S.st.ST_KERNELS_TMA, "cpasync": S.st.ST_KERNELS_CPASYNC, "tma2d": S.st.ST_KERNELS_TMA2D,
                   "generic": S.st.ST_KERNELS_GENERIC}  # st_options_t kernel_family


@pytest.mark.parametrize("variant", sorted(KERNEL_VARIANTS))
@pytest.mark.parametrize("case", [(2, 32, 32, "smooth_tc", True), (2, 16, 16, "uniform", False),
                                  (2, 40, 7, "uniform", False), (2, 64, 24, "smooth_tc", True),
                                  (3, 8, 6, "smooth_tc", True)],
                         ids=lambda c: f"{c[0]}d-{c[1]}x{c[2]}-{'tc' if c[4] else 'st'}")
def test_operator_parity_all_kernel_variants(variant, case):
    """Every (2+1)D operator kernel (TMA ring, cp.async ring, generic) gives the oracle's K x and
    K^T x on every level kind it serves; the grids span several 32 x 8 tiles with ragged tails and
    split (tile, plane) work ranges across CTAs."""
    sdim, n, nt, design, tc = case
    solver, prob = make_pair(sdim, n, nt, mats=CFG4_MATS, T0=0.3, time_constant=tc, rtol=1e-12, maxit=400,
                             kernel_family=KERNEL_VARIANTS[variant])
    rho = _rho(sdim, n, nt, design, 5, tc)
    K = prob.K(rho)
    Kbc, _, _, _ = prob.system(rho)
    x = I.rand_vector(prob.mesh.n_nodes, 11)
    xd, yd = dev(x), torch.empty(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    for trans in (False, True):
        for bc in (False, True):
            ref = ((Kbc if bc else K).T if trans else (Kbc if bc else K)) @ x
            solver.apply(dev(rho), xd, yd, transpose=trans, bc=bc)
            assert rel(host(yd), ref) <= 1e-12, (variant, trans, bc, rel(host(yd), ref))
    # a full solve exercises every level operator / mode of this kernel family
    T_ref = prob.forward(rho)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(rho), T)
    assert solver.stats()["converged"] == 1
    assert rel(host(T), T_ref) <= 1e-8
    solver.close()


@pytest.mark.parametrize("sdim,n,nt,tc,mats", [(2, 12, 10, True, CFG1_MATS), (2, 8, 12, False, CFG4_MATS),
                                               (3, 4, 6, True, CFG4_MATS),
                                               # uniform capacity, space-time design: the closed-form k~-table
                                               # kernel (gersh_tv2d_kernel)
                                               (2, 10, 12, False, CFG1_MATS), (2, 33 - 1, 6, False, CFG1_MATS)])
def test_jacobi_weight_bound(sdim, n, nt, tc, mats):
    """The fine level's Gershgorin ratio equals max_i sum_j |A_ij| / |A_ii| of the
    oracle's K_bc over free rows, bounds the spectral radius of D^-1 K_bc, and omega = min(cap, 1.9/R)."""
    solver, prob = make_pair(sdim, n, nt, mats=mats, time_constant=tc)
    rho = _rho(sdim, n, nt, "uniform", 2, tc)
    x = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.apply(dev(rho), x, torch.empty_like(x))      # binds rho
    solver.rhs(dev(rho), None, None)                    # rho-dependent setup (incl. the weights)
    H = solver.hierarchy()
    Kbc, _, cons, _ = prob.system(rho)
    A = abs(Kbc).tocsr()
    d = np.abs(Kbc.diagonal())
    ratio = np.asarray(A.sum(axis=1)).ravel() / d
    R_ref = ratio[~cons].max()
    assert abs(H[0]["lam_max"] - R_ref) <= 1e-12 * R_ref, (H[0]["lam_max"], R_ref)
    DinvK = (Kbc.toarray() / Kbc.diagonal()[:, None])
    rho_spec = np.abs(np.linalg.eigvals(DinvK)).max()
    assert rho_spec <= H[0]["lam_max"] * (1 + 1e-12)
    assert abs(H[0]["omega"] - min(0.75, 1.9 / R_ref)) <= 1e-14
    solver.close()


@pytest.mark.parametrize("tc", [False, True])
def test_config5_design_loop_matches_oracle(tc):
    """BASELINE config 5 (replica: 16^2 x 16, 3 OC iterations from rho = 0.4; R-13): the
    GPU loop (st_filter / st_solve / st_adjoint / st_sensitivity / st_oc_update) gives the oracle's
    designs and compliance history."""
    import paper_2508_09589_b200 as S
    n, nt = 16, 16
    shape = (n, n) if tc else (nt, n, n)
    solver, prob = make_pair(2, n, nt, time_constant=tc, rtol=1e-11, maxit=400)
    rho0 = np.full(shape, 0.4)
    designs, hist = O.design_loop(prob, rho0, 3)
    rho = dev(rho0).reshape(-1).clone()
    hist_g = S.design_loop(solver, rho, 3)
    assert np.allclose(hist_g, hist, rtol=1e-9), (hist_g, hist)
    assert rel(host(rho).reshape(shape), designs[-1]) <= 1e-7, rel(host(rho).reshape(shape), designs[-1])
    solver.close()


def test_filter_and_oc_kernels_match_oracle():
    solver, prob = make_pair(2, 12, 10)
    rng = np.random.default_rng(4)
    a = rng.uniform(0, 1, (10, 12, 12))
    out = torch.empty(a.size, dtype=torch.float64, device=DEV)
    solver.filter(dev(a), out)
    assert rel(host(out).reshape(a.shape), O.density_filter(a)) <= 1e-14
    solver.filter(dev(a), out, transpose=True)
    assert rel(host(out).reshape(a.shape), O.density_filter(a, transpose=True)) <= 1e-14
    dJ = -rng.uniform(1e-6, 1e-3, a.shape)
    new = torch.empty_like(out)
    lam = solver.oc_update(dev(a), dev(dJ), new)
    ref, lam_ref = O.oc_update(a, dJ)
    assert abs(lam - lam_ref) <= 1e-10 * lam_ref
    assert rel(host(new).reshape(a.shape), ref) <= 1e-12
    solver.close()


@pytest.mark.parametrize("sdim,n,nt,tc", [(2, 12, 10, False), (3, 4, 6, True)])
def test_pnorm_objective_and_adjoint_rhs(sdim, n, nt, tc):
    """The paper's objective phi = (sum Tavg^P)^(1/P), P = 20 and its gradient
     equal the oracle's; the adjoint with that RHS matches the oracle's too."""
    solver, prob = make_pair(sdim, n, nt, mats=CFG4_MATS, time_constant=tc, rtol=1e-11, maxit=400)
    rho = _rho(sdim, n, nt, "uniform", 8, tc)
    T_ref = prob.forward(rho)
    phi_ref, g_ref = O.pnorm_objective(prob.mesh, T_ref, 20.0)
    T = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(rho), T)
    g = torch.empty_like(T)
    phi = solver.pnorm(T, 20.0, g)
    assert abs(phi - phi_ref) <= 1e-10 * abs(phi_ref)
    assert rel(host(g), g_ref) <= 1e-9
    lam = torch.zeros_like(T)
    solver.adjoint(dev(rho), g, lam)
    lam_ref = prob.adjoint(rho, g_ref)
    assert rel(host(lam), lam_ref) <= 1e-8
    solver.close()


def test_per_design_tables_follow_the_design_across_hooks():
    """The per-design k~ table of a space-time design (tv2d) is rebuilt when rho changes and is not
    left stale by a test hook that binds another rho: solve(A), apply(B), solve(A) gives the first
    solution again, and solve(B) the oracle's solution for B."""
    solver, prob = make_pair(2, 32, 16, rtol=1e-10, maxit=400)
    ra = I.rho_uniform((16, 32, 32), 1)
    rb = I.rho_uniform((16, 32, 32), 2)
    T1 = torch.zeros(prob.mesh.n_nodes, dtype=torch.float64, device=DEV)
    solver.solve(dev(ra), T1)
    y = torch.empty_like(T1)
    solver.apply(dev(rb), dev(I.rand_vector(prob.mesh.n_nodes, 3)), y)
    T2 = torch.zeros_like(T1)
    solver.solve(dev(ra), T2)
    assert rel(host(T2), host(T1)) <= 1e-12
    T3 = torch.zeros_like(T1)
    solver.solve(dev(rb), T3)
    assert rel(host(T3), prob.forward(rb)) <= 1e-8
    solver.close()


@pytest.mark.parametrize("n,nt,design,tc", [(64, 32, "smooth_tc", True), (40, 12, "uniform", True),
                                             (128, 16, "smooth_tc", True)])
def test_prolongation_fused_into_post_sweep_equals_separate_kernels(n, nt, design, tc):
    """The V-cycle with the prolongation + correction fused into the first post-smoothing sweep
    (tc2d PRO variant on the coarse time-constant levels, default) is the same linear map as the
    separate prolongation kernel followed by the sweep (options fuse_prolong = 0), forward and adjoint,
    on multi-tile ragged grids with the sink patch; and the fused path is taken (fewer launches per
    V-cycle)."""
    rho = _rho(2, n, nt, design, 5, tc) if design == "uniform" else I.design_for(2, n, nt, design, 5)
    x = I.rand_vector((n + 1) ** 2 * (nt + 1), 13)
    outs, launches = {}, {}
    for flag in ("1", "0"):  # "1": separate kernels, "0": fused (as the former ST_NO_PRO flag)
        solver, prob = make_pair(2, n, nt, time_constant=tc, use_graphs=0, fuse_prolong=0 if flag == "1" else 1)
        z = torch.empty(x.size, dtype=torch.float64, device=DEV)
        zt = torch.empty_like(z)
        solver.vcycle(dev(rho), dev(x), z)
        k0 = solver.kernel_launches()
        solver.vcycle(dev(rho), dev(x), z)
        launches[flag] = solver.kernel_launches() - k0
        solver.vcycle(dev(rho), dev(x), zt, transpose=True)
        outs[flag] = (host(z), host(zt))
        solver.close()
    assert rel(outs["0"][0], outs["1"][0]) <= 1e-12
    assert rel(outs["0"][1], outs["1"][1]) <= 1e-12
    assert launches["0"] < launches["1"], launches


# ------------------------------------------------------------------ the paper's example presets
PAPER_MATS = (0.5, 1.0, 2.0, 0.03, 3.0, 3.0)   # C 0.5 / 1, k 0.03 / 3, p_c 2, p_k 3
EX_CASES = [
    # Example 1: oscillating uniform source Q0 = 100, tau = 1, sink patch
    ("ex1", 2, 16, 32, dict(source=("ex1", 100.0, 0.0, 0.0), tau=1.0)),
    ("ex1-3d", 3, 6, 12, dict(source=("ex1", 100.0, 0.0, 0.0), tau=1.0)),
    # Example 2: moving Gaussian, Q0 = 1, sigma 0.05, R 0.25, w = pi, tau = 6, cold walls
    ("ex2", 2, 24, 48, dict(source=("ex2", 1.0, 0.0, np.pi, 0.05, 0.25), tau=6.0, all_walls=True, has_patch=False)),
    ("ex2-T0", 2, 16, 24, dict(source=("ex2", 1.0, 0.0, np.pi, 0.05, 0.25), tau=6.0, all_walls=True, T0=0.3)),
]


@pytest.mark.parametrize("case", EX_CASES, ids=lambda c: c[0])
def test_paper_example_presets_match_oracle(case):
    """The sources of Examples 1 and 2 (ST_SRC_EX1 / ST_SRC_EX2, the latter by 2 x 2 x 2-point Gauss
    quadrature of the moving Gaussian, R-5) and Example 2's cold walls (all_walls): RHS f,
    operator, forward, adjoint (p-norm objective) and sensitivities equal the
    oracle's."""
    name, sdim, n, nt, kw = case
    tc = sdim == 3
    solver, prob = make_pair(sdim, n, nt, mats=PAPER_MATS, time_constant=tc, rtol=1e-11, maxit=600, **kw)
    rho = I.rho_smooth((n,) * sdim, seed=3) if tc else I.rho_uniform((nt,) + (n,) * sdim, 3)
    N = prob.mesh.n_nodes
    f = torch.empty(N, dtype=torch.float64, device=DEV)
    solver.rhs(dev(rho), f, None)
    f_ref = prob.f()
    assert rel(host(f), f_ref) <= 1e-13, rel(host(f), f_ref)
    Kbc, _, _, _ = prob.system(rho)
    x = I.rand_vector(N, 9)
    y = torch.empty(N, dtype=torch.float64, device=DEV)
    solver.apply(dev(rho), dev(x), y)
    assert rel(host(y), Kbc @ x) <= 1e-12
    T_ref = prob.forward(rho)
    T = torch.zeros(N, dtype=torch.float64, device=DEV)
    solver.solve(dev(rho), T)
    assert rel(host(T), T_ref) <= 1e-8
    phi_ref, g_ref = O.pnorm_objective(prob.mesh, T_ref, 20.0)
    g = torch.empty_like(T)
    solver.pnorm(T, 20.0, g)
    lam = torch.zeros_like(T)
    solver.adjoint(dev(rho), g, lam)
    lam_ref = prob.adjoint(rho, g_ref)
    assert rel(host(lam), lam_ref) <= 1e-8
    dJ_ref = prob.sensitivity(rho, T_ref, lam_ref)
    dJ = torch.empty(rho.size, dtype=torch.float64, device=DEV)
    solver.sensitivity(dev(rho), T, lam, dJ)
    assert rel(host(dJ).reshape(dJ_ref.shape), dJ_ref) <= 1e-7
    solver.close()


@pytest.mark.parametrize("case", [(2, 16, 16, CFG1_MATS, 0.0, "uniform", False, ("uniform", 1.0, 0.0, 0.0)),
                                  (2, 32, 32, CFG1_MATS, 0.0, "smooth_tc", True, ("uniform", 1.0, 0.0, 0.0)),
                                  (2, 12, 20, CFG4_MATS, 0.7, "uniform", False, ("sin", 1.0, 1.0, 2 * np.pi)),
                                  (3, 6, 12, CFG4_MATS, 0.0, "smooth_tc", True, ("uniform", 1.0, 0.0, 0.0))],
                         ids=["cfg1", "cfg2-replica", "nonzero-T0", "cfg4-replica"])
@pytest.mark.parametrize("where", ["device", "host"])
@pytest.mark.parametrize("rhs", ["compliance", "caller"])
def test_design_step_matches_oracle_and_separate_calls(case, where, rhs):
    """st_design_step (forward solve, adjoint solve, sensitivities in one call; host results copied
    back on a side stream while the next phase runs) gives the oracle's T, lambda and dJ
     and the same vectors as st_solve + st_adjoint + st_sensitivity."""
    sdim, n, nt, mats, T0, design, tc, src = case
    solver, prob = make_pair(sdim, n, nt, mats=mats, T0=T0, source=src, time_constant=tc, rtol=1e-10, maxit=400)
    rho = _rho(sdim, n, nt, design, 0, tc).reshape(-1)
    rho_o = rho.reshape(((n,) * sdim) if tc else ((nt,) + (n,) * sdim))
    T_ref, lam_ref = prob.solve_both(rho_o)
    dJ_ref = prob.sensitivity(rho_o, T_ref, lam_ref)
    g = prob.compliance_rhs() if rhs == "caller" else None
    N = prob.mesh.n_nodes
    if where == "device":
        mk = lambda a: dev(a)
        back = host
    else:
        mk = lambda a: np.ascontiguousarray(a, dtype=np.float64).copy()
        back = lambda a: a
    T, lam, dJ = mk(np.zeros(N)), mk(np.zeros(N)), mk(np.zeros(rho.size))
    fs, as_ = solver.design_step(mk(rho), None if g is None else mk(g), T, lam, dJ, allow_nc=True)
    assert fs["converged"] == 1 and as_["converged"] == 1 and fs["rel_residual"] <= 1e-10, (fs, as_)
    assert rel(back(T), T_ref) <= 1e-8, rel(back(T), T_ref)
    assert rel(back(lam), lam_ref) <= 1e-8, rel(back(lam), lam_ref)
    assert rel(back(dJ).reshape(dJ_ref.shape), dJ_ref) <= 1e-7
    # the three separate calls from the same initial guesses: the same kernels in the same order
    T2, lam2, dJ2 = mk(np.zeros(N)), mk(np.zeros(N)), mk(np.zeros(rho.size))
    solver.solve(mk(rho), T2)
    solver.adjoint(mk(rho), None if g is None else mk(g), lam2)
    solver.sensitivity(mk(rho), T2, lam2, dJ2)
    for a, b in ((T, T2), (lam, lam2), (dJ, dJ2)):
        assert rel(back(a), back(b)) <= 1e-14, rel(back(a), back(b))
    solver.close()
