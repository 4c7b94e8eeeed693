"""Full-size parity (R-21): at BASELINE sizes the oracle cannot factorise the system, so
the GPU result is certified by the oracle's own element matrices on sampled rows and elements.

For a solve to true relative residual rtol, every row satisfies |b_i - (K_bc T)_i| <= ||b - K_bc T||
<= rtol ||b||; the test recomputes (K_bc T)_i with oracle.row_apply (quadrature element matrices,
no code shared with the CUDA path) at random rows plus every row of the first, second and last time
planes, and bounds the residual there. Sensitivities of sampled elements are recomputed from the GPU
T and lambda with oracle.sensitivity_elements. Launch configuration = bench.py's (config 2: default
options, rtol 1e-8)."""
import numpy as np
import pytest

import oracle as O
import st_inputs as I
from gpu_util import CFG1_MATS, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

DEV = torch.device("cuda:0")


def _rows(mesh, rng, k):
    P = (mesh.n + 1) ** mesh.sdim
    planes = [0, 1, 2, mesh.nt // 2, mesh.nt - 1, mesh.nt]
    fixed = np.concatenate([np.arange(p * P, (p + 1) * P)[:: max(1, P // 400)] for p in planes])
    return np.unique(np.concatenate([fixed, rng.integers(0, mesh.n_nodes, k)]))


@pytest.mark.parametrize("name", ["config2", "config3-shaped-256"])
def test_fullsize_solution_certified_by_oracle_rows(name):
    import paper_2508_09589_b200 as S
    if name == "config2":
        sdim, n, nt, tc, design, src = 2, 256, 256, True, "smooth_tc", ("uniform", 1.0, 0.0, 0.0)
    else:
        sdim, n, nt, tc, design, src = 2, 256, 256, False, "smooth_layers", ("sin", 1.0, 1.0, 2 * np.pi)
    rtol = 1e-8
    solver = S.Solver(sdim, n, nt, mats=CFG1_MATS, source=src, time_constant=tc, rtol=rtol, maxit=500)
    rho = I.design_for(sdim, n, nt, design, 0)
    rd = torch.as_tensor(np.ascontiguousarray(rho), device=DEV)
    prob = O.Problem(O.Mesh(sdim, n, nt), O.Materials(*CFG1_MATS), O.BCs(), O.Source(*src))
    N = prob.mesh.n_nodes
    T = torch.zeros(N, dtype=torch.float64, device=DEV)
    solver.solve(rd, T)
    st = solver.stats()
    assert st["converged"] == 1 and st["rel_residual"] <= rtol
    f = prob.f()
    cons, xD = prob.constraints()
    b = np.where(cons, xD, f)  # T0 = 0: b = f on free rows (R-1)
    bnorm = np.linalg.norm(b)
    rng = np.random.default_rng(5)
    rows = _rows(prob.mesh, rng, 3000)
    Th = T.cpu().numpy()
    r = b[rows] - O.row_apply(prob, rho, Th, rows)
    assert np.max(np.abs(r)) <= rtol * bnorm * (1 + 1e-6), (np.max(np.abs(r)), rtol * bnorm)
    # constrained rows hold the prescribed values exactly
    assert np.array_equal(Th[cons], xD[cons])
    # adjoint of the compliance: K_bc^T lambda = m_f f
    g = prob.compliance_rhs()
    lam = torch.zeros_like(T)
    solver.adjoint(rd, torch.as_tensor(g, device=DEV), lam)
    assert solver.stats()["converged"] == 1
    Lh = lam.cpu().numpy()
    ra = g[rows] - O.row_apply(prob, rho, Lh, rows, transpose=True)
    assert np.max(np.abs(ra)) <= rtol * np.linalg.norm(g) * (1 + 1e-6)
    assert np.all(Lh[cons] == 0.0)
    # sensitivities of sampled elements from the GPU T and lambda
    nsp = n ** sdim
    dJ = torch.empty(nsp if tc else nsp * nt, dtype=torch.float64, device=DEV)
    solver.sensitivity(rd, T, lam, dJ)
    dJh = dJ.cpu().numpy()
    rho_st = np.broadcast_to(rho, (nt,) + rho.shape).copy() if tc else rho
    if tc:
        sp = rng.integers(0, nsp, 24)
        ref = np.array([O.sensitivity_elements(prob, rho_st, Th, Lh, e + nsp * np.arange(nt)).sum() for e in sp])
        got = dJh[sp]
    else:
        el = rng.integers(0, nsp * nt, 3000)
        ref = O.sensitivity_elements(prob, rho_st, Th, Lh, el)
        got = dJh[el]
    assert rel(got, ref) <= 1e-10, rel(got, ref)
    solver.close()
