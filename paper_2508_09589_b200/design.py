"""Config-5 design loop (BASELINE configs[4]; R-13): density filter -> forward solve ->
compliance adjoint -> sensitivities -> filter transpose -> optimality-criteria update, every step
a libst call (st_filter, st_solve, st_adjoint, st_sensitivity, st_oc_update, st_dot) on device
tensors. Driver level: not the paper's method (PDE filter, projection, MMA).
Works on one GPU or on time slabs (rank-local owned layers / planes)."""
from __future__ import annotations


def design_loop(solver, rho, iterations, volfrac=0.4, radius=2.0, move=0.2, rho_min=1e-3, callback=None):
    """Run `iterations` OC steps from the design `rho` (this rank's owned element layers, updated in
    place). Returns the compliance history phi = f^T T (one value per iteration)."""
    import torch
    lay = solver.layout()
    dev = rho.device
    nsp = rho.numel() // max(1, lay["n_layers"] if lay["rho_layers"] else 1)
    rt = torch.empty(nsp * (lay["rho_layers"] or 1), dtype=torch.float64, device=dev)
    T = torch.zeros(lay["nodes_local"], dtype=torch.float64, device=dev)
    lam = torch.zeros_like(T)
    f = torch.empty_like(T)
    dJt = torch.empty_like(rho)
    dJ = torch.empty_like(rho)
    new = torch.empty_like(rho)
    hist = []
    for it in range(iterations):
        solver.filter(rho, rt, transpose=False, radius=radius)
        if it == 0:
            solver.rhs(rt, f, None)
        solver.solve(rt, T)                       # warm start from the previous design
        hist.append(solver.dot(f, T))
        solver.adjoint(rt, f, lam)
        solver.sensitivity(rt, T, lam, dJt)
        solver.filter(dJt, dJ, transpose=True, radius=radius)
        solver.oc_update(rho, dJ, new, volfrac=volfrac, move=move, rho_min=rho_min)
        rho.copy_(new)
        if callback is not None:
            callback(it, hist[-1])
    return hist
