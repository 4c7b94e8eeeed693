"""st_design_step vs three calls, device and pinned-host vectors (config 2 or the 512^2 x 512 slab)."""
import sys, time
import numpy as np
import torch
import paper_2508_09589_b200 as S
import st_inputs as I

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
if cfg == "2":
    s = S.Solver(2, 256, 256, time_constant=True)
    rho = I.design_for(2, 256, 256, "smooth_tc", 0).reshape(-1)
else:
    s = S.Solver(2, 512, 512, time_constant=False, source=("sin", 1.0, 1.0, 2 * np.pi))
    rho = I.design_for(2, 512, 512, "smooth_layers", 0).reshape(-1)
N = s.n_nodes
pin = lambda n: torch.zeros(n, dtype=torch.float64).pin_memory().numpy()
rh = pin(rho.size); rh[:] = rho
Th, lh, jh = pin(N), pin(N), pin(rho.size)
rd = torch.as_tensor(rho, device="cuda")
Td, ld, jd = (torch.zeros(N, dtype=torch.float64, device="cuda") for _ in range(2)), None, None
Td = torch.zeros(N, dtype=torch.float64, device="cuda"); ld = torch.zeros_like(Td); jd = torch.zeros_like(rd)


def t(f, reps=3):
    out = []
    for k in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(k); torch.cuda.synchronize(); out.append((time.perf_counter() - t0) * 1e3)
    return ["%.1f" % x for x in out]


def flip(k, r):
    if k > 0:
        np.subtract(1.01, r, out=r) if isinstance(r, np.ndarray) else torch.sub(1.01, r, out=r)


def three(k, r, T, l, j):
    flip(k, r); T[:] = 0; l[:] = 0
    s.solve(r, T); s.adjoint(r, None, l); s.sensitivity(r, T, l, j)


def fused(k, r, T, l, j):
    flip(k, r); T[:] = 0; l[:] = 0
    fs, as_ = s.design_step(r, None, T, l, j, allow_nc=True)
    if not (fs["converged"] and as_["converged"]):
        print("NOT CONVERGED", k, fs, as_)


print("device three", t(lambda k: three(k, rd, Td, ld, jd)))
print("device fused", t(lambda k: fused(k, rd, Td, ld, jd)))
print("host   three", t(lambda k: three(k, rh, Th, lh, jh)))
print("host   fused", t(lambda k: fused(k, rh, Th, lh, jh)))
x = torch.empty(N, dtype=torch.float64, device="cuda")
print("H2D %d MB" % (8 * N // 2**20), t(lambda k: x.copy_(torch.from_numpy(Th), non_blocking=True)))
print("D2H", t(lambda k: torch.from_numpy(Th).copy_(x, non_blocking=True)))
print("host fused again", t(lambda k: fused(k, rh, Th, lh, jh)))
print("stats", s.stats())
