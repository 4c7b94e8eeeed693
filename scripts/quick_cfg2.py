"""Quick timing probe of config 2 (not the bench; development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import st_inputs as I
import paper_2508_09589_b200 as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device("cuda:0")
s = S.Solver(2, n, n, time_constant=True, rtol=1e-8)
print(s.hierarchy())
rho = torch.as_tensor(I.rho_smooth((n, n), 0), device=dev)
T = torch.zeros(s.n_nodes, dtype=torch.float64, device=dev)
f = torch.empty_like(T); b = torch.empty_like(T)
s.rhs(rho, f, b)
for rep in range(3):
    T.zero_()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.solve(rho, T)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st = s.stats()
    print(f"solve: {1e3*(t1-t0):.1f} ms wall, its {st['iterations']}, rel {st['rel_residual']:.2e}, solve_ms {st['solve_ms']:.1f} setup_ms {st['setup_ms']:.1f}")
    lam = torch.zeros_like(T)
    g = f.clone()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.adjoint(rho, g, lam)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st = s.stats()
    print(f"adjoint: {1e3*(t1-t0):.1f} ms, its {st['iterations']}, rel {st['rel_residual']:.2e}")
# operator apply timing
x = torch.rand(s.n_nodes, dtype=torch.float64, device=dev); y = torch.empty_like(x)
for _ in range(3): s.apply(rho, x, y)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
for _ in range(20): s.apply(rho, x, y)
torch.cuda.synchronize(); t1 = time.perf_counter()
dt = (t1 - t0) / 20
print(f"apply (wall incl. ABI overhead): {dt*1e3:.3f} ms -> {16*s.n_nodes/dt/1e9:.0f} GB/s algorithmic")
