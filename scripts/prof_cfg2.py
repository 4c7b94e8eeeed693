"""Profiling probe: config-2 setup + one forward solve (kernel launch list under ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import st_inputs as I
import paper_2508_09589_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
s = S.Solver(2, n, n, time_constant=True, rtol=1e-8, maxit=maxit)
rho = torch.as_tensor(I.rho_smooth((n, n), 0), device=dev)
T = torch.zeros(s.n_nodes, dtype=torch.float64, device=dev)
s.solve(rho, T, allow_nc=True)
x = torch.rand(s.n_nodes, dtype=torch.float64, device=dev); y = torch.empty_like(x)
for _ in range(3): s.apply(rho, x, y)
torch.cuda.synchronize()
print("ok", s.stats())
