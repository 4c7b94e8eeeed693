"""Development sweep: outer iterations and solve time vs smoother settings (config 2)."""
import sys, os, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import st_inputs as I
import paper_2508_09589_b200 as S
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
if cfg == "2":
    sdim, n, nt, tc, design, src = 2, 256, 256, True, "smooth_tc", ("uniform", 1.0, 0.0, 0.0)
else:
    sdim, n, nt, tc, design, src = 2, 256, 256, False, "smooth_layers", ("sin", 1.0, 1.0, 6.283185307179586)
rho = torch.as_tensor(I.design_for(sdim, n, nt, design, 0), device=dev).contiguous()
res = []
for nu, om, cmax, m in [(2, 0.6, 400, 30), (3, 0.7, 400, 30), (3, 0.8, 400, 30), (4, 0.7, 400, 30), (4, 0.8, 400, 30),
                         (3, 0.75, 400, 16), (4, 0.75, 400, 16), (3, 0.75, 400, 12), (5, 0.75, 400, 30), (6, 0.75, 400, 30)]:
    s = S.Solver(sdim, n, nt, time_constant=tc, source=src, stream=stream.cuda_stream, rtol=1e-8, maxit=300,
                 nu_pre=nu, nu_post=nu, omega=om, coarse_max_nodes=cmax, restart=m)
    T = torch.zeros(s.n_nodes, dtype=torch.float64, device=dev)
    f = torch.empty_like(T)
    with torch.cuda.stream(stream):
        s.rhs(rho, f, None)
        out = {}
        for rep in range(2):
            T.zero_()
            rc = s.solve(rho, T, allow_nc=True)
            a = s.stats()
            lam = torch.zeros_like(T)
            s.adjoint(rho, f, lam, allow_nc=True)
            b = s.stats()
        out = dict(nu=nu, omega=om, cmax=cmax, m=m, fwd_its=a["iterations"], fwd_ms=round(a["solve_ms"], 2),
                   adj_its=b["iterations"], adj_ms=round(b["solve_ms"], 2), levels=len(s.hierarchy()),
                   conv=(a["converged"], b["converged"]))
    print(json.dumps(out), flush=True)
    s.close()
