"""Debug: convergence of small replicas under smoother / graph settings."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import st_inputs as I
import paper_2508_09589_b200 as S
dev = torch.device("cuda:0")
CFG1 = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0); CFG4 = (0.1, 1.0, 1.0, 1e-4, 1.0, 3.0)
cases = [("cfg2-rep", 2, 32, 32, CFG1, True, "smooth_tc"), ("cfg4-rep", 3, 6, 12, CFG4, True, "smooth_tc"),
         ("cfg4-16", 3, 16, 32, CFG4, True, "smooth_tc"), ("cfg2-256", 2, 256, 256, CFG1, True, "smooth_tc"),
         ("cfg3-256", 2, 256, 256, CFG1, False, "smooth_layers"), ("cfg4-64", 3, 64, 128, CFG4, True, "smooth_tc")]
for name, sd, n, nt, mats, tc, design in cases:
    rho = torch.as_tensor(np.ascontiguousarray(I.design_for(sd, n, nt, design, 0)), device=dev)
    for opts in [dict(), dict(omega=0.8), dict(nu_pre=2, nu_post=2), dict(nu_pre=4, nu_post=4)]:
        for fast in ("0",):
            os.environ["ST_NO_FAST"] = fast
            s = S.Solver(sd, n, nt, mats=mats, time_constant=tc, rtol=1e-10, maxit=200, **opts)
            T = torch.zeros(s.n_nodes, dtype=torch.float64, device=dev)
            s.solve(rho, T, allow_nc=True)
            st = s.stats()
            print(json.dumps(dict(case=name, opts=opts, generic=fast == "1", its=st["iterations"],
                                  conv=st["converged"], rel=st["rel_residual"], ms=st["solve_ms"],
                                  om=[round(h["omega"], 3) for h in s.hierarchy()],
                                  R=[round(h["lam_max"], 2) for h in s.hierarchy()])), flush=True)
            s.close()
