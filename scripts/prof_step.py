"""Profiling probe: one bench step (rho setup + forward + adjoint + sensitivities) of a bench.py
workload, after one warm-up step; the profiled step is bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` captures exactly one step's launch list.

    python scripts/prof_step.py CONFIG [maxit]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_09589_b200 as S  # noqa: E402
import st_inputs as I  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = bench.WORKLOADS[cfg]
dev = torch.device("cuda:0")
s = S.Solver(wl["sdim"], wl["n"], wl["nt"], mats=wl["mats"], source=wl["source"], tau=wl["tau"],
             time_constant=wl["tc"], rtol=1e-8, maxit=maxit, **wl["opts"])
rho = torch.as_tensor(np.ascontiguousarray(I.design_for(wl["sdim"], wl["n"], wl["nt"], wl["design"], 0)),
                      device=dev).reshape(-1)
T = torch.zeros(s.n_nodes, dtype=torch.float64, device=dev)
lam = torch.zeros_like(T)
nsp = wl["n"] ** wl["sdim"]
dJ = torch.empty(nsp if wl["tc"] else nsp * wl["nt"], dtype=torch.float64, device=dev)


def step():
    T.zero_(); lam.zero_()
    s.solve(rho, T, allow_nc=True)
    a = s.stats()
    s.adjoint(rho, None, lam, allow_nc=True)
    b = s.stats()
    s.sensitivity(rho, T, lam, dJ)
    return a, b


step()
torch.sub(1.01, rho, out=rho)  # a new design: the profiled step includes the rho setup
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
a, b = step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", round(time.perf_counter() - t0, 3), "s", a["iterations"], b["iterations"], a["vcycles"], b["vcycles"])
