"""ncu / timing target: a level operator kernel (bench_op) of a config-shaped problem.
usage: prof_op.py MODE LEVEL [SDIM N NT tc|tv [c4]] [option=value ...]   (st_options_t fields)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import st_inputs as I
import paper_2508_09589_b200 as S
a = [x for x in sys.argv[1:] if "=" not in x]
kv = dict(x.split("=", 1) for x in sys.argv[1:] if "=" in x)
mode = int(a[0]) if len(a) > 0 else 2
level = int(a[1]) if len(a) > 1 else 0
sdim = int(a[2]) if len(a) > 2 else 2
n = int(a[3]) if len(a) > 3 else 256
nt = int(a[4]) if len(a) > 4 else n
tc = (a[5] != "tv") if len(a) > 5 else True
mats = (0.1, 1.0, 1.0, 1e-4, 1.0, 3.0) if (len(a) > 6 and a[6] == "c4") else (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)
opts = dict(krylov=1, restart=2)  # small Krylov pool: hooks only
opts.update({k: (float(v) if "." in v or "e" in v else int(v)) for k, v in kv.items()})
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
s = S.Solver(sdim, n, nt, mats=mats, time_constant=tc, stream=st.cuda_stream, **opts)
rho = torch.as_tensor(I.design_for(sdim, n, nt, "smooth_tc" if tc else "smooth_layers", 0), device=dev).contiguous().reshape(-1)
H = s.hierarchy()
N = H[level]["nodes"]
with torch.cuda.stream(st):
    s.rhs(rho, None, None)            # rho-dependent setup (coarse levels, weights)
    s.bench_op(rho, level, mode, 3)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); s.bench_op(rho, level, mode, 10); e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 10 * 1e3
print(f"{' '.join(sys.argv[1:])}: us per launch {us:.2f} nodes {N} -> {32 * N / us / 1e3:.0f} GB/s (32 B/node); "
      f"rho setup {s.stats()['setup_ms']:.2f} ms; level {level}: {H[level]['n']}^{sdim} x {H[level]['nt']} {H[level]['kind']}")
