"""Per-level damped-Jacobi sweep time (us per launch, 50 back-to-back eager launches) of a config-shaped
hierarchy for each (2+1)D kernel family: TMA ring (default), cp.async ring, generic.
usage: level_lat.py [N NT tc|tv]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import st_inputs as I
import paper_2508_09589_b200 as S
a = sys.argv[1:]
n = int(a[0]) if a else 256
nt = int(a[1]) if len(a) > 1 else n
tc = (a[2] != "tv") if len(a) > 2 else True
dev = torch.device("cuda:0")
rho = torch.as_tensor(I.design_for(2, n, nt, "smooth_tc" if tc else "smooth_layers", 0), device=dev).contiguous()
res = {}
for name, nf, fk in (("tma", "0", "0"), ("cpasync", "0", "1"), ("generic", "1", "0")):
    os.environ["ST_NO_FAST"], os.environ["ST_FAST_KIND"] = nf, fk
    st = torch.cuda.Stream()
    s = S.Solver(2, n, nt, time_constant=tc, stream=st.cuda_stream)
    H = s.hierarchy()
    with torch.cuda.stream(st):
        s.rhs(rho, None, None)
        for l in range(1, len(H) - 1):
            s.bench_op(rho, l, 2, 5)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st); s.bench_op(rho, l, 2, 50); e1.record(st)
            torch.cuda.synchronize()
            res.setdefault(l, {"nodes": H[l]["nodes"]})[name] = e0.elapsed_time(e1) / 50 * 1e3
    s.close()
print("level nodes " + " ".join(f"{k:>8s}" for k in ("tma", "cpasync", "generic")))
for l, r in res.items():
    print(f"{l:5d} {r['nodes']:9d} " + " ".join(f"{r[k]:8.2f}" for k in ("tma", "cpasync", "generic")))
