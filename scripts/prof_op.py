"""ncu target: config-2 fine-level operator kernel (bench_op) in a given mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import st_inputs as I
import paper_2508_09589_b200 as S
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256
tc = (sys.argv[4] != "tv") if len(sys.argv) > 4 else True
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
s = S.Solver(2, n, n, time_constant=tc, stream=st.cuda_stream)
rho = torch.as_tensor(I.rho_smooth((n, n), 0) if tc else I.rho_uniform((n, n, n), 0), device=dev)
H = s.hierarchy()
N = H[level]["nodes"]
x = torch.rand(N, dtype=torch.float64, device=dev); b = torch.rand_like(x); y = torch.empty_like(x)
with torch.cuda.stream(st):
    s.bench_op(rho, level, mode, 3)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); s.bench_op(rho, level, mode, 10); e1.record(st)
torch.cuda.synchronize()
print("us per launch", e0.elapsed_time(e1) / 10 * 1e3, "nodes", N)
