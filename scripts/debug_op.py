"""Debug: locate rows where the masked operator differs from the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O, st_inputs as I
from gpu_util import make_pair, CFG1_MATS
n, nt = int(sys.argv[1]), int(sys.argv[2])
solver, prob = make_pair(2, n, nt, mats=CFG1_MATS, time_constant=True)
rho = I.design_for(2, n, nt, "smooth_tc", 0)
Kbc, _, _, _ = prob.system(rho)
x = I.rand_vector(prob.mesh.n_nodes, 1)
dev = torch.device("cuda:0")
y = torch.empty(prob.mesh.n_nodes, dtype=torch.float64, device=dev)
for trans in (False, True):
    solver.apply(torch.as_tensor(rho, device=dev), torch.as_tensor(x, device=dev), y, transpose=trans, bc=True)
    ref = (Kbc.T if trans else Kbc) @ x
    d = np.abs(y.cpu().numpy() - ref)
    bad = np.nonzero(d > 1e-12 * np.abs(ref).max())[0]
    nn = n + 1
    print("trans", trans, "bad rows", len(bad))
    for b in bad[:20]:
        p, rem = divmod(b, nn * nn); j, i = divmod(rem, nn)
        print(f"  p={p} j={j} i={i} gpu={y[b].item():.6e} ref={ref[b]:.6e}")
