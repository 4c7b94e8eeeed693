"""Time slabs on one GPU: G ranks, each a process with its own slab of the
space-time grid on cuda:0, exchanging halo planes, Krylov sums and agglomerated coarse levels
through the host-callback transport (torch.distributed gloo). The kernels never wait on each
other: every exchange is a host call. Results are compared with the oracle's direct solution
(north_star tolerances) and with the single-rank iteration count (partition invariance)."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import st_inputs as I
from gpu_util import CFG1_MATS, CFG4_MATS, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, case, q):
    try:
        import torch
        import torch.distributed as dist
        import paper_2508_09589_b200 as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import datetime
        dist.init_process_group("gloo", rank=rank, world_size=size, timeout=datetime.timedelta(seconds=180))
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        sdim, n, nt, mats, T0, src, tau, design, tc, agg, opts = case
        hc = S.TorchHostComm() if size > 1 else None
        solver = S.Solver(sdim, n, nt, mats=mats, T0=T0, source=src, tau=tau, time_constant=tc, rank=rank,
                          size=size, host_comm=hc, rtol=1e-10, maxit=400, agg_nodes=agg, **opts)
        lay = solver.layout()
        rho = I.rho_uniform((n,) * sdim if tc else (nt,) + (n,) * sdim, 0) if design == "uniform" else \
            I.design_for(sdim, n, nt, design, 0)
        prob = O.Problem(O.Mesh(sdim, n, nt, tau=tau), O.Materials(*mats), O.BCs(T0=T0), O.Source(*src))
        P = (n + 1) ** sdim
        p0, npl = lay["plane0"], lay["n_planes"]
        if tc:
            rho_loc = rho
        else:
            rho_loc = rho[lay["layer0"]:lay["layer0"] + lay["rho_layers"]]
        rd = torch.as_tensor(np.ascontiguousarray(rho_loc), device=dev)
        # diagnostics: the eliminated operator and one V-cycle (forward, adjoint) on a seeded vector
        xg = I.rand_vector(prob.mesh.n_nodes, 9)[p0 * P:(p0 + npl) * P]
        xd = torch.as_tensor(xg, device=dev)
        Ax = torch.zeros_like(xd)
        solver.apply(rd, xd, Ax, bc=True)
        Mx = torch.zeros_like(xd)
        solver.vcycle(rd, xd, Mx)
        Mtx = torch.zeros_like(xd)
        solver.vcycle(rd, xd, Mtx, transpose=True)
        T = torch.zeros(npl * P, dtype=torch.float64, device=dev)
        solver.solve(rd, T, allow_nc=True)
        st_f = solver.stats()
        g = prob.compliance_rhs()[p0 * P:(p0 + npl) * P]
        lam = torch.zeros_like(T)
        solver.adjoint(rd, torch.as_tensor(g, device=dev), lam, allow_nc=True)
        st_a = solver.stats()
        nd = n ** sdim * (1 if tc else lay["n_layers"])
        dJ = torch.zeros(nd, dtype=torch.float64, device=dev)
        solver.sensitivity(rd, T, lam, dJ)
        torch.cuda.synchronize()
        # st_design_step with HOST vectors on the slab (side-stream copies, ghost refreshes): the same
        # vectors as the three calls above
        Th, lh, jh = np.zeros(npl * P), np.zeros(npl * P), np.zeros(nd)
        solver.design_step(np.ascontiguousarray(rho_loc).reshape(-1), np.ascontiguousarray(g), Th, lh, jh,
                           allow_nc=True)
        ds = max(rel(Th, T.cpu().numpy()), rel(lh, lam.cpu().numpy()), rel(jh, dJ.cpu().numpy()))
        out = dict(rank=rank, lay=lay, T=T.cpu().numpy(), lam=lam.cpu().numpy(), dJ=dJ.cpu().numpy(), ds=ds,
                   Ax=Ax.cpu().numpy(), Mx=Mx.cpu().numpy(), Mtx=Mtx.cpu().numpy(),
                   its=(st_f["iterations"], st_a["iterations"]), conv=(st_f["converged"], st_a["converged"]))
        solver.close()
        if size > 1:
            dist.barrier()
        dist.destroy_process_group()
        q.put(out)
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(dict(rank=rank, error=traceback.format_exc()))


def _run(case, size):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, case, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            r = q.get(timeout=400)
            assert "error" not in r, r["error"]  # report the first failing rank at once
            res.append(r)
    finally:
        for p in procs:
            p.join(timeout=5)
            if p.is_alive():
                p.terminate()
    return sorted(res, key=lambda r: r["rank"])


CASES = {
    # sdim, n, nt, mats, T0, source, tau, design, time-constant, agg_nodes, options
    "cfg1": (2, 16, 16, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "uniform", False, 64, {}),
    "cfg2-replica": (2, 32, 32, CFG1_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "smooth_tc", True, 64, {}),
    "cfg3-replica": (2, 32, 32, CFG1_MATS, 0.0, ("sin", 1.0, 1.0, 2 * np.pi), 1.0, "smooth_layers", False, 64, {}),
    # the bench's config-3 launch configuration (right-preconditioned GMRES(6), big coarse levels sweeping
    # like the fine one) on slabs
    "cfg3-bench-opts": (2, 32, 32, CFG1_MATS, 0.0, ("sin", 1.0, 1.0, 2 * np.pi), 1.0, "smooth_layers", False, 64,
                        dict(krylov=1, restart=6, nu_fine_nodes=5000)),
    "cfg4-replica": (3, 6, 12, CFG4_MATS, 0.0, ("uniform", 1.0, 0.0, 0.0), 1.0, "smooth_tc", True, 64, {}),
    "T0-cfg4mats": (2, 12, 16, CFG4_MATS, 0.7, ("sin", 1.0, 1.0, 2 * np.pi), 1.0, "uniform", False, 64, {}),
}


@pytest.mark.parametrize("size", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_time_slabs_match_oracle(name, size):
    case = CASES[name]
    sdim, n, nt, mats, T0, src, tau, design, tc, agg, _ = case
    if nt % size:
        pytest.skip("nt not divisible")
    import paper_2508_09589_b200.st as stmod
    try:
        stmod.plan(sdim, n, nt, 0, size, mats=mats, tau=tau, agg_nodes=agg)
    except stmod.StError:
        pytest.skip("the hierarchy does not split over this rank count (DESIGN.md sec. 11)")
    res = _run(case, size)
    ref1 = _run(case, 1)[0]
    # the operator and the preconditioner are the same linear maps on every partition
    for key, tol in (("Ax", 1e-13), ("Mx", 1e-12), ("Mtx", 1e-12)):
        got = np.concatenate([r[key] for r in res])
        assert rel(got, ref1[key]) <= tol, (key, rel(got, ref1[key]))
    assert all(r["ds"] <= 1e-13 for r in res), [r["ds"] for r in res]  # st_design_step == 3 calls
    T = np.concatenate([r["T"] for r in res])
    lam = np.concatenate([r["lam"] for r in res])
    dJ = sum(r["dJ"] for r in res) / size if tc else np.concatenate([r["dJ"] for r in res])
    if tc:  # every rank returns the same globally summed field
        for r in res:
            assert rel(r["dJ"], res[0]["dJ"]) <= 1e-14
    rho = I.rho_uniform((n,) * sdim if tc else (nt,) + (n,) * sdim, 0) if design == "uniform" else \
        I.design_for(sdim, n, nt, design, 0)
    prob = O.Problem(O.Mesh(sdim, n, nt, tau=tau), O.Materials(*mats), O.BCs(T0=T0), O.Source(*src))
    T_ref, lam_ref = prob.solve_both(rho)
    dJ_ref = prob.sensitivity(rho, T_ref, lam_ref)
    assert all(r["conv"] == (1, 1) for r in res)
    assert rel(T, T_ref) <= 1e-8, rel(T, T_ref)
    assert rel(lam, lam_ref) <= 1e-8, rel(lam, lam_ref)
    assert rel(dJ.reshape(dJ_ref.shape), dJ_ref) <= 1e-7, rel(dJ.reshape(dJ_ref.shape), dJ_ref)
    # partition invariance of the method: the same iteration counts as one rank (+-1: rounding order)
    assert abs(res[0]["its"][0] - ref1["its"][0]) <= 1 and abs(res[0]["its"][1] - ref1["its"][1]) <= 1, \
        (res[0]["its"], ref1["its"])


def _design_worker(rank, size, port, q):
    """Config-5 loop (3 OC iterations, 16^2 x 16 replica) on `size` time slabs."""
    try:
        import datetime
        import torch
        import torch.distributed as dist
        import paper_2508_09589_b200 as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=size, timeout=datetime.timedelta(seconds=180))
        torch.cuda.set_device(0)
        hc = S.TorchHostComm() if size > 1 else None
        solver = S.Solver(2, 16, 16, mats=CFG1_MATS, rank=rank, size=size, host_comm=hc, rtol=1e-11, maxit=400,
                          agg_nodes=64)
        lay = solver.layout()
        # the design kernels on slabs, one at a time, on seeded global fields
        a = np.random.default_rng(3).uniform(0.1, 1.0, (16, 16, 16))
        g = -np.random.default_rng(4).uniform(1e-6, 1e-3, (16, 16, 16))
        l0, nl = lay["layer0"], lay["n_layers"]
        ad = torch.as_tensor(np.ascontiguousarray(a[l0:l0 + nl]).reshape(-1), device="cuda:0")
        gd = torch.as_tensor(np.ascontiguousarray(g[l0:l0 + nl]).reshape(-1), device="cuda:0")
        fa = torch.empty(lay["rho_layers"] * 256, dtype=torch.float64, device="cuda:0")
        solver.filter(ad, fa)
        fta = torch.empty_like(gd)
        solver.filter(gd, fta, transpose=True)
        oc = torch.empty_like(ad)
        lam_oc = solver.oc_update(ad, gd, oc)
        rho = torch.full((nl * 256,), 0.4, dtype=torch.float64, device="cuda:0")
        hist = S.design_loop(solver, rho, 3)
        out = dict(rank=rank, rho=rho.cpu().numpy(), hist=hist, fa=fa.cpu().numpy(), fta=fta.cpu().numpy(),
                   oc=oc.cpu().numpy(), lam_oc=lam_oc, l0=l0, nl=nl, rl=lay["rho_layers"])
        solver.close()
        if size > 1:
            dist.barrier()
        dist.destroy_process_group()
        q.put(out)
    except Exception:  # noqa: BLE001
        import traceback
        q.put(dict(rank=rank, error=traceback.format_exc()))


def test_config5_design_loop_on_slabs():
    """The config-5 loop (density filter across slab boundaries, global OC volume, ...) on 2 slabs
    gives the oracle's designs and compliance history (R-13, sec. 11)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_design_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            res.append(qq.get(timeout=400))
        errs = [r["error"] for r in res if "error" in r]
        assert not errs, "\n".join(errs)
    finally:
        for p in procs:
            p.join(timeout=5)
            if p.is_alive():
                p.terminate()
    res.sort(key=lambda r: r["rank"])
    a = np.random.default_rng(3).uniform(0.1, 1.0, (16, 16, 16))
    g = -np.random.default_rng(4).uniform(1e-6, 1e-3, (16, 16, 16))
    Fa, Fta = O.density_filter(a), O.density_filter(g, transpose=True)
    oc_ref, lam_ref = O.oc_update(a, g)
    for r in res:
        l0, nl, rl = r["l0"], r["nl"], r["rl"]
        assert rel(r["fa"].reshape(rl, 16, 16), Fa[l0:l0 + rl]) <= 1e-14, ("F", r["rank"])
        assert rel(r["fta"].reshape(nl, 16, 16), Fta[l0:l0 + nl]) <= 1e-14, ("F^T", r["rank"])
        assert abs(r["lam_oc"] - lam_ref) <= 1e-10 * lam_ref, ("Lambda", r["rank"], r["lam_oc"], lam_ref)
        assert rel(r["oc"].reshape(nl, 16, 16), oc_ref[l0:l0 + nl]) <= 1e-12, ("OC", r["rank"])
    prob = O.Problem(O.Mesh(2, 16, 16), O.Materials(*CFG1_MATS), O.BCs(), O.Source())
    designs, hist = O.design_loop(prob, np.full((16, 16, 16), 0.4), 3)
    for r in res:
        assert np.allclose(r["hist"], hist, rtol=1e-9), (r["hist"], hist)
    rho = np.concatenate([r["rho"] for r in res]).reshape(16, 16, 16)
    assert rel(rho, designs[-1]) <= 1e-7, rel(rho, designs[-1])
