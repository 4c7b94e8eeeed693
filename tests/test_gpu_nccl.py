"""The NCCL transport of the time-slab path: on one GPU, a single-rank
communicator drives every NCCL entry point libst calls (ncclCommCount / ncclCommUserRank, ncclAllReduce,
ncclAllGather, grouped ncclSend / ncclRecv — to itself) through st_nccl_selftest and checks the values;
with two or more GPUs, one process per GPU solves a time-slab problem over NCCL and matches the oracle
and the single-rank result (skipped on a one-GPU box: ranks sharing a GPU may not wait on each other in
kernels, /opt/skills/guides/B200_PROFILING.md)."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import st_inputs as I
from gpu_util import CFG1_MATS, rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def test_nccl_single_rank_selftest():
    import paper_2508_09589_b200 as S
    torch.cuda.set_device(0)
    uid = S.nccl_unique_id()
    comm = S.nccl_comm_init(uid, 0, 1)
    try:
        assert S.nccl_selftest(comm, 0, 1) == 1
        with pytest.raises(S.StError, match="ranks"):
            S.nccl_selftest(comm, 0, 2)  # a communicator of the wrong size is refused
    finally:
        S.load_library().st_nccl_comm_destroy(comm)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    try:
        import datetime
        import torch
        import torch.distributed as dist
        import paper_2508_09589_b200 as S
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=size, timeout=datetime.timedelta(seconds=180))
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = S.nccl_comm_init(obj[0], rank, size)
        assert S.nccl_selftest(comm, rank, size) == size
        n, nt = 32, 32
        solver = S.Solver(2, n, nt, mats=CFG1_MATS, source=("sin", 1.0, 1.0, 2 * np.pi), rank=rank, size=size,
                          nccl_comm=comm, device=rank, rtol=1e-10, maxit=400, agg_nodes=64, krylov=1, restart=6)
        lay = solver.layout()
        rho = I.design_for(2, n, nt, "smooth_layers", 0)
        dev = torch.device("cuda", rank)
        rd = torch.as_tensor(np.ascontiguousarray(rho[lay["layer0"]:lay["layer0"] + lay["rho_layers"]]), device=dev)
        T = torch.zeros(lay["nodes_local"], dtype=torch.float64, device=dev)
        solver.solve(rd, T)
        lam = torch.zeros_like(T)
        solver.adjoint(rd, None, lam)
        torch.cuda.synchronize()
        q.put(dict(rank=rank, T=T.cpu().numpy(), lam=lam.cpu().numpy(), its=solver.stats()["iterations"]))
        solver.close()
        dist.barrier()
        S.load_library().st_nccl_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put(dict(rank=rank, error=traceback.format_exc()))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (one process per GPU)")
def test_nccl_time_slabs_two_gpus_match_oracle():
    import torch.multiprocessing as mp
    size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            r = q.get(timeout=400)
            assert "error" not in r, r["error"]
            res.append(r)
    finally:
        for p in procs:
            p.join(timeout=5)
            if p.is_alive():
                p.terminate()
    res.sort(key=lambda r: r["rank"])
    rho = I.design_for(2, 32, 32, "smooth_layers", 0)
    prob = O.Problem(O.Mesh(2, 32, 32), O.Materials(*CFG1_MATS), O.BCs(), O.Source("sin", 1.0, 1.0, 2 * np.pi))
    T_ref, lam_ref = prob.solve_both(rho)
    assert rel(np.concatenate([r["T"] for r in res]), T_ref) <= 1e-8
    assert rel(np.concatenate([r["lam"] for r in res]), lam_ref) <= 1e-8
