"""Time-slab host logic on CPU (no GPU): the partition plan of every level (st_plan, the same code
st_setup runs) and the host-callback transport over torch.distributed with gloo, world size 2.

DESIGN.md sec. 11: rank r owns element layers [r nt/G, (r+1) nt/G) and node planes
(r nt/G, (r+1) nt/G] (rank 0 also plane 0); a slab level holds one ghost layer (the next slab's
first) except on the last rank; the first replicated level must still split into G slabs."""
import ctypes
import os
import socket

import numpy as np
import pytest

import paper_2508_09589_b200 as S
from paper_2508_09589_b200 import st

CFG1 = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)


@pytest.mark.parametrize("shape", [(2, 16, 16), (2, 64, 64), (2, 256, 256), (2, 1024, 1024), (3, 64, 128),
                                   (2, 512, 4096)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_slab_plan_partitions_every_distributed_level(shape, G):
    sdim, n, nt = shape
    ref = st.plan(sdim, n, nt, 0, 1, mats=CFG1, tau=nt / 512 if nt == 4096 else 1.0)
    plans = [st.plan(sdim, n, nt, r, G, mats=CFG1, tau=nt / 512 if nt == 4096 else 1.0) for r in range(G)]
    # same hierarchy as one rank (Algorithm 1 runs on the global grid)
    for p in plans:
        assert [(L["n"], L["nt"], L["kind"]) for L in p["levels"]] == \
               [(L["n"], L["nt"], L["kind"]) for L in ref["levels"]]
        assert p["n_dist"] == plans[0]["n_dist"]
    nd = plans[0]["n_dist"]
    assert (nd >= 1) == (G > 1) and not plans[0]["levels"][-1]["dist"]  # coarsest replicated
    # owned fine planes partition [0, nt]
    planes = sorted((p["plane0"], p["n_planes"]) for p in plans)
    nxt = 0
    for p0, cnt in planes:
        assert p0 == nxt and cnt >= 1
        nxt = p0 + cnt
    assert nxt == nt + 1
    for l in range(len(ref["levels"])):
        Ls = [p["levels"][l] for p in plans]
        if l < nd:
            assert all(L["dist"] for L in Ls)
            ntl = Ls[0]["nt"]
            assert ntl % G == 0
            # owned layers partition [0, nt_l); local layers = owned + the next slab's first layer
            assert [L["layer0"] for L in Ls] == [r * ntl // G for r in range(G)]
            assert all(L["n_layers"] == ntl // G for L in Ls)
            assert [L["local_layers"] for L in Ls] == [ntl // G + (1 if r < G - 1 else 0) for r in range(G)]
        else:
            assert not any(L["dist"] for L in Ls)
            assert all(L["local_layers"] == L["nt"] for L in Ls)
            if l == nd and G > 1:
                assert Ls[0]["nt"] % G == 0  # gathered from slab form


def test_slab_plan_rejects_indivisible_time_extent():
    with pytest.raises(st.StError):
        st.plan(2, 16, 18, 0, 4, mats=CFG1)


# ---- world size 2 with gloo: the TorchHostComm callbacks used by ST_COMM_HOST -------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=size)
        hc = S.TorchHostComm()
        n = 7
        # sendrecv with the neighbour: each sends its rank-tagged vector
        send = (np.arange(n, dtype=np.float64) + 100.0 * rank)
        recv = np.zeros(n)
        peer = 1 - rank
        DP = ctypes.POINTER(ctypes.c_double)
        rc1 = hc.struct.sendrecv(None, peer, send.ctypes.data_as(DP), recv.ctypes.data_as(DP), n)
        ok1 = rc1 == 0 and np.array_equal(recv, np.arange(n) + 100.0 * peer)
        # allreduce (sum) in place
        buf = np.full(3, rank + 1.0)
        rc2 = hc.struct.allreduce_sum(None, buf.ctypes.data_as(DP), 3)
        ok2 = rc2 == 0 and np.array_equal(buf, np.full(3, 3.0))
        # allgather in rank order
        out = np.zeros(2 * n)
        rc3 = hc.struct.allgather(None, send.ctypes.data_as(DP), out.ctypes.data_as(DP), n)
        ok3 = rc3 == 0 and np.array_equal(out, np.concatenate([np.arange(n), np.arange(n) + 100.0]))
        # the plans of the two ranks agree on the slab boundary: rank 0's ghost layer is rank 1's first
        p = st.plan(2, 32, 32, rank, size, mats=CFG1)
        mine = np.array([p["levels"][0]["layer0"], p["levels"][0]["n_layers"], p["plane0"], p["n_planes"]], float)
        other = np.zeros(4)
        hc.struct.sendrecv(None, peer, mine.ctypes.data_as(DP), other.ctypes.data_as(DP), 4)
        lo, hi = (mine, other) if rank == 0 else (other, mine)
        ok4 = lo[0] + lo[1] == hi[0] and lo[2] + lo[3] == hi[2] and hi[2] + hi[3] == 33
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok1, ok2, ok3, ok4))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_host_transport_world_size_2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5 and all(r[1:]), r
