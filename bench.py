#!/usr/bin/env python
"""bench.py — driver benchmark of the all-at-once space-time solve (arxiv 2508.09589 hot path).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One STEP = one pass of the whole hot path on a fresh synthetic design:
rho-dependent setup (Galerkin coarse operators, coarsest inverse, RHS), forward FGMRES+MG
solve to true-residual rtol 1e-8 from T = 0, adjoint solve of the time-integrated thermal
compliance (dJ/dT = f), element sensitivities. Workload at N = 1: BASELINE config 2
(configs[1]): (2+1)D 256^2 x 256 elements, 16,974,593 space-time DOFs, time-constant smooth
design. value = 2 N_n (forward + adjoint DOFs solved) per step time, summed over ranks.
For N > 1 the space-time grid is split into N time slabs (one per GPU, NCCL over NVLink:
halo planes, Krylov sums, agglomerated coarse levels) and the time extent
grows with N (weak scaling in time, as BASELINE config 5): 256^2 x 256N elements, tau = N, the
config-2 design; every rank holds a config-2-sized slab.
Inputs are resident in HBM before the timed region; L2 is flushed (256 MB write) between
steps. `e2e` repeats the step through the C ABI with pinned HOST buffers (copies inside).
`--impl reference` times the CPU oracle (oracle/, SuperLU direct) on a bounded replica.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG1_MATS = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)
CFG4_MATS = (0.1, 1.0, 1.0, 1e-4, 1.0, 3.0)
WORKLOADS = {
    2: dict(name="config2: (2+1)D 256^2x256 elements, time-constant smooth rho (sigma 3, [0.01,1]), "
                 "k=1e-3+rho^3(1-1e-3), c=1, Q=1, T=0 sink patch (10% of x1=0), T0=0",
            sdim=2, n=256, nt=256, mats=CFG1_MATS, tc=True, design="smooth_tc", source=("uniform", 1.0, 0.0, 0.0),
            tau=1.0),
    1: dict(name="config1: (2+1)D 16^3, rho~U[0.1,1] space-time", sdim=2, n=16, nt=16, mats=CFG1_MATS, tc=False,
            design="uniform", source=("uniform", 1.0, 0.0, 0.0), tau=1.0),
    4: dict(name="config4: (3+1)D 64^3x128, time-constant smooth rho, c=0.1+0.9rho, k_min=1e-4", sdim=3, n=64,
            nt=128, mats=CFG4_MATS, tc=True, design="smooth_tc", source=("uniform", 1.0, 0.0, 0.0), tau=1.0),
    5: dict(name="config5 (per GPU): (2+1)D 512^2x512, space-time design; a step = one OC design iteration "
                 "(density filter r=2, forward, adjoint, sensitivities, filter^T, OC volfrac 0.4) from rho=0.4",
            sdim=2, n=512, nt=512, mats=CFG1_MATS, tc=False, design="const", source=("uniform", 1.0, 0.0, 0.0),
            tau=1.0),
    3: dict(name="config3-shaped (1/8 of config 3 on one GPU): (2+1)D 512^2x512, an independent smooth field per "
                 "time layer, Q(t) = 1 + sin(2 pi t)", sdim=2, n=512, nt=512, mats=CFG1_MATS, tc=False,
            design="smooth_layers", source=("sin", 1.0, 1.0, 6.283185307179586), tau=1.0),
}
METRIC = "space-time DOFs solved/sec (FGMRES+MG to rtol 1e-8) & operator GB/s vs HBM peak"


def solver_opts(args):
    o = dict(smoother=2 if args.smoother == "gmres" else 0)
    nu = args.nu or (10 if args.smoother == "gmres" else 0)  # 0: the library defaults
    if nu:
        o["nu_pre"] = o["nu_post"] = nu
    if args.nu_coarse >= 0:
        o["nu_coarse"] = args.nu_coarse
    if args.omega > 0:
        o["omega"] = args.omega
    if args.restart > 0:
        o["restart"] = args.restart
    if args.full_coarsening:
        o["full_coarsening"] = 1
    return o


def precond_desc(args, solver):
    o = solver.options()
    sm = ("GMRES(%d)-Jacobi smoother" % o["nu_pre"] if args.smoother == "gmres" else
          "damped Jacobi %d+%d sweeps on the fine level, %d+%d on the coarse levels"
          % (o["nu_pre"], o["nu_post"], o["nu_coarse"] or o["nu_pre"], o["nu_coarse"] or o["nu_post"]))
    return "FGMRES(%d) + V-cycle, %s, %s" % (o["restart"], sm, "full space-time coarsening" if args.full_coarsening
                                             else "semi-coarsening (Algorithm 1)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--smoother", default="jacobi", choices=["jacobi", "gmres"],
                    help="jacobi: damped Jacobi nu+nu (default); gmres: the paper's GMRES(nu)-Jacobi smoother")
    ap.add_argument("--nu", type=int, default=0,
                    help="fine-level Jacobi sweeps / GMRES steps (default: the library's 2 for jacobi, 10 for gmres)")
    ap.add_argument("--nu-coarse", type=int, default=-1,
                    help="Jacobi sweeps on the coarse levels (default: the library's 5; 0 = --nu)")
    ap.add_argument("--full-coarsening", action="store_true", help="the paper's full space-time coarsening")
    ap.add_argument("--omega", type=float, default=0.0, help="Jacobi weight cap (default: the library's 0.75)")
    ap.add_argument("--restart", type=int, default=0, help="FGMRES restart length (default: the library's 16)")
    ap.add_argument("--cpu-worker", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--cpu-reps", type=int, default=1, help=argparse.SUPPRESS)
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
# CPU oracle timing (the reference arm and cpu_baseline): a bounded replica of the workload
def oracle_step_seconds(n: int, reps: int = 1):
    import numpy as np
    import oracle as O
    import st_inputs as I
    mats = O.Materials(*CFG1_MATS)
    mesh = O.Mesh(2, n, n)
    prob = O.Problem(mesh, mats, O.BCs(), O.Source())
    times = []
    for r in range(reps):
        rho = I.rho_smooth((n, n), seed=r)
        t0 = time.perf_counter()
        T, lam = prob.solve_both(rho)            # assembly + SuperLU factorisation + fwd + adj
        prob.sensitivity(rho, T, lam)
        times.append(time.perf_counter() - t0)
    return mesh.n_nodes, times


def cpu_worker(n: int, reps: int):
    dofs, times = oracle_step_seconds(n, reps)
    print(json.dumps({"dofs": dofs, "times": times}))


def run_cpu_subprocess(n: int, reps: int):
    env = dict(os.environ)
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
        env[k] = "1"
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-worker", str(n), "--cpu-reps", str(reps)],
                         capture_output=True, text=True, env=env, timeout=900)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode != 0 or not line:
        raise RuntimeError(out.stderr[-2000:])
    return json.loads(line[-1])


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(k)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
def run_cuda(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import st_inputs as I
    import paper_2508_09589_b200 as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    wl = dict(WORKLOADS[args.config])
    nccl_comm = None
    if world > 1:  # time slabs over NCCL: the time extent grows with the GPU count
        wl["nt"] = wl["nt"] * world
        wl["tau"] = wl["tau"] * world
        wl["name"] = wl["name"] + f" extended in time to nt={wl['nt']}, tau={wl['tau']:g} (time slabs)"
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_comm = S.nccl_comm_init(obj[0], rank, world)
    solver = S.Solver(wl["sdim"], wl["n"], wl["nt"], mats=wl["mats"], source=wl["source"], tau=wl["tau"],
                      time_constant=wl["tc"], stream=stream.cuda_stream, device=local, rtol=args.rtol, maxit=1000,
                      rank=rank, size=world, nccl_comm=nccl_comm, **solver_opts(args))
    N = solver.n_nodes            # this rank's owned nodes
    nd = solver.n_design
    N_global = (wl["n"] + 1) ** wl["sdim"] * (wl["nt"] + 1)
    nsteps = args.warmup + args.steps
    # time-constant designs are replicated on every rank (same seed); the config-5 design is uniform
    lay = solver.layout()
    sl = slice(None) if wl["tc"] else slice(lay["layer0"], lay["layer0"] + lay["rho_layers"])  # this rank's layers
    rhos = [torch.as_tensor(np.ascontiguousarray(I.design_for(wl["sdim"], wl["n"], wl["nt"], wl["design"], seed=s)[sl]),
                            device=dev) for s in range(nsteps)] if wl["design"] != "const" else \
        [torch.full((nd,), 0.4 + 0.01 * s, dtype=torch.float64, device=dev) for s in range(nsteps)]
    T = torch.zeros(N, dtype=torch.float64, device=dev)
    lam = torch.zeros_like(T)
    f = torch.empty_like(T)
    dJ = torch.empty(nd, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    with torch.cuda.stream(stream):
        solver.rhs(rhos[0], f, None)
    its = []

    design = args.config == 5  # a step is one config-5 design iteration (R-13)
    if design:
        rho_d = torch.full((solver.layout()["n_layers"] * wl["n"] ** wl["sdim"],), 0.4, dtype=torch.float64, device=dev)
        rt = torch.empty(nd, dtype=torch.float64, device=dev)
        dJt = torch.empty_like(rho_d)
        dJd = torch.empty_like(rho_d)
        rnew = torch.empty_like(rho_d)

    def step(i):
        if design:  # filter -> solve -> adjoint -> sensitivities -> F^T -> OC (warm starts kept)
            solver.filter(rho_d, rt)
            solver.solve(rt, T)
            a = solver.stats()
            solver.adjoint(rt, f, lam)
            b = solver.stats()
            solver.sensitivity(rt, T, lam, dJt)
            solver.filter(dJt, dJd, transpose=True)
            solver.oc_update(rho_d, dJd, rnew)
            rho_d.copy_(rnew)
        else:
            solver.solve(rhos[i], T)
            a = solver.stats()
            solver.adjoint(rhos[i], f, lam)
            b = solver.stats()
            solver.sensitivity(rhos[i], T, lam, dJ)
        its.append((a["iterations"], b["iterations"], a["solve_ms"], b["solve_ms"], b["setup_ms"],
                    a["rel_residual"], b["rel_residual"]))

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            if not design:
                T.zero_(); lam.zero_()
            step(i)
        its.clear()
        if design:  # the e2e leg below repeats the timed design iterations from the same state
            snap = (rho_d.clone(), T.clone(), lam.clone())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        l0 = solver.kernel_launches()
        times = []
        for k in range(args.steps):
            flush.fill_(float(k))                      # L2 flush, outside the timed events
            if not design:                             # design loop: warm start
                T.zero_(); lam.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(args.warmup + k)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        launches = solver.kernel_launches() - l0
        clocks = sampler.stop()
        if world > 1:
            dist.barrier()
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 2.0 * N_global / (ms / 1e3)

    # ---- dominant kernel: fine-level damped-Jacobi sweep (live CUDA-event timing) ---------
    reps = 20
    with torch.cuda.stream(stream):
        solver.bench_op(rhos[0], 0, 2, 3)
        k0 = torch.cuda.Event(enable_timing=True); k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        solver.bench_op(rhos[0], 0, 2, reps)
        k1.record(stream)
        k1.synchronize()
    t_sweep = k0.elapsed_time(k1) / reps / 1e3
    rho_bytes = 8 * nd
    alg_bytes = 24 * N + rho_bytes           # read x, b; write y; rho (once)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes / t_sweep / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        ent = tj.get("configs", {}).get(str(args.config))
        if ent is None and tj.get("config") == args.config:
            ent = tj
        if ent is not None:
            traffic = ent.get("traffic_bytes_per_launch")

    # ---- end-to-end through the C ABI with pinned host buffers ------------------------------
    e2e = None
    if args.e2e_steps > 0 and design:
        # the design iteration through the public API, repeating the timed iterations from their
        # starting state: this step's design comes from pinned host memory, the new design and the
        # compliance go back to the host
        rho_ht = torch.empty(rho_d.numel(), dtype=torch.float64).pin_memory()
        new_ht = torch.empty_like(rho_ht).pin_memory()
        saved = list(its)
        et = []
        rho_d.copy_(snap[0]); T.copy_(snap[1]); lam.copy_(snap[2])
        del snap
        with torch.cuda.stream(stream):
            for k in range(args.e2e_steps):
                rho_ht.copy_(rho_d)
                flush.fill_(1.0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rho_d.copy_(rho_ht, non_blocking=True)
                step(0)
                phi = solver.dot(f, T)
                new_ht.copy_(rho_d, non_blocking=True)
                stream.synchronize()
                et.append(time.perf_counter() - t0)
        its[:] = saved
        ems = statistics.mean(et) * 1e3
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": 2.0 * N_global / (ems / 1e3), "unit": "DOF/s", "ms_per_step": ems,
               "h2d_bytes_per_step": 8 * rho_d.numel(), "d2h_bytes_per_step": 8 * rho_d.numel() + 8,
               "compliance": phi}
    elif args.e2e_steps > 0:
        def pinned(n_):
            return torch.zeros(n_, dtype=torch.float64).pin_memory().numpy()
        rho_h = pinned(nd); T_h = pinned(N); lam_h = pinned(N); f_h = pinned(N); dJ_h = pinned(nd)
        f_h[:] = f.cpu().numpy()
        et = []
        for k in range(args.e2e_steps):
            rho_h[:] = rhos[k % len(rhos)].cpu().numpy().reshape(-1)
            T_h[:] = 0.0; lam_h[:] = 0.0
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            solver.solve(rho_h, T_h)
            solver.adjoint(rho_h, f_h, lam_h)
            solver.sensitivity(rho_h, T_h, lam_h, dJ_h)
            torch.cuda.synchronize()
            et.append(time.perf_counter() - t0)
        ems = statistics.mean(et) * 1e3
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = 3 * 8 * nd + 8 * N * 5          # rho x3; T in (solve, sens); g; lambda in (adjoint, sens)
        d2h = 8 * N * 2 + 8 * nd              # T, lambda, dJ
        e2e = {"value": 2.0 * N_global / (ems / 1e3), "unit": "DOF/s", "ms_per_step": ems,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    # ---- CPU oracle baseline (rank 0, N = 1 only) ----------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nrep = 32
            res = run_cpu_subprocess(nrep, 1)
            secs = statistics.mean(res["times"])
            cpu = {"value": 2.0 * res["dofs"] / secs, "unit": "DOF/s", "cores": 1, "kind": "oracle",
                   "sample": f"oracle (NumPy/SciPy SuperLU, single thread) on a {nrep}^2x{nrep} replica of the "
                             f"workload ({res['dofs']} DOFs): assembly+LU+forward+adjoint+sensitivity, "
                             f"{secs:.1f} s; host {cpu_model()}"}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "DOF/s", "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"[:300]}

    fi = [a for a, *_ in its]; ai = [b for _, b, *_ in its]
    out = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded smooth random designs, st_inputs)",
        "config": {"workload": wl["name"], "dofs": N_global, "dofs_per_rank": N, "design_vars": nd,
                   "rtol": args.rtol,
                   "step": ("density filter + rho setup + forward solve (warm start) + adjoint solve + sensitivities "
                            "+ filter^T + OC update" if design else
                            "rho setup + forward solve + adjoint solve + sensitivities"),
                   "parallelism": f"{world} time slabs (NCCL)" if world > 1 else "1 GPU",
                   "l2": "flushed (256 MB write) between steps",
                   "preconditioner": precond_desc(args, solver)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "fine-level damped-Jacobi sweep (" + ("tc2d_kernel, time-constant rho" if wl["tc"] and wl["sdim"] == 2
                                                              else "tv2d_kernel, space-time rho, uniform capacity" if wl["sdim"] == 2
                                                              else "tc3d_kernel, (3+1)D time-constant rho") + ")",
                     "bytes_per_launch": alg_bytes, "us_per_launch": t_sweep * 1e6,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        "solver": {"fwd_its": fi, "adj_its": ai,
                   "fwd_ms": [round(x[2], 2) for x in its], "adj_ms": [round(x[3], 2) for x in its],
                   "setup_ms": [round(x[4], 2) for x in its],
                   "fwd_dofs_per_s": N / (statistics.mean(x[2] for x in its) / 1e3),
                   "adj_dofs_per_s": N / (statistics.mean(x[3] for x in its) / 1e3),
                   "rel_res": max(max(x[5], x[6]) for x in its),
                   "levels": len(solver.hierarchy())},
    }
    if rank == 0:
        print(json.dumps(out))
    solver.close()
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.config]
    n = 24
    res = run_cpu_subprocess(n, args.warmup + args.steps)
    times = res["times"][args.warmup:]
    ms = statistics.mean(times) * 1e3
    value = 2.0 * res["dofs"] / (ms / 1e3)
    sample = (f"oracle (NumPy/SciPy SuperLU direct, single thread) per step on a {n}^2x{n} replica of "
              f"{wl['name'].split(':')[0]} ({res['dofs']} DOFs): assembly+LU+forward+adjoint+sensitivity; "
              f"host {cpu_model()}")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": wl["name"], "sample": f"{n}^2x{n}"},
           "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    a = parse()
    if a.cpu_worker:
        cpu_worker(a.cpu_worker, a.cpu_reps)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_cuda(a)
