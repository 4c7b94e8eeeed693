#!/usr/bin/env python
"""bench.py — driver benchmark of the all-at-once space-time solve (arxiv 2508.09589 hot path).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One STEP = one pass of the whole hot path on a fresh synthetic design:
rho-dependent setup (Galerkin coarse operators, coarsest inverse, RHS), forward (F)GMRES+MG
solve to true-residual rtol 1e-8 from T = 0, adjoint solve of the time-integrated thermal
compliance (dJ/dT = f), element sensitivities - one st_design_step call. Workload at N = 1:
BASELINE config 3 (configs[2]) at full size: (2+1)D 1024^2 x 1024 elements, 1,076,890,625
space-time DOFs, an independent smooth design per time layer, Q(t) = 1 + sin 2 pi t (the
north_star's "largest config"; it fits one B200 with the memory plan of DESIGN.md sec. 6).
--config 2|4|5|33 runs the other workloads. value = 2 N_n (forward + adjoint DOFs solved)
per step time.
For N > 1 the SAME problem is split into N time slabs (one per GPU, NCCL over NVLink: halo
planes, Krylov sums, agglomerated coarse levels): strong scaling; config 5
grows in time with N (weak scaling).
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
SIN_SRC = ("sin", 1.0, 1.0, 6.283185307179586)
# opts: library options of the workload's launch configuration; scaling: how the
# workload is split over N GPUs ("strong": the same global problem in N time slabs; "weak": the time
# extent grows with N, BASELINE config 5); bpd_iter: SURVEY.md sec. 8(d)'s model bytes per DOF and
# FGMRES iteration (the whole-step roofline); sweep_bpd: sec. 8(d)'s damped-Jacobi bytes per DOF
WORKLOADS = {
    2: dict(name="config2: (2+1)D 256^2x256 elements, time-constant smooth rho (sigma 3, [0.01,1]), "
                 "k=1e-3+rho^3(1-1e-3), c=1, Q=1, T=0 sink patch (10% of x1=0), T0=0",
            sdim=2, n=256, nt=256, mats=CFG1_MATS, tc=True, design="smooth_tc", source=("uniform", 1.0, 0.0, 0.0),
            # FGMRES(8): the same 10-13 iterations as FGMRES(16) with a cheaper Gram-Schmidt tail
            # (profiles/r02/restart_ab.log: 704.6 -> 737.8 MDOF/s)
            tau=1.0, opts=dict(restart=8), scaling="strong", bpd_iter=435.0, sweep_bpd=32.0),
    1: dict(name="config1: (2+1)D 16^3, rho~U[0.1,1] space-time", sdim=2, n=16, nt=16, mats=CFG1_MATS, tc=False,
            design="uniform", source=("uniform", 1.0, 0.0, 0.0), tau=1.0, opts={}, scaling="strong",
            bpd_iter=580.0, sweep_bpd=40.0),
    4: dict(name="config4: (3+1)D 64^3x128, time-constant smooth rho, c=0.1+0.9rho, k_min=1e-4", sdim=3, n=64,
            nt=128, mats=CFG4_MATS, tc=True, design="smooth_tc", source=("uniform", 1.0, 0.0, 0.0), tau=1.0,
            # FGMRES(8): 25-31 iterations as with FGMRES(16) (profiles/r02/restart_ab.log: 220-222 -> 227 MDOF/s)
            opts=dict(restart=8), scaling="strong", bpd_iter=412.0, sweep_bpd=32.0),
    5: dict(name="config5 (per GPU): (2+1)D 512^2x512, space-time design; a step = one OC design iteration "
                 "(density filter r=2, forward, adjoint, sensitivities, filter^T, OC volfrac 0.4) from rho=0.4",
            sdim=2, n=512, nt=512, mats=CFG1_MATS, tc=False, design="const", source=("uniform", 1.0, 0.0, 0.0),
            # FGMRES(8): as configs 2 and 4 (profiles/r02/restart_ab.log: 277.4 -> 289.9 MDOF/s, same iterations)
            tau=1.0, opts=dict(restart=8), scaling="weak", bpd_iter=583.0, sweep_bpd=40.0),
    # BASELINE config 3 at full size: 1,076,890,625 DOFs (8.6 GB per vector). One GPU holds it with the
    # memory plan of DESIGN.md sec. 6: right-preconditioned GMRES(7) (no Z vectors; 188.9 of 192 GB),
    # stepping down to GMRES(6) (180.2 GB) on a box with less free memory; the Krylov pool as the hooks'
    # and the V-cycle's level-0 scratch, the compliance adjoint RHS generated in the library. Sweeps 1 + 2 on
    # the fine and big coarse levels (profiles/r02/nu_split_r02.log: 653 -> 693 MDOF/s at 14 + 14
    # iterations; 2 + 2 stays the library default, better on configs 2, 4 and the 512^2 slab)
    3: dict(name="config3: (2+1)D 1024^2x1024 elements (1,076,890,625 DOFs), an independent smooth field per "
                 "time layer (sigma 3, [0.01,1]), Q(t) = 1 + sin(2 pi t), k=1e-3+rho^3(1-1e-3), c=1, T=0 sink "
                 "patch (10% of x1=0), T0=0",
            sdim=2, n=1024, nt=1024, mats=CFG1_MATS, tc=False, design="smooth_layers", source=SIN_SRC, tau=1.0,
            opts=dict(krylov=1, restart=7, nu_pre=1), scaling="strong", bpd_iter=580.0, sweep_bpd=40.0),
    # the 1/8 slab of config 3 on one GPU (round-1 "config 3 shape"): parity / profiling case
    33: dict(name="config3-shaped (1/8 of config 3 on one GPU): (2+1)D 512^2x512, an independent smooth field per "
                  "time layer, Q(t) = 1 + sin(2 pi t)", sdim=2, n=512, nt=512, mats=CFG1_MATS, tc=False,
             design="smooth_layers", source=SIN_SRC, tau=1.0, opts=dict(restart=8), scaling="strong", bpd_iter=580.0,
             sweep_bpd=40.0),  # FGMRES(8): 577.9 -> 589.3 MDOF/s (profiles/r02/restart_ab.log)
}
DEFAULT_CONFIG = 3
METRIC = "space-time DOFs solved/sec (FGMRES+MG to rtol 1e-8) & operator GB/s vs HBM peak"
# the paper's own results, quoted as context (CPU supercomputer LUMI-C: 2x AMD EPYC 7763 per node, 128 cores,
# 256 GiB); not comparable measurements and not targets
PAPER_CONTEXT = {
    "hardware": "LUMI-C CPU nodes, 2x AMD EPYC 7763 (64 cores each), 128 cores / 256 GiB per node (PAPER.md:615-616)",
    "speedup_vs_time_stepping": "52.1x at 7.7x the core-hours (16.4 s vs 855 s), Example 1, 640^2x1280 = 526,338,561 "
                                "DOFs, 10 design iterations, 400 nodes / 51,200 cores (PAPER.md:660, 705-712)",
    "largest_solve": "4,202,501,121 DOFs (1280^2x2560), full optimisation in 1,035 s on 500 nodes / 64,000 cores, "
                     "24.0x faster than time-stepping at 5.2x the cost (PAPER.md:1036-1038)",
}


def solver_opts(args):
    o = dict(smoother=2 if args.smoother == "gmres" else 0)
    nu = args.nu or (10 if args.smoother == "gmres" else 0)  # 0: the library defaults
    if nu:
        o["nu_pre"] = o["nu_post"] = nu
    if args.nu_pre > 0:
        o["nu_pre"] = args.nu_pre
    if args.nu_post >= 0:
        o["nu_post"] = args.nu_post
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
    kr = "right-preconditioned GMRES(%d)" if o["krylov"] == 1 else "FGMRES(%d)"
    return (kr + " + V-cycle, %s, %s") % (o["restart"], sm, "full space-time coarsening" if args.full_coarsening
                                         else "semi-coarsening (Algorithm 1)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG,
                    help="BASELINE config (1-5); 33 = the 512^2x512 one-eighth slab of config 3")
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--smoother", default="jacobi", choices=["jacobi", "gmres"],
                    help="jacobi: damped Jacobi nu+nu (default); gmres: the paper's GMRES(nu)-Jacobi smoother")
    ap.add_argument("--nu", type=int, default=0,
                    help="fine-level Jacobi sweeps / GMRES steps (default: the library's 2 for jacobi, 10 for gmres)")
    ap.add_argument("--nu-pre", type=int, default=0, help="fine-level pre-smoothing sweeps (overrides --nu)")
    ap.add_argument("--nu-post", type=int, default=-1, help="fine-level post-smoothing sweeps (overrides --nu)")
    ap.add_argument("--nu-coarse", type=int, default=-1,
                    help="Jacobi sweeps on the coarse levels (default: the library's 5; 0 = --nu)")
    ap.add_argument("--full-coarsening", action="store_true", help="the paper's full space-time coarsening")
    ap.add_argument("--omega", type=float, default=0.0, help="Jacobi weight cap (default: the library's 0.75)")
    ap.add_argument("--restart", type=int, default=0, help="FGMRES restart length (default: the library's 16)")
    ap.add_argument("--krylov", default="", choices=["", "fgmres", "gmres"],
                    help="outer Krylov method (default: the workload's; config 3: gmres)")
    ap.add_argument("--coarse-max-nodes", type=int, default=0, help="coarsest-level size (default: the library's 400)")
    ap.add_argument("--nu-fine-nodes", type=int, default=-1,
                    help="coarse levels with at least this many nodes use the fine-level sweep counts (default: the "
                         "workload's)")
    ap.add_argument("--fuse-prolong", type=int, default=-1,
                    help="prolongation fused into the first post-sweep (1) or separate kernels (0); default: the library's")
    ap.add_argument("--timestepping", action="store_true",
                    help="also time the GPU time-stepping baseline (st_timestep, backward Euler with nt steps and a "
                         "spatial-MG PCG per step; time-constant workloads) against the space-time forward solve")
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
        self.skip = 0

    def wait_first(self, timeout_s: float = 5.0):
        """Block until nvidia-smi has written its first sample: its start-up (NVML initialisation, which
        stalls CUDA calls of this process for a few hundred ms) must not land in a short timed region
        (config 2: 5 steps of 46 ms measured 74 ms each with the sampler started at the region's start)."""
        if self.p is None:
            return
        t0 = time.time()
        while time.time() - t0 < timeout_s:
            try:
                if os.path.getsize(self.f.name) > 0:
                    return
            except OSError:
                return
            time.sleep(0.02)

    def mark(self):
        """Start of the timed region: only the samples from here on (and the one just before) count."""
        try:
            self.skip = max(0, len(open(self.f.name).read().splitlines()) - 1)
        except OSError:
            self.skip = 0

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().splitlines()[self.skip:] if l.strip()]
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
def solver_opts_for(wl, args):
    o = dict(wl["opts"])
    o.update(solver_opts(args))
    if args.krylov:
        o["krylov"] = 1 if args.krylov == "gmres" else 0
    if args.coarse_max_nodes > 0:
        o["coarse_max_nodes"] = args.coarse_max_nodes
    if args.nu_fine_nodes >= 0:
        o["nu_fine_nodes"] = args.nu_fine_nodes
    if args.fuse_prolong >= 0:
        o["fuse_prolong"] = args.fuse_prolong
    return o


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
    if world > 1:
        if wl["scaling"] == "weak":  # BASELINE config 5: the time extent grows with the GPU count
            wl["nt"] = wl["nt"] * world
            wl["tau"] = wl["tau"] * world
            wl["name"] = wl["name"] + f" extended in time to nt={wl['nt']}, tau={wl['tau']:g} (time slabs)"
        else:                        # the same global problem in `world` time slabs
            wl["name"] = wl["name"] + f", split into {world} time slabs"
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_comm = S.nccl_comm_init(obj[0], rank, world)
        S.nccl_selftest(nccl_comm, rank, world)  # fail loudly before any timing if the transport is broken
    opts = solver_opts_for(wl, args)
    N_global = (wl["n"] + 1) ** wl["sdim"] * (wl["nt"] + 1)
    nsteps = args.warmup + args.steps
    big = N_global > 4e8          # config 3: one design on the device, a new one per step by rho <- 1.01 - rho
    # memory plan: config 3 on one GPU uses ~180 of the B200's 183 GiB with GMRES(6). Should
    # a box have less free memory, the restart length steps down (each step frees one 8.6 GB Krylov vector)
    # rather than the run failing; the line reports the options actually used
    mem_note = None
    while True:
        try:
            solver = S.Solver(wl["sdim"], wl["n"], wl["nt"], mats=wl["mats"], source=wl["source"], tau=wl["tau"],
                              time_constant=wl["tc"], stream=stream.cuda_stream, device=local, rtol=args.rtol,
                              maxit=1000, rank=rank, size=world, nccl_comm=nccl_comm, **opts)
            N = solver.n_nodes    # this rank's owned nodes
            nd = solver.n_design
            lay = solver.layout()
            reserve = [torch.empty(n_, dtype=torch.float64, device=dev) for n_ in
                       (N, N, nd if wl["tc"] else lay["n_layers"] * wl["n"] ** wl["sdim"], nd + 256 * 1024 * 1024 // 8)]
            del reserve           # the caller's vectors fit next to the library's workspaces
            free_b, _ = torch.cuda.mem_get_info(dev)
            if big and free_b < 1.5e9 and opts.get("restart", 16) > 6:
                raise torch.OutOfMemoryError("less than 1.5 GB of headroom")  # keep a margin: one step down
            break
        except (S.StError, torch.OutOfMemoryError) as ex:
            oom = isinstance(ex, torch.OutOfMemoryError) or getattr(ex, "code", 0) == -5
            r = opts.get("restart", 16)
            if not oom or r <= 2:
                raise
            try:
                solver.close()
            except Exception:  # noqa: BLE001
                pass
            solver = None
            torch.cuda.empty_cache()
            opts["restart"] = r - 1
            mem_note = f"restart lowered to {r - 1} (device memory)"
    design = args.config == 5     # a step is one config-5 design iteration (R-13)
    t_gen = time.perf_counter()
    if wl["design"] == "const":
        rhos = [torch.full((nd,), 0.4 + 0.01 * s, dtype=torch.float64, device=dev) for s in range(nsteps)]
    elif wl["tc"]:  # time-constant designs are replicated on every rank (same seed)
        rhos = [torch.as_tensor(np.ascontiguousarray(I.design_for(wl["sdim"], wl["n"], wl["nt"], wl["design"], seed=s)),
                                device=dev).reshape(-1) for s in range(nsteps)]
    else:           # space-time designs: this rank's layers (owned + the ghost layer of the next slab)
        layers = (lay["layer0"], lay["layer0"] + lay["rho_layers"])
        nr = 1 if big else nsteps
        rhos = [torch.as_tensor(I.design_for(wl["sdim"], wl["n"], wl["nt"], wl["design"], seed=s, layers=layers),
                                device=dev).reshape(-1) for s in range(nr)]
    t_gen = time.perf_counter() - t_gen

    def rho_for(i):
        if big:  # a different design every step, in place, outside the timed region ([0.01, 1] -> [0.01, 1])
            if i > 0:
                torch.sub(1.01, rhos[0], out=rhos[0])
            return rhos[0]
        return rhos[i % len(rhos)]

    T = torch.zeros(N, dtype=torch.float64, device=dev)
    lam = torch.zeros_like(T)
    dJ = torch.empty(nd if wl["tc"] else lay["n_layers"] * wl["n"] ** wl["sdim"], dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    its = []

    if design:
        f = torch.empty_like(T)
        with torch.cuda.stream(stream):
            solver.rhs(rhos[0], f, None)
        rho_d = torch.full((lay["n_layers"] * wl["n"] ** wl["sdim"],), 0.4, dtype=torch.float64, device=dev)
        rt = torch.empty(nd, dtype=torch.float64, device=dev)
        dJt = torch.empty_like(rho_d)
        dJd = torch.empty_like(rho_d)
        rnew = torch.empty_like(rho_d)
        dJ = dJt

    def step(rho):
        if design:  # filter -> solve -> adjoint -> sensitivities -> F^T -> OC (warm starts kept)
            solver.filter(rho_d, rt)
            solver.solve(rt, T)
            a = solver.stats()
            solver.adjoint(rt, None, lam)
            b = solver.stats()
            solver.sensitivity(rt, T, lam, dJt)
            solver.filter(dJt, dJd, transpose=True)
            solver.oc_update(rho_d, dJd, rnew)
            rho_d.copy_(rnew)
        else:  # st_design_step = st_solve + st_adjoint (compliance: dphi/dT = f, R-8) + st_sensitivity
            a, b = solver.design_step(rho, None, T, lam, dJ)
        its.append((a["iterations"], b["iterations"], a["solve_ms"], b["solve_ms"], b["setup_ms"],
                    a["rel_residual"], b["rel_residual"], a["vcycles"], b["vcycles"]))

    # the sampler runs from before the warm-up (its start-up stalls CUDA calls) and is read from the start
    # of the timed region on
    sampler = ClockSampler(local)
    sampler.wait_first()
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            r = rho_for(i)
            if not design:
                T.zero_(); lam.zero_()
            step(r)
        its.clear()
        if design:  # the e2e leg below repeats the timed design iterations from the same state
            snap = (rho_d.clone(), T.clone(), lam.clone())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.mark()
        l0 = solver.kernel_launches()
        times = []
        for k in range(args.steps):
            r = rho_for(args.warmup + k)
            flush.fill_(float(k))                      # L2 flush, outside the timed events
            if not design:                             # design loop: warm start
                T.zero_(); lam.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(r)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        launches = solver.kernel_launches() - l0
        clocks = sampler.stop()
        free_b, total_b = torch.cuda.mem_get_info(dev)
        mem_used = total_b - free_b
        if world > 1:
            dist.barrier()
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 2.0 * N_global / (ms / 1e3)

    # ---- dominant kernel: fine-level damped-Jacobi sweep (live CUDA-event timing) ---------
    reps = 20 if not big else 6
    rb = rho_for(0) if big else rhos[0]
    with torch.cuda.stream(stream):
        solver.bench_op(rb, 0, 2, 3)
        k0 = torch.cuda.Event(enable_timing=True); k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        solver.bench_op(rb, 0, 2, reps)
        k1.record(stream)
        k1.synchronize()
    t_sweep = k0.elapsed_time(k1) / reps / 1e3
    # algorithmic bytes per launch: damped-Jacobi sweep 32 B/DOF (time-constant rho)
    # / 40 B/DOF (time-varying), x the DOFs of one launch; that model reads a stored diagonal the
    # kernel does not need, so the bytes the kernel must move are reported beside it (24 / 32 B/DOF:
    # x, b, y + the k~ layer)
    alg_bytes = wl["sweep_bpd"] * N
    min_bytes = (24.0 if wl["tc"] else 32.0) * N
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes / t_sweep / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        ent = json.load(open(tpath)).get("configs", {}).get(str(args.config))
        if ent is not None:
            traffic = ent.get("traffic_bytes_per_launch")
    fi = [x[0] for x in its]; ai = [x[1] for x in its]
    # whole-step model: sec. 8(d)'s bytes per DOF and FGMRES iteration x DOFs x
    # the iterations of the step, over the step time
    step_bytes = wl["bpd_iter"] * N_global * statistics.mean(f_ + a_ for f_, a_ in zip(fi, ai))
    step_roof = {"bytes_per_dof_iteration": wl["bpd_iter"], "iterations_per_step": statistics.mean(
        f_ + a_ for f_, a_ in zip(fi, ai)), "achieved": step_bytes / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
        "frac": step_bytes / (ms / 1e3) / 1e9 / peak,
        "model": "SURVEY.md sec. 8(d) per-iteration bytes (nu 2+2, m 20) x N_n x (forward + adjoint iterations)"}

    # ---- GPU time-stepping baseline ---------------------
    tsres = None
    if args.timestepping and wl["tc"] and world == 1:
        Tts = torch.empty((wl["nt"] + 1) * (wl["n"] + 1) ** wl["sdim"], dtype=torch.float64, device=dev)
        with torch.cuda.stream(stream):
            solver.timestep(rhos[0], wl["nt"], Tts)       # warm-up (graph capture)
            tsr = [solver.timestep(rhos[k % len(rhos)], wl["nt"], Tts) for k in range(2)]
        ts_ms = statistics.mean(x["ms"] for x in tsr)
        st_fwd = statistics.mean(x[2] for x in its)
        tsres = {"method": "backward Euler, nt steps, spatial-MG PCG per step (same rtol), CUDA graph per CG iteration",
                 "steps": wl["nt"], "ms_forward": ts_ms, "cg_iterations": tsr[-1]["cg_iterations"],
                 "max_step_iterations": tsr[-1]["max_step_iterations"],
                 "space_time_forward_ms": st_fwd, "space_time_speedup_forward": ts_ms / st_fwd,
                 "note": "forward solves only, same mesh / design / rtol; the paper's 52x (PAPER.md:712) compares "
                         "whole design iterations on CPU clusters"}
        del Tts

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
                step(None)
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
        # host copies of this step's designs; the device-side vectors are released first (config 3: the
        # library's staging buffers take their place)
        ndj = dJ.numel()
        rho_h = torch.zeros(nd, dtype=torch.float64).pin_memory().numpy()
        rho_h[:] = rho_for(args.warmup + args.steps).cpu().numpy()
        del T, lam, dJ, rhos, r, rb
        torch.cuda.empty_cache()

        def pinned(n_):
            return torch.zeros(n_, dtype=torch.float64).pin_memory().numpy()
        T_h = pinned(N); lam_h = pinned(N); dJ_h = pinned(ndj)
        et = []
        for k in range(args.e2e_steps):
            if k > 0:  # a new design every step, as in the timed leg
                np.subtract(1.01, rho_h, out=rho_h)
            T_h[:] = 0.0; lam_h[:] = 0.0
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            solver.design_step(rho_h, None, T_h, lam_h, dJ_h)
            torch.cuda.synchronize()
            et.append(time.perf_counter() - t0)
        ems = statistics.mean(et) * 1e3
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = 8 * nd + 8 * N * 2              # rho once; T and lambda initial guesses (st_design_step)
        d2h = 8 * N * 2 + 8 * ndj             # T (during the adjoint solve), lambda, dJ
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
                   "host_cpus": os.cpu_count(),
                   "sample": f"oracle (NumPy/SciPy SuperLU, single thread; the host has {os.cpu_count()} logical "
                             f"CPUs, {cpu_model()}) on a {nrep}^2x{nrep} replica of the workload ({res['dofs']} DOFs): "
                             f"assembly+LU+forward+adjoint+sensitivity, {secs:.1f} s"}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "DOF/s", "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"[:300]}

    hier = solver.hierarchy()
    out = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if (wl["scaling"] == "weak" or world == 1) else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded smooth random designs, st_inputs)",
        "config": {"workload": wl["name"], "dofs": N_global, "dofs_per_rank": N, "design_vars": nd,
                   "rtol": args.rtol,
                   "step": ("density filter + rho setup + forward solve (warm start) + adjoint solve + sensitivities "
                            "+ filter^T + OC update" if design else
                            "rho setup (new design) + forward solve + adjoint solve (compliance) + sensitivities"),
                   "parallelism": f"{world} time slabs (NCCL)" if world > 1 else "1 GPU",
                   "l2": "flushed (256 MB write) between steps" + ("; inputs (8.6 GB per vector) exceed L2" if big else ""),
                   "preconditioner": precond_desc(args, solver), "options": {k: v for k, v in opts.items()},
                   "memory_note": mem_note,
                   "design_generation_s": round(t_gen, 1)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "fine-level damped-Jacobi sweep (" + ("tc2d_kernel, time-constant rho" if wl["tc"] and wl["sdim"] == 2
                                                              else "tv2d_kernel, space-time rho, uniform capacity" if wl["sdim"] == 2
                                                              else "tc3r_kernel, (3+1)D time-constant rho, element layers") + ")",
                     "bytes_per_launch": alg_bytes, "bytes_per_dof": wl["sweep_bpd"],
                     "bytes_source": "SURVEY.md sec. 8(d) damped-Jacobi sweep",
                     "min_bytes_per_launch": min_bytes, "min_frac": min_bytes / t_sweep / 1e9 / peak,
                     "us_per_launch": t_sweep * 1e6,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
        "step_roofline": step_roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        "solver": {"fwd_its": fi, "adj_its": ai, "fwd_vcycles": [x[7] for x in its], "adj_vcycles": [x[8] for x in its],
                   "fwd_ms": [round(x[2], 2) for x in its], "adj_ms": [round(x[3], 2) for x in its],
                   "setup_ms": [round(x[4], 2) for x in its],
                   "fwd_dofs_per_s": N_global / (statistics.mean(x[2] for x in its) / 1e3),
                   "adj_dofs_per_s": N_global / (statistics.mean(x[3] for x in its) / 1e3),
                   "rel_res": max(max(x[5], x[6]) for x in its),
                   "levels": len(hier), "hierarchy": [f"{h['n']}^{wl['sdim']}x{h['nt']} {h['kind']}" for h in hier],
                   "device_mem_used_gb": round(mem_used / 1e9, 1)},
        "paper_context": PAPER_CONTEXT,
    }
    if tsres is not None:
        out["timestepping"] = tsres
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
