#!/usr/bin/env python
"""Benchmark of the pseudo-time wall-distance iteration (HJ, GLUPS fp64).

Default workload = BASELINE config 4 (the metric's target case): 3-D channel
512^3 on [0,1]^3, walls at y = 0, 1, periodic x and z, HJ (eps = 0.2),
explicit 6th order (E6), implicit filter alpha_f = 0.49, CFL 0.5, from
phi = 0.  One "step" = one full pseudo-iteration (local dt, 4 RK stages,
BCs, 3 filter sweeps, convergence reduction) over all 134,217,728 nodes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference runs the CPU oracle port (oracle/wd.py, the reference's
numpy algorithm restated) on rank 0 over a bounded sample of the same
workload.  Under torchrun (N > 1) the 512^3 grid is slab-decomposed over the
N GPUs (paper_2111_09859_b200/dist.py: ghost-plane exchange per RK stage,
all_to_all transposes around the axis-0 filter, all_reduce of the stop
test) -- strong scaling, max time over ranks.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HJ grid-point updates/s (GLUPS, fp64)"
UNIT = "GLUPS"

CONFIGS = {
    "c4": dict(workload="c4_channel3d_512^3_hj_E6_F0.49", dims=(512, 512, 512),
               periodic=(True, False, True), kind="hj", scheme="E6", alpha_f=0.49,
               faces={"imin": "periodic", "imax": "periodic", "jmin": "wall",
                      "jmax": "wall", "kmin": "periodic", "kmax": "periodic"}),
}

# Algorithmic fp64 words per node update: stages S1 4,
# S2 6, S3 6, S4 5 (= 21) + filter 2 per axis + convergence read 1.
WORDS_STAGE = {1: 4, 2: 6, 3: 6, 4: 5}


def words_per_update(nd, filt):
    return 21 + (2 * nd if filt else 0) + 1


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ CPU arm
def cpu_sample(cfg, steps, warmup):
    """The oracle (reference algorithm, numpy, 1 thread) on a bounded slab
    of the same workload: (32, 512, 64) nodes with the 512^3 spacings."""
    from oracle import wd
    n = cfg["dims"]
    sd = (32, n[1], 64)
    og = wd.cartesian(sd[0], sd[1], sd[2], Lx=sd[0] / n[0], Ly=1.0, Lz=sd[2] / n[2],
                      periodic=cfg["periodic"])
    bnd = wd.Boundary({k: v for k, v in cfg["faces"].items() if v != "periodic"})
    c = wd.Config(wd.Formulation(cfg["kind"]), cfg["scheme"], cfg["alpha_f"], 0.5, 1e-15, 10**9)
    phi = wd.apply_bc(np.zeros(sd), bnd)
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        dt = wd.local_timestep(phi, og, c.formulation, c.cfl, c.scheme)
        phi = wd.rk4_step(phi, og, c, dt, bnd)
        if s >= warmup:
            times.append(time.perf_counter() - t0)
    nodes = int(np.prod(sd))
    total = float(sum(times))
    return {"value": nodes * len(times) / total / 1e9, "unit": UNIT, "cores": 1,
            "kind": "port",
            "sample": f"{len(times)} pseudo-iterations of a {sd[0]}x{sd[1]}x{sd[2]} slab "
                      f"(same spacing/BCs as 512^3), oracle/wd.py numpy, 1 thread "
                      f"of {os.cpu_count()} host cores",
            "seconds": total}


def run_reference(args, world, rank):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    cb = cpu_sample(cfg, args.steps, args.warmup)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "sample_dims": [32, 512, 64]},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def _device_steps(grid, cfg, fc, filt, K, Wm, arith):
    """K device-timed steps of the same workload in another arithmetic mode."""
    import torch
    from paper_2111_09859_b200 import _context, _native as nat
    ctx = _context.NativeSolver(grid, cfg["faces"], None, cfg["scheme"], fc, filt, 0.5, 1e-15,
                                10**9, arith=arith)
    dims = tuple(grid.dims)
    phi = torch.zeros(dims, dtype=torch.float64, device="cuda")
    hist = torch.zeros(K + Wm + 8, dtype=torch.float64, device="cuda")
    nat.check(ctx.lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
    stream = ctx.stream()
    nat.check(ctx.lib.wd_steps(ctx.ptr, Wm))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    nat.check(ctx.lib.wd_steps(ctx.ptr, K))
    e1.record(stream)
    e1.synchronize()
    secs = e0.elapsed_time(e1) / 1e3
    ctx.close()
    del phi, hist
    torch.cuda.empty_cache()
    N = int(np.prod(dims))
    return {"arith": arith, "value": round(N * K / secs / 1e9, 4), "unit": UNIT,
            "ms_per_step": round(secs / K * 1e3, 4),
            "parity": "bit-identical to the reference algorithm (oracle/wd.py)"}


def _time_to_converge(ms_per_step, arith):
    """Iterations to tol 1e-8 for this configuration: the oracle's count
    (bit-exact x/z-invariant strip, tests/golden/strip_c4_ny512.npz) and the
    full 512^3 solve measured through solve_steady on one B200
    (tools/converge_c4.py -> profiles/converge.json)."""
    path = os.path.join(ROOT, "profiles", "converge.json")
    try:
        rec = json.load(open(path))["c4"]
    except Exception:
        return None
    iters = rec.get("iters")
    out = {"iters_to_tol_1e-8": iters, "source": rec.get("source"),
           "est_seconds_at_this_step_time": round(iters * ms_per_step / 1e3, 2) if iters else None}
    if rec.get("measured_s") and rec.get("arith") == arith:
        out.update(measured_seconds=rec["measured_s"], measured_iters=rec.get("measured_iters"),
                   measured_rel_dev_vs_oracle=rec.get("measured_rel_dev_vs_oracle"),
                   measured_on=rec.get("measured_on"))
    return out


def run_b200_dist(args, world, rank, local):
    """Slab decomposition of the same global grid over the N ranks (strong
    scaling; also at N = 1 with --dist): the native step program of
    csrc/wd_dist.cuh with the NCCL communicator, k steps per CUDA graph."""
    import ctypes
    import torch
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import dist, _native as nat

    cfg = CONFIGS[args.config]
    dims = tuple(args.n if args.n else d for d in cfg["dims"])
    grid = W.build_cartesian(*dims, Lx=dims[0] / 512 if args.n else 1.0, Ly=1.0,
                             Lz=dims[2] / 512 if args.n else 1.0, periodic=cfg["periodic"])
    fc = W.FormulationConfig(kind=cfg["kind"])
    filt = W.FilterConfig(cfg["alpha_f"])
    K, Wm = args.steps, args.warmup
    chunk = 2
    scfg = W.SolveConfig(formulation=fc, scheme=cfg["scheme"], filter_config=filt, cfl=0.5,
                         tol=1e-15, max_iters=10**9, arith=args.arith)
    comm = dist.NcclComm.from_torch() if world > 1 else dist.NcclComm(0, 1)
    ds = dist.DistributedSolve(grid, cfg["faces"], scfg, comm, filter0=args.filter0,
                               overlap=not args.no_overlap, hist_len=K + Wm + 8)
    ds.bind(None)
    warm_steps = 0
    for _ in range((Wm + chunk - 1) // chunk):
        ds.steps(chunk)
        warm_steps += chunk
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    stream = ds.stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done = 0
    while done < K:
        c = min(chunk, K - done)
        ds.steps(c)
        done += c
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    secs = allreduce_max(e0.elapsed_time(e1) / 1e3, world)
    st = ds.status()
    if st.state != nat.STATE_RUNNING or st.iters != warm_steps + K:
        raise RuntimeError(f"benchmark run stopped early (state {st.state}, {st.iters} of "
                           f"{warm_steps + K} steps)")
    N = int(np.prod(dims))
    Nl = N // world
    value = N * K / secs / 1e9
    peak, peak_kind = _peaks()
    # dominant kernel of this rank's slab: the RK stage kernels on its planes
    lib = ds.lib
    lctx = lib.wd_dist_context(ds.ptr)
    kern, kwords = {}, {}
    avg = ctypes.c_double(0.0)
    for kid in (1, 2, 3, 4):
        if ds.fused and lib.wd_time_kernel(lctx, kid, 5, ctypes.byref(avg)) == 0:
            kern[f"stage{kid}"] = avg.value
            kwords[f"stage{kid}"] = lib.wd_kernel_words(lctx, kid)
    roof = None
    if kern:
        dom = max(kern, key=kern.get)
        ach = kwords[dom] * 8 * Nl / (kern[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": None, "kernel": dom + " (rank slab)",
                "alg_bytes_per_launch": kwords[dom] * 8 * Nl, "peak_source": peak_kind}
    w_upd = words_per_update(3, True)
    step_ach = w_upd * 8 * Nl / (secs / K) / 1e9
    ranges = 3 if ds.overlap else 1
    launches = 4 * ranges * 2 + (2 if ds.filter0 == "partitioned" else 3) + 2 + 1 + \
        (2 if world > 1 else 0)
    ds.close()
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        phi0 = torch.zeros(dims, dtype=torch.float64).pin_memory()
        ecfg = W.SolveConfig(formulation=fc, scheme=cfg["scheme"], filter_config=filt, cfl=0.5,
                             tol=1e-15, max_iters=K, arith=args.arith)
        bnd = W.BoundarySpec(cfg["faces"])
        for _ in range(2):
            rep = W.solve_steady(grid, bnd, ecfg, phi0=phi0, chunk=chunk, comm=comm)
            del rep
            gc.collect()
        samples = []
        for _ in range(3):
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            rep = W.solve_steady(grid, bnd, ecfg, phi0=phi0, chunk=chunk, comm=comm)
            torch.cuda.synchronize()
            samples.append(allreduce_max(time.perf_counter() - t0, world))
            assert rep.iters == K
            del rep
            gc.collect()
        t_e2e = sorted(samples)[1]
        e2e = {"value": N * K / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(N * 8 / K),
               "d2h_bytes_per_step": int(world * (N * 8 + 8 * K) / K),
               "seconds": t_e2e, "samples_s": [round(x, 4) for x in samples],
               "includes": "median of 3 solve_steady(comm=) calls on every rank, each: context "
                           "setup + H2D of the rank's slab of phi0 (pinned) + K steps + "
                           "all_gather of the slabs + D2H of the global field on every rank"}
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": round(secs / K * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "dims": list(dims), "arith": args.arith,
                       "global_nodes": N, "parallelism": f"slab{world}",
                       "axis0_filter": ds.filter0, "overlap": ds.overlap, "cuda_graph": ds.graph,
                       "comm": "nccl (libwd_b200: wd_comm_init)" if world > 1 else "none (1 rank)",
                       "l2": "inputs larger than L2"},
            "roofline": roof,
            "step_roofline": {"achieved": round(step_ach, 1), "per": "gpu", "peak": peak,
                              "unit": "GB/s", "frac": round(step_ach / peak, 4),
                              "words_per_update": w_upd, "peak_source": peak_kind},
            "kernel_ms": {k: round(v, 4) for k, v in kern.items()},
            "gpu_launches": K * launches, "clocks": clk, "e2e": e2e,
            "time_to_converge": _time_to_converge(secs / K * 1e3, args.arith)}
    if rank == 0 and not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_sample(cfg, 9, 1)
    comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_b200(args, world, rank, local):
    import ctypes
    import torch
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import _context, _native as nat

    cfg = CONFIGS[args.config]
    dims = tuple(args.n if args.n else d for d in cfg["dims"])
    grid = W.build_cartesian(*dims, Lx=dims[0] / 512 if args.n else 1.0, Ly=1.0,
                             Lz=dims[2] / 512 if args.n else 1.0, periodic=cfg["periodic"])
    fc = W.FormulationConfig(kind=cfg["kind"])
    filt = W.FilterConfig(cfg["alpha_f"]) if cfg["alpha_f"] else None
    K, Wm = args.steps, args.warmup
    ctx = _context.NativeSolver(grid, cfg["faces"], None, cfg["scheme"], fc, filt, 0.5, 1e-15,
                                10**9, arith=args.arith)
    lib = ctx.lib
    N = int(np.prod(dims))
    phi = torch.zeros(dims, dtype=torch.float64, device="cuda")
    hist = torch.zeros(K + Wm + 8, dtype=torch.float64, device="cuda")
    nat.check(lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
    stream = ctx.stream()
    chunk = 2
    warm_steps = 0
    for _ in range((Wm + chunk - 1) // chunk):
        nat.check(lib.wd_steps(ctx.ptr, chunk))
        warm_steps += chunk
    torch.cuda.synchronize()
    # timed region
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done = 0
    while done < K:
        c = min(chunk, K - done)
        nat.check(lib.wd_steps(ctx.ptr, c))
        done += c
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    secs = e0.elapsed_time(e1) / 1e3
    st = nat.Status()
    nat.check(lib.wd_read_status(ctx.ptr, ctypes.byref(st)))
    # a status that left RUNNING would turn the remaining replays into
    # no-ops and inflate the number: every timed step must have run
    if st.state != nat.STATE_RUNNING or st.iters != warm_steps + K:
        raise RuntimeError(f"benchmark run stopped early (state {st.state}, {st.iters} of "
                           f"{warm_steps + K} steps)")
    secs_max = allreduce_max(secs, world)
    value = N * K * world / secs_max / 1e9

    # per-kernel device time (CUDA events on the solver stream)
    kern = {}
    if ctx.fused:
        avg = ctypes.c_double(0.0)
        names = {1: "stage1", 2: "stage2", 3: "stage3", 4: "stage4", 5: "filter_axis0",
                 6: "filter_axis1", 7: "filter_axis2", 8: "change"}
        if filt is not None:
            del names[8]  # the change reduction is fused into the last sweep
        for kid, name in names.items():
            if lib.wd_time_kernel(ctx.ptr, kid, 5, ctypes.byref(avg)) == 0:
                kern[name] = avg.value
    peak, peak_kind = _peaks()
    nd = len(dims)
    roof = None
    if kern:
        # algorithmic words per node of each kernel as run (the fast stage
        # kernels use a low-storage RK4: 3 / 5 / 4 / 5)
        kwords = {name: lib.wd_kernel_words(ctx.ptr, kid) for kid, name in names.items()}
        # dominant launch: the longest one; the four RK-stage launches are one
        # kernel template and within ~2 % of each other, so launches within
        # 3 % of the longest count as tied and the tie goes to the one moving
        # the most data (every launch's own fraction is listed in
        # kernel_rooflines)
        tmax = max(kern.values())
        dom = max((k for k in kern if kern[k] >= 0.97 * tmax), key=lambda k: (kwords[k], kern[k]))
        ach = kwords[dom] * 8 * N / (kern[dom] / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(dom)
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "kernel": dom,
                "alg_bytes_per_launch": kwords[dom] * 8 * N, "peak_source": peak_kind}
    w_upd = words_per_update(nd, filt is not None)
    step_ach = w_upd * 8 * N / (secs / K) / 1e9
    ctx.close()
    del phi, hist
    torch.cuda.empty_cache()

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        phi0 = torch.zeros(dims, dtype=torch.float64).pin_memory()
        scfg = W.SolveConfig(formulation=fc, scheme=cfg["scheme"], filter_config=filt, cfl=0.5,
                             tol=1e-15, max_iters=K, arith=args.arith)
        bnd = W.BoundarySpec(cfg["faces"])
        # untimed warm-up calls: the first solve allocates the page-locked
        # result buffer (~0.4 s) and the field workspace that later solves
        # recycle; reports dropped
        for _ in range(2):
            del_rep = W.solve_steady(grid, bnd, scfg, phi0=phi0, chunk=chunk)
            del del_rep
            gc.collect()  # the result array must be gone for its buffer to recycle
        torch.cuda.synchronize()
        # three complete timed solves (each: context, H2D, K steps, D2H), the
        # median reported and all samples listed
        samples = []
        for _ in range(3):
            barrier(world)
            t0 = time.perf_counter()
            rep = W.solve_steady(grid, bnd, scfg, phi0=phi0, chunk=chunk)
            torch.cuda.synchronize()
            samples.append(allreduce_max(time.perf_counter() - t0, world))
            assert rep.iters == K
            del rep
            gc.collect()
        t_e2e = sorted(samples)[1]
        e2e = {"value": N * K * world / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(N * 8 / K),
               "d2h_bytes_per_step": int((N * 8 + 8 * K) / K),
               "seconds": t_e2e, "samples_s": [round(x, 4) for x in samples],
               "includes": "median of 3 solve_steady calls, each: context setup + H2D phi0 "
                           "(pinned) + K steps + residual history + D2H phi (into pinned host "
                           "memory, returned as numpy)"}
    exact_side = None
    if args.arith == "fast" and not args.no_exact:
        exact_side = _device_steps(grid, cfg, fc, filt, K, Wm, "exact")
    ttc = _time_to_converge(secs_max / K * 1e3, args.arith)
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": round(secs_max / K * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "dims": list(dims), "arith": args.arith,
                       "global_nodes": N * world, "parallelism": "slab1 (single-GPU fused step)",
                       "l2": "inputs larger than L2 (1.07 GB per field)",
                       "fused": True if kern else False},
            "roofline": roof,
            "step_roofline": {"achieved": round(step_ach, 1), "peak": peak, "unit": "GB/s",
                              "frac": round(step_ach / peak, 4), "words_per_update": w_upd,
                              "model": "SURVEY 8(d) B_alg (21 stage words + 2 per filter "
                                       "sweep + 1 convergence read)",
                              "words_moved": (sum(kwords[k] for k in kwords)
                                              if kern else None)},
            "kernel_ms": {k: round(v, 4) for k, v in kern.items()},
            "kernel_rooflines": ({k: {"words": kwords[k],
                                      "achieved": round(kwords[k] * 8 * N / (v / 1e3) / 1e9, 1),
                                      "frac": round(kwords[k] * 8 * N / (v / 1e3) / 1e9 / peak, 4)}
                                  for k, v in kern.items()} if kern else None),
            "gpu_launches": K * (12 if kern else 0),
            "clocks": clk, "e2e": e2e,
            "exact_mode": exact_side, "time_to_converge": ttc}
    if rank == 0 and not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_sample(cfg, 9, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override grid size (debug)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--arith", default="fast", choices=["exact", "fast"],
                    help="fast: FMA + composite Laplacian (round-off differences, parity "
                         "within 1e-10); exact: bit-identical to the reference algorithm")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-mode side run")
    ap.add_argument("--dist", action="store_true", help="slab-decomposed path even at N=1")
    ap.add_argument("--no-overlap", action="store_true",
                    help="decomposed path: ghost exchange not overlapped with interior planes")
    ap.add_argument("--filter0", default=None, choices=["partitioned", "transpose"],
                    help="decomposed axis-0 filter (default: partitioned in fast arithmetic)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif world > 1 or args.dist:
        run_b200_dist(args, world, rank, local)
    else:
        run_b200(args, world, rank, local)
    import torch.distributed as tdist
    if tdist.is_available() and tdist.is_initialized():
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
