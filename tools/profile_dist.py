#!/usr/bin/env python
"""Per-GPU cost of the slab-decomposed step measured on ONE GPU: rank 0 of a
P-way split of the 512^3 workload runs alone with the "solo" communicator
(its slab wraps onto itself; ghost planes, carries and pencils move as
device copies of the real volume), captured in the same CUDA graph as the
NCCL program.  Prints one JSON line per P: ms per step of the rank, the
single-GPU fused step measured in the same process, and the parallel
efficiency the kernels alone would allow (no NVLink time: an upper bound).
Also the profiling target for ncu (--profile: cudaProfilerStart/Stop around
the timed steps, use with --profile-from-start off).

  python tools/profile_dist.py [--P 1 2 4 8] [--n 512] [--filter0 partitioned|transpose]
                               [--steps 20] [--no-overlap] [--profile]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FACES = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
         "kmin": "periodic", "kmax": "periodic"}


def timed(stream, fn, K):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done = 0
    while done < K:
        fn(2)
        done += 2
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / done


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--filter0", default=None)
    ap.add_argument("--arith", default="fast")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    import ctypes
    import torch
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import dist, _context, _native as nat
    n = args.n
    g = W.build_cartesian(n, n, n, Lx=n / 512, Ly=1.0, Lz=n / 512, periodic=(True, False, True))
    fc = W.FormulationConfig(kind="hj")
    filt = W.FilterConfig(0.49)
    cfg = W.SolveConfig(formulation=fc, scheme="E6", filter_config=filt, tol=1e-15,
                        max_iters=10**9, arith=args.arith)
    K = args.steps
    # the single-GPU fused step, same process
    ctx = _context.NativeSolver(g, FACES, None, "E6", fc, filt, 0.5, 1e-15, 10**9, arith=args.arith)
    phi = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    hist = torch.zeros(K + 64, dtype=torch.float64, device="cuda")
    nat.check(ctx.lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
    step1 = lambda k: nat.check(ctx.lib.wd_steps(ctx.ptr, k))
    step1(2), step1(2)
    torch.cuda.synchronize()
    ms1 = timed(ctx.stream(), step1, K)
    ctx.close()
    del phi
    torch.cuda.empty_cache()
    for P in args.P:
        comm = dist.SoloComm(P, 0)
        ds = dist.DistributedSolve(g, FACES, cfg, comm, filter0=args.filter0,
                                   overlap=not args.no_overlap, hist_len=K + 64)
        ds.bind(None)
        ds.steps(2), ds.steps(2)
        torch.cuda.synchronize()
        if args.profile:
            torch.cuda.profiler.start()
        ms = timed(ds.stream(), ds.steps, K)
        if args.profile:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        st = ds.status()
        print(json.dumps({"P": P, "nl": ds.nl, "ms_per_step_rank": round(ms, 4),
                          "ms_per_step_single_gpu": round(ms1, 4),
                          "kernel_bound_efficiency": round(ms1 / (P * ms), 4),
                          "filter0": ds.filter0, "overlap": ds.overlap, "graph": ds.graph,
                          "state": st.state, "iters": st.iters}), flush=True)
        ds.close()
        comm.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
