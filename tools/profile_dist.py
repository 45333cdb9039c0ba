#!/usr/bin/env python
"""Pseudo-steps of the slab-decomposed path (dist.py) with P simulated ranks
on one GPU between cudaProfilerStart/Stop (ncu --profile-from-start off):
per-kernel costs of the decomposition at the 512^3 workload.

  python tools/profile_dist.py [--P 1] [--filter0 partitioned|transpose] [--steps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=1)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--filter0", default="partitioned")
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import dist
    n = args.n
    dims = (n, n, n)
    sp = (1.0 / n, 1.0 / (n - 1), 1.0 / n)
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    P = args.P
    ds = dist.DistributedSolve(dims, sp, faces, "E6", W.FormulationConfig(kind="hj"),
                               W.FilterConfig(0.49), 0.5, 1e-15, 100, "fast",
                               dist.LocalComm(P), list(range(P)), filter0=args.filter0)
    nl = n // P
    ds.set_state([torch.zeros((nl, n, n), dtype=torch.float64, device="cuda") for _ in range(P)])
    for _ in range(2):
        ds.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        ds.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ds.close()


if __name__ == "__main__":
    main()
