#!/usr/bin/env python
"""One pseudo-step of the bench workload between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch lists and full captures of exactly one
step).  Usage: python tools/profile_step.py [--arith fast|exact] [--n 512]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arith", default="fast")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2111_09859_b200 as W
    from paper_2111_09859_b200 import _context, _native as nat
    n = args.n
    g = W.build_cartesian(n, n, n, Lx=n / 512, Ly=1.0, Lz=n / 512, periodic=(True, False, True))
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    ctx = _context.NativeSolver(g, faces, None, "E6", W.FormulationConfig(kind="hj"),
                                W.FilterConfig(0.49), 0.5, 1e-15, 100, arith=args.arith)
    phi = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
    hist = torch.zeros(100, dtype=torch.float64, device="cuda")
    nat.check(ctx.lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
    for _ in range(2):
        nat.check(ctx.lib.wd_steps(ctx.ptr, 2))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        nat.check(ctx.lib.wd_steps(ctx.ptr, 1))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ctx.close()


if __name__ == "__main__":
    main()
