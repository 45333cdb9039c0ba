#!/usr/bin/env python
"""Pseudo-steps of one BASELINE configuration between cudaProfilerStart/Stop,
for `ncu --profile-from-start off` (launch lists and full captures of exactly
the profiled steps).

  python tools/profile_step.py [--case c4|c1|c2|c3|c5|c5p] [--arith fast|exact]
                               [--n 512] [--steps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def case(name, n):
    """(grid, faces, scheme, formulation, filter) of a BASELINE config."""
    import paper_2111_09859_b200 as W
    plate = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    if name == "c1":
        return (W.build_cartesian(201, 101, Lx=2.0, Ly=1.0), plate, "E4",
                W.FormulationConfig(kind="hj"), W.FilterConfig(0.49))
    if name == "c2":
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
        return (W.build_annulus(257, 129, scheme="C6"), faces, "C6",
                W.FormulationConfig(kind="hj_curvature"), W.FilterConfig(0.495))
    if name == "c3":
        return (W.build_sinusoidal_bump(1025, 513, scheme="E6"), plate, "E6",
                W.FormulationConfig(kind="hj"), W.FilterConfig(0.49))
    if name == "c5p":
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
                 "kmin": "periodic", "kmax": "periodic"}
        return (W.build_cylinder(1024, 512, 256, scheme="C6"), faces, "C6",
                W.FormulationConfig(kind="poisson"), W.FilterConfig(0.48))
    if name == "c5":
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
                 "kmin": "periodic", "kmax": "periodic"}
        return (W.build_cylinder(1024, 512, 256, scheme="C6"), faces, "C6",
                W.FormulationConfig(kind="hj_curvature"), W.FilterConfig(0.48))
    g = W.build_cartesian(n, n, n, Lx=n / 512, Ly=1.0, Lz=n / 512, periodic=(True, False, True))
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    return g, faces, "E6", W.FormulationConfig(kind="hj"), W.FilterConfig(0.49)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c4")
    ap.add_argument("--arith", default="fast")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch
    from paper_2111_09859_b200 import _context, _native as nat
    g, faces, scheme, fc, filt = case(args.case, args.n)
    ctx = _context.NativeSolver(g, faces, None, scheme, fc, filt, 0.5, 1e-15, 100,
                                arith=args.arith)
    phi = torch.zeros(tuple(g.dims), dtype=torch.float64, device="cuda")
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
