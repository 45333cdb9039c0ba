#!/usr/bin/env python
"""Time-to-converge of the BASELINE configs through the public API
(solve_steady), one JSON line per run.  Times are CUDA-event loop seconds
(SolveReport.wall_seconds, the reference's timing semantics) plus the wall
clock of the whole call.

  python tools/converge.py c1 c3 c2 [--c4 fast|exact] [--c5-steps K]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def run(name, grid, faces, kind, scheme, af, tol, max_iters, arith="exact", exact_fn=None,
        chunk=None):
    import paper_2111_09859_b200 as W
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=kind), scheme=scheme,
                        filter_config=None if af is None else W.FilterConfig(af), tol=tol,
                        max_iters=max_iters, arith=arith)
    t0 = time.perf_counter()
    err = None
    try:
        rep = W.solve_steady(grid, W.BoundarySpec(faces), cfg, chunk=chunk)
    except Exception as exc:  # DivergenceError
        err = f"{type(exc).__name__}: {exc}"
        rep = None
    wall = time.perf_counter() - t0
    out = {"config": name, "dims": list(grid.dims), "kind": kind, "scheme": scheme,
           "alpha_f": af, "tol": tol, "arith": arith, "wall_s": round(wall, 3)}
    if rep is None:
        out["error"] = err
    else:
        n = int(np.prod(grid.dims))
        out.update(iters=rep.iters, converged=rep.converged,
                   loop_s=round(rep.loop_seconds, 4),
                   ms_per_iter=round(1e3 * rep.loop_seconds / max(rep.iters, 1), 4),
                   glups=round(n * rep.iters / max(rep.loop_seconds, 1e-12) / 1e9, 4),
                   final_change=float(rep.residual_history[-1]) if rep.iters else None)
        if exact_fn is not None:
            phi = rep.phi
            ex = exact_fn(grid)
            out["max_err"] = float(np.max(np.abs(phi - ex)))
            out["max_err_near_wall"] = float(np.max(np.abs(phi - ex)[ex <= 0.1 * ex.max()]))
            out["max_err_within_2"] = float(np.max(np.abs(phi - ex)[ex <= 2.0]))
    print(json.dumps(out), flush=True)
    return rep


def main():
    import paper_2111_09859_b200 as W
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c3", "c2"])
    ap.add_argument("--c4", default=None)
    ap.add_argument("--c4-n", type=int, default=512)
    ap.add_argument("--c5-steps", type=int, default=0)
    ap.add_argument("--c5-dims", default="1024x512x256")
    ap.add_argument("--c5-converge", type=int, default=0,
                    help="max_iters of a C5 HJ-curvature fast solve to tol 1e-8 (full size)")
    args = ap.parse_args()
    wall_plate = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    if "c1" in args.configs:
        g = W.build_cartesian(201, 101, Lx=2.0, Ly=1.0)
        run("c1_plate_201x101_hj_E4_F0.49", g, wall_plate, "hj", "E4", 0.49, 1e-8, 50000,
            exact_fn=lambda gr: gr.y)
    if "c3" in args.configs:
        g = W.build_sinusoidal_bump(1025, 513, scheme="E6")
        for kind, sch, af in (("hj", "E6", 0.49), ("hj", "E4", 0.49)):
            run(f"c3_sinbump_1025x513_{kind}_{sch}", g, wall_plate, kind, sch, af, 1e-8, 300000)
    if "c2" in args.configs:
        g = W.build_annulus(257, 129, scheme="C6")
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
        for kind, af in (("hj_curvature", 0.495), ("hj", 0.48)):
            run(f"c2_annulus_257x129_{kind}_C6", g, faces, kind, "C6", af, 1e-8, 200000,
                exact_fn=lambda gr: np.hypot(gr.x, gr.y) - 0.5)
    if args.c4:
        n = args.c4_n
        g = W.build_channel3d(n)
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
                 "kmin": "periodic", "kmax": "periodic"}
        run(f"c4_channel3d_{n}^3_hj_E6_F0.49", g, faces, "hj", "E6", 0.49, 1e-8, 400000,
            arith=args.c4, exact_fn=lambda gr: np.minimum(gr.y, 1.0 - gr.y), chunk=16)
    if args.c5_steps:
        g = W.build_cylinder(1024, 512, 256, scheme="C6")
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
                 "kmin": "periodic", "kmax": "periodic"}
        for kind, af in (("hj_curvature", 0.48), ("poisson", None)):
            run(f"c5_cylinder_1024x512x256_{kind}_C6", g, faces, kind, "C6", af, 1e-30,
                args.c5_steps)


    if args.c5_converge:
        n5 = tuple(int(v) for v in args.c5_dims.split("x"))
        g = W.build_cylinder(*n5, scheme="C6")
        faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
                 "kmin": "periodic", "kmax": "periodic"}
        run(f"c5_cylinder_{args.c5_dims}_hj_curvature_C6_F0.48", g, faces, "hj_curvature", "C6",
            0.48, 1e-8, args.c5_converge, arith="fast",
            exact_fn=lambda gr: np.hypot(gr.x, gr.y) - 0.5, chunk=8)


if __name__ == "__main__":
    main()
