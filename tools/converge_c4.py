#!/usr/bin/env python
"""Measured time-to-converge of the bench workload (BASELINE config 4:
512^3 channel, HJ eps=0.2, E6, filter 0.49, CFL 0.5, tol 1e-8) through the
public API (solve_steady), checked against the oracle.

The 512^3 field is x/z-invariant, so the oracle's answer is the 5 x 512 x 5
strip with the same spacings (tests/golden/strip_c4_ny512.npz, produced by
tests/golden/make_strip_golden.py with the oracle, which is pinned bitwise to
the reference).  Checks (north_star): |iters - oracle iters| <= 1 and
max |phi - profile| <= 1e-10 * max(profile) over all 512^3 nodes.

  python tools/converge_c4.py [--arith fast|exact] [--out gpurun_out/converge_c4.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arith", default="fast")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "converge_c4.json"))
    ap.add_argument("--comm", default=None,
                    help="run the slab-decomposed program: 'nccl1' (one-rank NCCL communicator; "
                         "set WD_NCCL_SELF=1 for real NCCL calls) or 'soloP' (rank 0 of a P-way "
                         "split alone: the field is x-invariant, so its 512/P planes wrapped "
                         "onto themselves are the same problem)")
    args = ap.parse_args()
    import torch
    import paper_2111_09859_b200 as W
    gold = np.load(os.path.join(ROOT, "tests", "golden", f"strip_c4_ny{args.n}.npz"))
    n = args.n
    g = W.build_channel3d(n)
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E6",
                        filter_config=W.FilterConfig(0.49), cfl=0.5, tol=float(gold["tol"]),
                        max_iters=int(gold["iters"]) + 20000, arith=args.arith)
    comm = None
    if args.comm:
        from paper_2111_09859_b200 import dist
        comm = dist.NcclComm(0, 1) if args.comm == "nccl1" else dist.SoloComm(int(args.comm[4:]), 0)
    t0 = time.perf_counter()
    rep = W.solve_steady(g, W.BoundarySpec(faces), cfg, device_result=True, comm=comm)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    phi = rep.phi
    prof = torch.from_numpy(np.asarray(gold["profile"], dtype=np.float64)).to(phi.device)
    dev = (phi - prof.view(1, n, 1)).abs().max().item()
    pmax = float(np.max(gold["profile"]))
    exact = torch.minimum(torch.linspace(0, 1, n, dtype=torch.float64, device=phi.device),
                          1 - torch.linspace(0, 1, n, dtype=torch.float64, device=phi.device))
    err_exact = (phi - exact.view(1, n, 1)).abs().max().item()
    gh = np.asarray(gold["residual_history"])
    m = min(len(gh), rep.iters)
    hist_rel = float(np.max(np.abs(rep.residual_history[:m] - gh[:m]) /
                            np.maximum(np.abs(gh[:m]), 1e-300))) if m else None
    out = {
        "config": f"c4_channel3d_{n}^3_hj_E6_F0.49",
        "arith": args.arith,
        "program": args.comm or "single GPU",
        "tol": float(gold["tol"]),
        "iters": int(rep.iters),
        "converged": bool(rep.converged),
        "oracle_iters": int(gold["iters"]),
        "iters_delta": int(rep.iters) - int(gold["iters"]),
        "measured_seconds": round(rep.loop_seconds, 3),
        "call_wall_seconds": round(wall, 3),
        "ms_per_iter": round(1e3 * rep.loop_seconds / max(rep.iters, 1), 4),
        "glups": round(n ** 3 * rep.iters / rep.loop_seconds / 1e9, 3),
        "max_abs_dev_vs_oracle_profile": dev,
        "rel_dev_vs_oracle_profile": dev / pmax,
        "max_abs_err_vs_exact_min_y_1my": err_exact,
        "history_max_rel_dev_vs_oracle": hist_rel,
        "final_change": float(rep.residual_history[-1]),
        "oracle": "tests/golden/strip_c4_ny512.npz: oracle/wd.py (pinned bitwise to the "
                  "reference) on the x/z-invariant 5 x 512 x 5 periodic strip",
        "pass": bool(abs(int(rep.iters) - int(gold["iters"])) <= 1 and dev <= 1e-10 * pmax),
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
