"""Golden fixtures for the validation metrics (reference walldist/metrics.py),
made by running the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_metrics_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from walldist import formulations as F  # noqa: E402
from walldist import grid as G  # noqa: E402
from walldist import metrics as M  # noqa: E402
from walldist import operators as O  # noqa: E402
from walldist import solver as S  # noqa: E402


def main():
    rng = np.random.default_rng(2111)
    out = {}
    # brute-force oracle: bump grid nodes vs the wall polyline (2-D) and a
    # seeded 3-D cloud
    params = G.BumpParams()
    g = G.build_bump_grid(65, 33, params, "E4")
    wall = params.wall_polyline(4001)
    pts = g.coords.reshape(2, -1).T
    out["sw2_pts"], out["sw2_wall"] = pts, wall
    out["sw2_out"] = M.sampled_wall_distance(pts, wall)
    p3 = rng.uniform(-1, 1, (3000, 3))
    w3 = rng.uniform(-1, 1, (2500, 3))
    out["sw3_pts"], out["sw3_wall"], out["sw3_out"] = p3, w3, M.sampled_wall_distance(p3, w3)
    # L2 norm on a curvilinear grid (1/J weights)
    phi = rng.standard_normal(g.dims)
    ex = rng.standard_normal(g.dims)
    out["l2_phi"], out["l2_ex"], out["l2_jac"] = phi, ex, g.jacobian
    out["l2_out"] = np.array(M.l2_norm(phi, ex, g))
    # |grad phi| of a smooth field with E4 and C6 metrics
    for s in ("E4", "C6"):
        gs = G.build_bump_grid(65, 33, params, s)
        f = np.sin(2.0 * gs.x) * np.cos(3.0 * gs.y) + gs.y
        out[f"gm_{s}_in"] = f
        out[f"gm_{s}_out"] = M.gradient_magnitude(f, gs, s)
    # percentage errors / histogram
    exact = np.abs(rng.standard_normal(500))
    exact[:20] = 0.0
    approx = exact * (1.0 + 0.03 * rng.standard_normal(500))
    excl = rng.random(500) < 0.1
    out["pe_phi"], out["pe_exact"], out["pe_excl"] = approx, exact, excl
    out["pe_out"] = M.percentage_errors(approx, exact, exclude=excl)
    # L2 history sampled by solve_steady (solver.py:266-268)
    gp = G.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    cfg = S.SolveConfig(formulation=F.FormulationConfig(kind="hj"), scheme="E4",
                        filter_config=O.FilterConfig(0.49), tol=1e-12, max_iters=40, l2_every=5)
    rep = S.solve_steady(gp, S.BoundarySpec(faces), cfg, exact=gp.y.copy())
    out["l2h"] = np.asarray(rep.l2_history)
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print("wrote metrics.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
