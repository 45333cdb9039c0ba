"""Golden fixtures for the moving-body loop, made by running the REFERENCE
``solve_unsteady`` (walldist/solver.py:392-410).

Run in the build container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_unsteady_golden.py

Per case: the grid/config description, and per physical step the body
mask, iteration count, residual history and field.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from walldist import grid as G  # noqa: E402
from walldist import formulations as F  # noqa: E402
from walldist import operators as O  # noqa: E402
from walldist import solver as S  # noqa: E402

CASES = {
    # name: (ni, nj, Lx, Ly, motion kwargs, scheme, alpha_f, kind, tol, max_iters, n_steps)
    "piston_hj_UW": (41, 21, 1.0, 0.5, dict(kind="piston_sinusoid", physical_dt=0.1),
                     "UW", None, "hj", 1e-4, 400, 4),
    "cube_hj_UW": (33, 33, 1.0, 1.0, dict(kind="bouncing_cube", physical_dt=0.15),
                   "UW", None, "hj", 1e-4, 400, 4),
}


def main():
    for name, (ni, nj, lx, ly, mk, scheme, af, kind, tol, mi, ns) in CASES.items():
        g = G.build_cartesian(ni, nj, Lx=lx, Ly=ly)
        motion = S.MotionSpec(**mk)
        cfg = S.SolveConfig(formulation=F.FormulationConfig(kind=kind), scheme=scheme,
                            filter_config=O.FilterConfig(af) if af else None, cfl=0.5,
                            tol=tol, max_iters=mi)
        reps = S.solve_unsteady(g, motion, cfg, ns)
        kw = dict(dims=np.array([ni, nj]), extents=np.array([lx, ly]),
                  motion_kind=np.array(mk["kind"]), physical_dt=np.array(mk["physical_dt"]),
                  scheme=np.array(scheme), alpha_f=np.array(np.nan if af is None else af),
                  kind=np.array(kind), tol=np.array(tol), max_iters=np.array(mi),
                  n_steps=np.array(ns), iters=np.array([r.iters for r in reps]),
                  times=np.array([r.time for r in reps]))
        for s, r in enumerate(reps):
            kw[f"mask_{s}"] = motion.body_mask(g, r.time)
            kw[f"res_{s}"] = r.residual_history
            kw[f"phi_{s}"] = r.phi
        path = os.path.join(HERE, f"unsteady_{name}.npz")
        np.savez_compressed(path, **kw)
        print(f"wrote {path}: iters {kw['iters'].tolist()}")


if __name__ == "__main__":
    main()
