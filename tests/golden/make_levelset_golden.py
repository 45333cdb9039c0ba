"""Golden fixtures for the level-set burnback application (reference
walldist/levelset.py), made by running the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_levelset_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from walldist import grid as G  # noqa: E402
from walldist import levelset as LS  # noqa: E402


def main():
    out = {}
    g = G.build_cartesian(49, 49, Lx=2.0, Ly=2.0)
    star = LS.GrainShape.star(n_legs=6, center=(1.0, 1.0))
    out["star_poly"] = star.polygon
    pts = g.coords.reshape(2, -1).T
    out["inside"] = LS.point_in_polygon(pts, star.polygon).reshape(g.dims)
    sdf = LS.init_signed_distance(g, star)
    out["sdf0"] = sdf.values
    s = sdf
    for k in range(3):
        s = LS.levelset_step(s, 0.3, 0.01, scheme="UW")
        out[f"step{k + 1}"] = s.values
    out["step_aw"] = LS.levelset_step(sdf, 0.3, 0.01, scheme="E4", mode="as_written").values
    lines = LS.extract_isolines(sdf, 0.0)
    out["iso_n"] = np.array(len(lines))
    for q, ln in enumerate(lines):
        out[f"iso_{q}"] = ln
    out["iso_perim"] = np.array(LS.perimeter(lines))
    res = LS.burnback_run(g, LS.GrainShape.circle(0.5, center=(1.0, 1.0)), n_steps=4,
                          tracked_levels=(0.0, 0.05))
    out["bb_times"] = res.times
    out["bb_p0"] = res.perimeters[0.0]
    out["bb_p5"] = res.perimeters[0.05]
    out["bb_drift"] = res.grad_drift
    np.savez_compressed(os.path.join(HERE, "levelset.npz"), **out)
    print("wrote levelset.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
