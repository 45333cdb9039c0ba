"""Converged C4-strip goldens from the CPU oracle (EXTENSION configs: E6 and
periodic axes do not exist in the reference, so the oracle restatement --
pinned bit-for-bit to the reference on every shared path -- is the source).

BASELINE config 4 (512^3 channel, walls y = 0, 1, periodic x and z, HJ E6,
F 0.49) has an x/z-invariant solution (up to round-off: the cyclic filter of
a constant line is not exactly constant), so the (5, ny, 5) strip with the
same spacings gives the iteration count and profile of the full grid; the
full strip field is stored for bit-exact comparison on the same grid.  Usage:
    python tests/golden/make_strip_golden.py 129      # ~1 min
    python tests/golden/make_strip_golden.py 512      # BASELINE C4 column, long
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import wd  # noqa: E402


def main(ny, tol=1e-8, max_iters=200000):
    n = 512 if ny == 512 else ny
    # same spacings as the n^3 channel on [0,1]^3 (dx = dz = 1/n, dy = 1/(ny-1))
    g = wd.cartesian(5, ny, 5, Lx=5.0 / n, Ly=1.0, Lz=5.0 / n, periodic=(True, False, True))
    bnd = wd.Boundary({"jmin": "wall", "jmax": "wall"})
    cfg = wd.Config(wd.Formulation("hj", epsilon=0.2), "E6", 0.49, 0.5, tol, max_iters)
    t0 = time.time()
    rep = wd.solve(g, bnd, cfg)
    dt = time.time() - t0
    print(f"ny={ny}: iters={rep.iters} converged={rep.converged} {dt:.0f}s")
    np.savez_compressed(os.path.join(HERE, f"strip_c4_ny{ny}.npz"), ny=ny, n=n, tol=tol,
                        iters=rep.iters, converged=rep.converged,
                        residual_history=rep.residual_history, profile=rep.phi[2, :, 2],
                        phi=rep.phi,
                        seconds=dt)


if __name__ == "__main__":
    main(int(sys.argv[1]))
