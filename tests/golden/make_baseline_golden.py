"""Goldens at (or near) the BASELINE sizes of configs 2, 3 and 5, produced by
the CPU oracle (oracle/wd.py, pinned bit-for-bit to the reference by
tests/test_oracle_vs_reference.py).  These configs use EXTENSIONS (periodic
axes, E6, the annulus / sinusoidal-bump / cylinder generators), so the
oracle restatement is the source; no reference run exists for them.

Full fields are large (C3: 4.2 MB each), so a golden stores the residual
history of every step (bitwise), a SHA-256 of the field bytes after
``+ 0.0`` (which maps -0 to +0: the kernels skip the ``0 + x`` of Python
``sum`` and may differ in the sign of zero only), and a strided sample of
the field for diagnosis.  Usage (each case writes tests/golden/<name>.npz):

    python tests/golden/make_baseline_golden.py c2        # ~2,000 steps, ~4 min
    python tests/golden/make_baseline_golden.py c2full    # to tol 1e-8 / stall, long
    python tests/golden/make_baseline_golden.py c3hj c3eik c3lad
    python tests/golden/make_baseline_golden.py c5curv c5poisson          # 50 steps 128x64x32
    python tests/golden/make_baseline_golden.py c5conv_curv c5conv_poisson  # converged 64x32x16
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import wd  # noqa: E402

PLATE = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
RING = {"jmin": "wall", "jmax": "farfield"}


def field_hash(phi):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(phi, dtype=np.float64) + 0.0)
                          .tobytes()).hexdigest()


def sample(phi):
    sl = tuple(slice(None, None, max(1, n // 32)) for n in phi.shape)
    return np.ascontiguousarray(phi[sl])


def run(name, grid, faces, kind, scheme, af, tol, steps, phi0=None, store_field=False, **meta):
    cfg = wd.Config(wd.Formulation(kind), scheme, af, 0.5, tol, steps)
    t0 = time.time()
    rep = wd.solve(grid, wd.Boundary(faces), cfg, phi0=phi0, raise_on_divergence=False)
    dt = time.time() - t0
    out = dict(name=name, kind=kind, scheme=scheme, alpha_f=np.nan if af is None else af, tol=tol,
               max_iters=steps, iters=rep.iters, converged=rep.converged,
               diverged_at=-1 if rep.diverged_at is None else rep.diverged_at,
               residual_history=rep.residual_history, sha256=field_hash(rep.phi),
               sample=sample(rep.phi), phi_max=float(np.max(np.abs(rep.phi))), seconds=dt,
               **meta)
    if rep.phi_prime is not None:
        out["sha256_prime"] = field_hash(rep.phi_prime)
    if store_field:
        out["phi"] = rep.phi
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: iters={rep.iters} converged={rep.converged} diverged_at={rep.diverged_at} "
          f"{dt:.0f}s", flush=True)


def main(which):
    if which == "c2":
        g = wd.annulus(257, 129, scheme="C6")
        run("base_c2_annulus_curv_C6", g, RING, "hj_curvature", "C6", 0.495, 1e-8, 2000,
            store_field=True, dims=(257, 129))
    elif which == "c2full":
        g = wd.annulus(257, 129, scheme="C6")
        run("base_c2_annulus_curv_C6_full", g, RING, "hj_curvature", "C6", 0.495, 1e-8, 60000,
            store_field=True, dims=(257, 129))
    elif which in ("c3hj", "c3eik", "c3lad"):
        kind = {"c3hj": "hj", "c3eik": "eikonal", "c3lad": "hj_lad"}[which]
        steps = {"hj": 300, "eikonal": 3000, "hj_lad": 300}[kind]
        g = wd.sinusoidal_bump(1025, 513, scheme="E6")
        run(f"base_c3_bump_{kind}_E6", g, PLATE, kind, "E6", 0.49, 1e-8, steps, dims=(1025, 513))
    elif which in ("c5curv", "c5poisson"):
        kind = {"c5curv": "hj_curvature", "c5poisson": "poisson"}[which]
        g = wd.cylinder(128, 64, 32, scheme="C6")
        run(f"base_c5_cyl128_{kind}_C6", g, RING, kind, "C6", 0.48, 1e-8, 50,
            dims=(128, 64, 32))
    elif which in ("c5conv_curv", "c5conv_poisson"):
        kind = {"c5conv_curv": "hj_curvature", "c5conv_poisson": "poisson"}[which]
        dims = (64, 32, 16)
        g = wd.cylinder(*dims, scheme="C6")
        run(f"base_c5_cyl64_{kind}_C6_conv", g, RING, kind, "C6", 0.48, 1e-8, 40000,
            store_field=True, dims=dims)
    else:
        raise SystemExit(f"unknown case {which!r}")


if __name__ == "__main__":
    for w in sys.argv[1:]:
        main(w)
