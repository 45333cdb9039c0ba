"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--full]

Writes small .npz files next to this script.  Inputs are seeded and fully
described in each file, so the GPU-side tests can rebuild them without the
reference.  ``--full`` also runs the long reference solves (C1 flat plate to
tol 1e-8: 18,440 iterations, ~3 min on one core).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from walldist import formulations as F  # noqa: E402
from walldist import grid as G  # noqa: E402
from walldist import operators as O  # noqa: E402
from walldist import solver as S  # noqa: E402

FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {name}.npz ({os.path.getsize(path) / 1024:.1f} KiB)")


def operators_fixture():
    """Seeded line-operator inputs/outputs (operators.py:94-352)."""
    rng = np.random.default_rng(2111)
    out = {}
    f2 = rng.standard_normal((13, 17))
    f3 = rng.standard_normal((7, 9, 11))
    out["f2"], out["f3"] = f2, f3
    for s in ("E2", "E4", "C4", "C6"):
        for ax in range(2):
            out[f"d_{s}_2d_{ax}"] = O.central_derivative(f2, s, ax)
        for ax in range(3):
            out[f"d_{s}_3d_{ax}"] = O.central_derivative(f3, s, ax)
    for ax in range(3):
        out[f"d4_3d_{ax}"] = O.fourth_derivative(f3, ax)
    pin = rng.random(f2.shape) < 0.1
    out["pin2"] = pin
    for af in (0.4, 0.48, 0.49, 0.495, 0.5):
        tag = f"{af:.3f}".replace(".", "p")
        for ax in range(2):
            out[f"filt_{tag}_2d_{ax}"] = O.apply_filter(f2, ax, O.FilterConfig(af), pinned=pin)
        for ax in range(3):
            out[f"filt_{tag}_3d_{ax}"] = O.apply_filter(f3, ax, O.FilterConfig(af))
    # short filter lines (3..11 fall back to reduced order everywhere)
    for n in range(3, 13):
        g = rng.standard_normal((3, n))
        out[f"short_in_{n}"] = g
        out[f"short_out_{n}"] = O.apply_filter(g, 1, O.FilterConfig(0.49))
    save("operators", **out)


def residual_fixture():
    """Tendencies and time steps of every formulation x scheme on the
    reference bump grid (formulations.py:232-252, solver.py:160-180)."""
    g = G.build_bump_grid(41, 21, scheme="E4")
    rng = np.random.default_rng(7)
    y = g.y
    phi = np.abs(y - y.min()) + 1e-3 * rng.standard_normal(g.dims)
    out = dict(coords=g.coords, metrics=g.metrics, jacobian=g.jacobian, phi=phi)
    for kind in F.FORMULATIONS:
        fc = F.FormulationConfig(kind=kind)
        for s in ("UW", "E2", "E4", "C4", "C6"):
            out[f"k_{kind}_{s}"] = F.tendency(phi, g, s, fc)
            out[f"dt_{kind}_{s}"] = S.local_timestep(phi, g, fc, 0.5, s)
    pp = 0.05 * np.abs(phi)
    for s in ("E2", "E4", "C4", "C6"):
        out[f"post_{s}"] = F.poisson_postprocess(pp, g, s)
        out[f"metrics_{s}"] = G.compute_metrics(G.CurvilinearGrid(coords=g.coords.copy()), s).metrics
    out["pp"] = pp
    save("residuals", **out)


SHORT = [
    # name, grid, faces, kind, scheme, alpha_f, cfl, iters
    ("plate_hj_E4", ("cart", 41, 21, 2.0, 1.0), ("farfield", "farfield", "wall", "farfield"), "hj", "E4", 0.49, 0.5, 60),
    ("channel_hj_C6", ("cart", 25, 25, 1.0, 1.0), ("farfield", "farfield", "wall", "wall"), "hj", "C6", 0.48, 0.5, 40),
    ("channel_hj_C4", ("cart", 25, 25, 1.0, 1.0), ("farfield", "farfield", "wall", "wall"), "hj", "C4", 0.49, 0.5, 40),
    ("bump_curv_E4", ("bump", 41, 21), ("farfield", "farfield", "wall", "farfield"), "hj_curvature", "E4", 0.495, 0.5, 40),
    ("bump_curv_C6", ("bump", 41, 21), ("farfield", "farfield", "wall", "farfield"), "hj_curvature", "C6", 0.48, 0.5, 40),
    ("bump_lad_E4", ("bump", 41, 21), ("farfield", "farfield", "wall", "farfield"), "hj_lad", "E4", 0.49, 0.1, 40),
    ("bump_eik_E2", ("bump", 41, 21), ("farfield", "farfield", "wall", "farfield"), "eikonal", "E2", 0.49, 0.5, 40),
    ("bump_poisson_C6", ("bump", 41, 21), ("farfield", "farfield", "wall", "farfield"), "poisson", "C6", None, 0.5, 40),
    ("plate_hj_UW", ("cart", 41, 21, 2.0, 1.0), ("farfield", "farfield", "wall", "farfield"), "hj", "UW", None, 0.5, 40),
    ("plate_eik_UW", ("cart", 41, 21, 2.0, 1.0), ("farfield", "farfield", "wall", "farfield"), "eikonal", "UW", None, 0.5, 40),
    ("box3d_hj_E4", ("cart3", 11, 12, 13), ("farfield", "farfield", "wall", "wall", "farfield", "farfield"), "hj", "E4", 0.49, 0.5, 30),
    ("box3d_walls_hj_E4", ("cart3", 11, 12, 13), ("wall",) * 6, "hj", "E4", 0.49, 0.5, 30),
    ("box3d_curv_C6", ("cart3", 11, 12, 13), ("wall", "wall", "farfield", "wall", "farfield", "farfield"), "hj_curvature", "C6", 0.48, 0.5, 20),
]


def _grid(spec):
    if spec[0] == "cart":
        return G.build_cartesian(spec[1], spec[2], Lx=spec[3], Ly=spec[4])
    if spec[0] == "cart3":
        return G.build_cartesian(spec[1], spec[2], spec[3], Lx=1.0, Ly=1.1, Lz=1.2)
    return G.build_bump_grid(spec[1], spec[2], scheme="E4")


def run_case(name, spec, faces, kind, scheme, af, cfl, iters, tol=1e-12, mask=None):
    g = _grid(spec) if not isinstance(spec, G.CurvilinearGrid) else spec
    fc = dict(zip(FACES, faces))
    cfg = S.SolveConfig(formulation=F.FormulationConfig(kind=kind), scheme=scheme,
                        filter_config=None if af is None else O.FilterConfig(af),
                        cfl=cfl, tol=tol, max_iters=iters)
    t0 = time.perf_counter()
    diverged = -1
    try:
        r = S.solve_steady(g, S.BoundarySpec(fc, mask), cfg)
    except S.DivergenceError:
        # the reference does not report where; replay its own step functions
        bnd = S.BoundarySpec(fc, mask)
        phi = S.apply_boundary_conditions(g.new_field(), bnd)
        hist = []
        while True:
            dt = S.local_timestep(phi, g, cfg.formulation, cfg.cfl, cfg.scheme)
            try:
                new = S.rk4_step(phi, g, cfg, dt, bnd)
            except S.DivergenceError:
                diverged = len(hist) + 1
                break
            hist.append(float(np.max(np.abs(new - phi))) / g.ref_length)
            phi = new
        r = S.SolveReport(phi=phi, iters=len(hist), residual_history=np.asarray(hist),
                          wall_seconds=np.zeros(len(hist)), converged=False)
        print(name, "diverged at iteration", diverged)
    dt = time.perf_counter() - t0
    print(f"{name}: iters={r.iters} converged={r.converged} {dt:.1f}s")
    kw = dict(coords=g.coords, metrics=g.metrics, jacobian=g.jacobian,
              faces=np.array(faces), kind=kind, scheme=scheme,
              alpha_f=np.nan if af is None else af, cfl=cfl, tol=tol, max_iters=iters,
              iters=r.iters, converged=r.converged, residual_history=r.residual_history,
              phi=r.phi, diverged=diverged, seconds_per_iter=dt / max(r.iters, 1))
    if mask is not None:
        kw["solid_mask"] = mask
    if r.phi_prime is not None:
        kw["phi_prime"] = r.phi_prime
    save("solve_" + name, **kw)


def short_solves():
    for case in SHORT:
        run_case(*case)
    g = G.build_cartesian(21, 21)
    mask = np.zeros(g.dims, bool)
    mask[8:12, 6:10] = True
    run_case("mask_hj_E4", g, ("farfield",) * 4, "hj", "E4", 0.49, 0.5, 30, mask=mask)


def divergence_fixture():
    """HJ-E4 without the filter diverges; record where."""
    g = G.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    fc = dict(zip(FACES, ("farfield", "farfield", "wall", "farfield")))
    cfg = S.SolveConfig(formulation=F.FormulationConfig(kind="hj"), scheme="E4",
                        cfl=0.5, tol=1e-12, max_iters=5000)
    # count iterations by running with growing caps (reference does not
    # report the failing iteration)
    lo, hi = 0, 5000
    while hi - lo > 1:
        mid = (lo + hi) // 2
        try:
            S.solve_steady(g, S.BoundarySpec(fc), S.SolveConfig(**{**cfg.__dict__, "max_iters": mid}))
            lo = mid
        except Exception:
            hi = mid
    print("divergence at iteration", hi)
    save("diverge_plate_E4", diverged_at=hi, faces=np.array(list(fc.values())))


def long_solves():
    # C1 (BASELINE config 1): flat plate 201x101, HJ-E4 + F0.49, tol 1e-8
    g = G.build_cartesian(201, 101, Lx=2.0, Ly=1.0)
    run_case("c1_plate_hj_E4", g, ("farfield", "farfield", "wall", "farfield"),
             "hj", "E4", 0.49, 0.5, 50000, tol=1e-8)
    # channel 101^2, HJ-E4 + F0.49, default tol 1e-5 (2,364)
    g = G.build_cartesian(101, 101)
    run_case("channel101_hj_E4", g, ("farfield", "farfield", "wall", "wall"),
             "hj", "E4", 0.49, 0.5, 50000, tol=1e-5)
    # channel 101^2, HJ-C6 + F0.48 (App. C: 2,364)
    run_case("channel101_hj_C6", g, ("farfield", "farfield", "wall", "wall"),
             "hj", "C6", 0.48, 0.5, 50000, tol=1e-5)
    # sinusoidal bump 129x65 (beta = 2) HJ-E4 + F0.49 to 1e-8 (App. C: 2,158)
    x = np.linspace(0.0, 4.0, 129)
    s = np.linspace(0.0, 1.0, 65)
    t = 1.0 + np.tanh(2.0 * (s - 1.0)) / np.tanh(2.0)
    yw = 0.1 * np.sin(2.0 * np.pi * x)
    X = np.repeat(x[:, None], 65, axis=1)
    Y = yw[:, None] * (1.0 - t[None, :]) + t[None, :]
    gb = G.compute_metrics(G.CurvilinearGrid(coords=np.stack([X, Y])), "E4")
    run_case("sinbump129_hj_E4", gb, ("farfield", "farfield", "wall", "farfield"),
             "hj", "E4", 0.49, 0.5, 50000, tol=1e-8)
    run_case("sinbump129_curv_E4", gb, ("farfield", "farfield", "wall", "farfield"),
             "hj_curvature", "E4", 0.495, 0.5, 50000, tol=1e-8)
    # channel 101^2 Poisson-E4 (App. C: 3,697)
    run_case("channel101_poisson_E4", g, ("farfield", "farfield", "wall", "wall"),
             "poisson", "E4", None, 0.5, 50000, tol=1e-5)


if __name__ == "__main__":
    operators_fixture()
    residual_fixture()
    short_solves()
    divergence_fixture()
    if "--full" in sys.argv:
        long_solves()
