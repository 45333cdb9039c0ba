"""The oracle against the reference-generated golden fixtures (CPU only).

This is the oracle's pin on machines without /root/reference (the GPU box):
every fixture in tests/golden/ was produced by running the reference.
Long solves are marked slow-ish but still run (seconds each) except C1.
"""
import numpy as np
import pytest

import goldens
from helpers import same
from oracle import wd


def test_operators_golden():
    z = goldens.load("operators")
    for s in ("E2", "E4", "C4", "C6"):
        for ax in range(2):
            assert same(wd.deriv(z["f2"], s, ax), z[f"d_{s}_2d_{ax}"])
        for ax in range(3):
            assert same(wd.deriv(z["f3"], s, ax), z[f"d_{s}_3d_{ax}"])
    for ax in range(3):
        assert same(wd.d4(z["f3"], ax), z[f"d4_3d_{ax}"])
    for af in (0.4, 0.48, 0.49, 0.495, 0.5):
        tag = f"{af:.3f}".replace(".", "p")
        for ax in range(2):
            assert same(wd.apply_filter(z["f2"], ax, af, pinned=z["pin2"]),
                        z[f"filt_{tag}_2d_{ax}"])
        for ax in range(3):
            assert same(wd.apply_filter(z["f3"], ax, af), z[f"filt_{tag}_3d_{ax}"])
    for n in range(3, 13):
        assert same(wd.apply_filter(z[f"short_in_{n}"], 1, 0.49), z[f"short_out_{n}"])


def test_residuals_golden():
    z = goldens.load("residuals")
    g = wd.Grid(z["coords"], z["metrics"], z["jacobian"])
    for kind in ("eikonal", "hj", "hj_lad", "hj_curvature", "poisson"):
        fc = wd.Formulation(kind=kind)
        for s in ("UW", "E2", "E4", "C4", "C6"):
            assert same(wd.tendency(z["phi"], g, s, fc), z[f"k_{kind}_{s}"]), (kind, s)
            assert same(wd.local_timestep(z["phi"], g, fc, 0.5, s), z[f"dt_{kind}_{s}"])
    for s in ("E2", "E4", "C4", "C6"):
        assert same(wd.poisson_post(z["pp"], g, s), z[f"post_{s}"])
        assert same(wd.compute_metrics(wd.Grid(z["coords"].copy()), s).metrics,
                    z[f"metrics_{s}"])


def _run(z, iters=None):
    g = wd.Grid(z["coords"], z["metrics"], z["jacobian"])
    faces = goldens.case_faces(z)
    mask = z.get("solid_mask")
    cfg = wd.Config(wd.Formulation(kind=str(z["kind"])), str(z["scheme"]), goldens.case_alpha(z),
                    float(z["cfl"]), float(z["tol"]), int(z["max_iters"]))
    return wd.solve(g, wd.Boundary(faces, mask), cfg, raise_on_divergence=False,
                    max_iters=iters)


SHORT = [c for c in goldens.solve_cases()
         if not c.startswith(("c1_", "channel101", "sinbump129"))]


@pytest.mark.parametrize("case", SHORT)
def test_short_solves_golden(case):
    z = goldens.load("solve_" + case)
    rep = _run(z)
    assert rep.iters == int(z["iters"])
    assert same(rep.residual_history, z["residual_history"])
    if int(z["diverged"]) > 0:
        assert rep.diverged_at == int(z["diverged"])
    else:
        assert same(rep.phi, z["phi"])


def test_c1_prefix_golden():
    """First 300 iterations of the C1 flat-plate solve, bit-for-bit."""
    z = goldens.load("solve_c1_plate_hj_E4")
    rep = _run(z, iters=300)
    assert same(rep.residual_history, z["residual_history"][:300])


def test_c2_converged_golden_matches_exact_distance_near_wall():
    """BASELINE config 2 run to tol 1e-8 by the oracle (5,078 iterations):
    the field is the wall distance d = r - 0.5 to 1e-4 within two wall units
    (the far-field outer boundary bends the HJ solution further out)."""
    import goldens
    from oracle import wd
    z = goldens.load("base_c2_annulus_curv_C6_full")
    assert bool(z["converged"]) and int(z["iters"]) == 5078
    g = wd.annulus(257, 129, scheme="C6")
    d = np.sqrt(g.coords[0] ** 2 + g.coords[1] ** 2) - 0.5
    near = (d > 0) & (d <= 2.0)
    assert np.max(np.abs(z["phi"] - d)[near]) <= 1e-4
    assert np.max(np.abs(z["phi"] - d)[(d > 0) & (d <= 1.0)]) <= 1e-5
