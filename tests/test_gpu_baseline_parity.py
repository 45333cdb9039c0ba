"""CUDA path vs the oracle at (or near) the BASELINE sizes of configs 2, 3 and 5.

Goldens come from tests/golden/make_baseline_golden.py (the CPU oracle,
pinned bit-for-bit to the reference on every shared path).  Exact mode must
match bit for bit: iteration count, every entry of the residual history, the
stop outcome (converged / stalled at max_iters / the divergence iteration)
and the field, compared through a SHA-256 of its bytes after ``+ 0.0``
(sign of zero normalised; the kernels skip the ``0 + x`` of Python ``sum``).
Fast mode on the converged C5 cylinder: iteration count within 1 and the
field within 1e-10 of max |phi| (north_star's tolerance).
"""
import hashlib
import re

import numpy as np
import pytest

import goldens

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2111_09859_b200")
from paper_2111_09859_b200.errors import DivergenceError  # noqa: E402

RING = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
CYL = dict(RING, kmin="periodic", kmax="periodic")
PLATE = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_09859_b200 import _native
    _native.lib()


def _hash(phi):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(phi, dtype=np.float64) + 0.0)
                          .tobytes()).hexdigest()


def _alpha(z):
    a = float(z["alpha_f"])
    return None if np.isnan(a) else a


def _solve(grid, faces, z, arith="exact", max_iters=None):
    """solve_steady with the golden's settings; returns (report | None,
    diverged_iter | None)."""
    af = _alpha(z)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=str(z["kind"])),
                        scheme=str(z["scheme"]),
                        filter_config=None if af is None else W.FilterConfig(af),
                        cfl=0.5, tol=float(z["tol"]),
                        max_iters=int(z["max_iters"]) if max_iters is None else max_iters,
                        arith=arith)
    try:
        return W.solve_steady(grid, W.BoundarySpec(faces), cfg), None
    except DivergenceError as exc:
        m = re.search(r"at iteration (\d+)", str(exc))
        return None, int(m.group(1)) if m else -2


def _check_exact(rep, div, z):
    if int(z["diverged_at"]) > 0:
        assert rep is None and div == int(z["diverged_at"]), (div, int(z["diverged_at"]))
        return
    assert rep is not None, f"diverged at {div}"
    assert rep.iters == int(z["iters"])
    assert rep.converged == bool(z["converged"])
    assert np.array_equal(rep.residual_history, z["residual_history"])
    assert _hash(rep.phi) == str(z["sha256"])
    if "sha256_prime" in z:
        assert _hash(rep.phi_prime) == str(z["sha256_prime"])


# --------------------------------------------------------------- config 2
def test_c2_annulus_257x129_curvature_c6_2000_steps_exact():
    z = goldens.load("base_c2_annulus_curv_C6")
    g = W.build_annulus(257, 129, scheme="C6")
    rep, div = _solve(g, RING, z)
    _check_exact(rep, div, z)
    assert np.array_equal(rep.phi, z["phi"])


def test_c2_annulus_257x129_curvature_c6_outcome_exact():
    """The oracle's whole run (to tol 1e-8 or its stall at max_iters)."""
    z = goldens.load("base_c2_annulus_curv_C6_full")
    g = W.build_annulus(257, 129, scheme="C6")
    rep, div = _solve(g, RING, z)
    _check_exact(rep, div, z)
    assert np.array_equal(rep.phi, z["phi"])
    # the converged field against the configuration's exact answer d = r - 0.5:
    # within 1e-4 out to two wall units (5.7e-6 within one); the HJ solution
    # with a far-field outer boundary drifts from the distance further out
    d = np.sqrt(g.coords[0] ** 2 + g.coords[1] ** 2) - 0.5
    near = (d > 0) & (d <= 2.0)
    assert rep.converged and np.max(np.abs(rep.phi - d)[near]) <= 1e-4


def test_c2_annulus_257x129_curvature_c6_fast_converges_like_the_oracle():
    """Fast arithmetic (scan derivatives, Thomas factor) on the whole config-2
    run: the oracle's 5,078 iterations within 1, field within 1e-10 * max."""
    z = goldens.load("base_c2_annulus_curv_C6_full")
    g = W.build_annulus(257, 129, scheme="C6")
    rep, div = _solve(g, RING, z, arith="fast")
    assert rep is not None and rep.converged
    assert abs(rep.iters - int(z["iters"])) <= 1, rep.iters
    assert np.max(np.abs(rep.phi - z["phi"])) <= 1e-10 * float(np.max(np.abs(z["phi"])))


# --------------------------------------------------------------- config 3
@pytest.mark.parametrize("kind", ["hj", "eikonal", "hj_lad"])
def test_c3_bump_1025x513_e6_exact(kind):
    z = goldens.load(f"base_c3_bump_{kind}_E6")
    g = W.build_sinusoidal_bump(1025, 513, scheme="E6")
    rep, div = _solve(g, PLATE, z)
    _check_exact(rep, div, z)


@pytest.mark.parametrize("kind", ["hj", "eikonal"])
def test_c3_bump_1025x513_e6_fast(kind):
    """Fast arithmetic on config 3: lines of 1025 / 513 rows take the
    long-line scan filter (wd_filter_long.cuh).  Against the exact mode (bit
    identical to the oracle, above) over the golden's steps (300 / 1,033): the
    residual history to 1e-9 relative + 1e-13 absolute (the change per step
    falls to 1e-8, where round-off of phi ~ 0.06 shows), the field to
    1e-10 * max|phi| (north_star)."""
    z = goldens.load(f"base_c3_bump_{kind}_E6")
    g = W.build_sinusoidal_bump(1025, 513, scheme="E6")
    ex, _ = _solve(g, PLATE, z)
    fa, _ = _solve(g, PLATE, z, arith="fast")
    assert fa is not None and fa.iters == ex.iters
    np.testing.assert_allclose(fa.residual_history, ex.residual_history, rtol=1e-9, atol=1e-13)
    assert np.max(np.abs(fa.phi - ex.phi)) <= 1e-10 * float(np.max(np.abs(ex.phi)))


@pytest.mark.parametrize("dims", [(1024, 65), (700, 67), (2048, 33)])
def test_long_periodic_lines_fast_filter(dims):
    """The long-line scan filter on cyclic lines (a strip periodic in x with
    513..2048 rows per line; partial line tiles and partial segments; all
    three register-window instantiations) on rough data."""
    g = W.build_cartesian(*dims, Lx=dims[0] / 100.0, Ly=1.0, periodic=(True, False))
    rng = np.random.default_rng(dims[0])
    phi0 = 1e-3 * rng.random(dims)
    reps = []
    for arith in ("exact", "fast"):
        cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E6",
                            filter_config=W.FilterConfig(0.49), tol=1e-15, max_iters=40,
                            arith=arith)
        reps.append(W.solve_steady(g, W.BoundarySpec(RING), cfg, phi0=phi0))
    ex, fa = reps
    np.testing.assert_allclose(fa.residual_history, ex.residual_history, rtol=1e-9, atol=1e-15)
    assert np.max(np.abs(fa.phi - ex.phi)) <= 1e-12 * max(1.0, float(np.max(np.abs(ex.phi))))


# --------------------------------------------------------------- config 5
@pytest.mark.parametrize("kind", ["hj_curvature", "poisson"])
def test_c5_cylinder_128x64x32_c6_50_steps_exact(kind):
    z = goldens.load(f"base_c5_cyl128_{kind}_C6")
    g = W.build_cylinder(128, 64, 32, scheme="C6")
    rep, div = _solve(g, CYL, z)
    _check_exact(rep, div, z)


@pytest.mark.parametrize("kind", ["hj_curvature", "poisson"])
def test_c5_cylinder_64x32x16_c6_converged_fast(kind):
    """Fast arithmetic (scan derivatives / scan filter) to tol 1e-8: iteration
    count within 1 of the oracle's, field within 1e-10 * max|phi|.  The
    oracle's Poisson run is still at a change of 1.1e-4 after its 40,000
    steps (slow diffusive convergence): there both runs stop at max_iters
    and the fields are compared after the same 40,000 steps."""
    z = goldens.load(f"base_c5_cyl64_{kind}_C6_conv")
    g = W.build_cylinder(64, 32, 16, scheme="C6")
    if bool(z["converged"]):
        rep, div = _solve(g, CYL, z, arith="fast", max_iters=int(z["iters"]) + 50)
        assert rep is not None, f"diverged at {div}"
        assert rep.converged
        assert abs(rep.iters - int(z["iters"])) <= 1, (rep.iters, int(z["iters"]))
    else:
        rep, div = _solve(g, CYL, z, arith="fast")
        assert rep is not None, f"diverged at {div}"
        assert not rep.converged and rep.iters == int(z["iters"])
        assert np.allclose(rep.residual_history[-100:], z["residual_history"][-100:], rtol=1e-6)
    ref = z["phi"]
    err = float(np.max(np.abs(rep.phi - ref)))
    assert err <= 1e-10 * float(np.max(np.abs(ref))), err


@pytest.mark.parametrize("kind", ["hj_curvature", "poisson"])
def test_c5_cylinder_64x32x16_c6_converged_exact(kind):
    z = goldens.load(f"base_c5_cyl64_{kind}_C6_conv")
    g = W.build_cylinder(64, 32, 16, scheme="C6")
    rep, div = _solve(g, CYL, z)
    _check_exact(rep, div, z)
    assert np.array_equal(rep.phi, z["phi"])


def test_c5_cylinder_256x128x64_poisson_fast_tracks_exact():
    """Config 5 at a quarter of the resolution per axis, Poisson C6 + F0.48
    (the stable formulation): 400 steps in fast arithmetic -- scan
    derivatives with compile-time line lengths, the compact (i, j)-only
    metric terms (agreeing along z to 1e-12 only), the U-only assemble
    kernel, scan filters -- against exact arithmetic (bit-identical to the
    oracle at 128x64x32 above): history to 1e-9, field to 1e-10 * max."""
    g = W.build_cylinder(256, 128, 64, scheme="C6")
    reps = []
    for arith in ("exact", "fast"):
        cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="poisson"), scheme="C6",
                            filter_config=W.FilterConfig(0.48), tol=1e-15, max_iters=400,
                            arith=arith)
        reps.append(W.solve_steady(g, W.BoundarySpec(CYL), cfg))
    ex, fa = reps
    np.testing.assert_allclose(fa.residual_history, ex.residual_history, rtol=1e-9, atol=1e-14)
    assert np.max(np.abs(fa.phi - ex.phi)) <= 1e-10 * float(np.max(np.abs(ex.phi)))
    assert np.max(np.abs(fa.phi_prime - ex.phi_prime)) <= 1e-10 * float(np.max(np.abs(ex.phi_prime)))


# ------------------------------------------------- kernel variants, A/B
@pytest.mark.parametrize("kind", ["hj_curvature", "poisson", "hj_lad"])
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_two_node_assemble_kernel_is_bit_identical(kind, arith, monkeypatch):
    """k_assemble2 (two nodes per thread, compile-time non-zero-term pattern)
    evaluates k_assemble's expressions: the same solve with WD_NO_ASM2=1 must
    agree bit for bit in either arithmetic (the extruded-grid pattern on the
    cylinder, the full pattern on a sheared grid)."""
    from paper_2111_09859_b200 import _context
    for build in ("cyl", "full"):
        reps = []
        for off in (False, True):
            if off:
                monkeypatch.setenv("WD_NO_ASM2", "1")
            else:
                monkeypatch.delenv("WD_NO_ASM2", raising=False)
            _context.drop_cached()
            g = W.build_cylinder(32, 16, 12, scheme="C6")
            if build == "full":  # shear z with x: every metric term becomes non-zero
                c = np.array(g.coords, copy=True)
                c[2] = c[2] + 0.05 * c[0] + 0.03 * c[1]
                g = W.compute_metrics(W.CurvilinearGrid(coords=c, periodic=g.periodic,
                                                        periods=g.periods), "C6")
            cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=kind), scheme="C6",
                                filter_config=W.FilterConfig(0.48), tol=1e-15, max_iters=4,
                                arith=arith)
            d = np.sqrt(g.coords[0] ** 2 + g.coords[1] ** 2) - 0.5
            reps.append(W.solve_steady(g, W.BoundarySpec(CYL), cfg, phi0=0.5 * d))
        monkeypatch.delenv("WD_NO_ASM2", raising=False)
        a, b = reps
        assert np.array_equal(a.residual_history, b.residual_history), build
        assert np.array_equal(a.phi, b.phi), build
