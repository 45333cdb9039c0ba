"""CUDA path vs the reference (golden fixtures) and the oracle, bit-for-bit.

All comparisons use np.array_equal (equal values; +0 == -0).  Everything
here calls the sm_100a kernels through libwd_b200.so.
"""
import numpy as np
import pytest

import goldens
from helpers import same, maxdiff
from oracle import wd

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2111_09859_b200")
from paper_2111_09859_b200 import operators as ops  # noqa: E402
from paper_2111_09859_b200 import formulations as forms  # noqa: E402
from paper_2111_09859_b200 import solver as slv  # noqa: E402
from paper_2111_09859_b200 import grid as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_09859_b200 import _native
    _native.lib()


# ----------------------------------------------------------- operators
def test_derivatives_vs_reference():
    z = goldens.load("operators")
    for s in ("E2", "E4", "C4", "C6"):
        for ax in range(2):
            assert same(ops.central_derivative(z["f2"], s, ax), z[f"d_{s}_2d_{ax}"]), (s, ax)
        for ax in range(3):
            assert same(ops.central_derivative(z["f3"], s, ax), z[f"d_{s}_3d_{ax}"]), (s, ax)
    for ax in range(3):
        assert same(ops.fourth_derivative(z["f3"], ax), z[f"d4_3d_{ax}"])


def test_filter_vs_reference():
    z = goldens.load("operators")
    for af in (0.4, 0.48, 0.49, 0.495, 0.5):
        tag = f"{af:.3f}".replace(".", "p")
        fc = ops.FilterConfig(af)
        for ax in range(2):
            assert same(ops.apply_filter(z["f2"], ax, fc, pinned=z["pin2"]),
                        z[f"filt_{tag}_2d_{ax}"])
        for ax in range(3):
            assert same(ops.apply_filter(z["f3"], ax, fc), z[f"filt_{tag}_3d_{ax}"])
    for n in range(3, 13):
        assert same(ops.apply_filter(z[f"short_in_{n}"], 1, ops.FilterConfig(0.49)),
                    z[f"short_out_{n}"])


@pytest.mark.parametrize("scheme", ["E2", "E4", "E6", "C4", "C6"])
@pytest.mark.parametrize("n", [7, 8, 13, 64, 257])
def test_derivative_vs_oracle_lengths(scheme, n):
    rng = np.random.default_rng(n)
    f = rng.standard_normal((3, n, 4))
    assert same(ops.central_derivative(f, scheme, 1), wd.deriv(f, scheme, 1))


@pytest.mark.parametrize("scheme", ["E2", "E4", "E6", "C4", "C6"])
@pytest.mark.parametrize("n", [5, 9, 32, 129])
def test_periodic_derivative_vs_oracle(scheme, n):
    rng = np.random.default_rng(n + 7)
    f = rng.standard_normal((n, 6))
    assert same(ops.central_derivative(f, scheme, 0, periodic=True),
                wd.deriv(f, scheme, 0, periodic=True))


def test_periodic_filter_and_d4_vs_oracle():
    rng = np.random.default_rng(3)
    for n in (5, 11, 12, 64):
        f = rng.standard_normal((4, n))
        pin = rng.random((4, n)) < 0.1
        for af in (0.4, 0.49, 0.495):
            assert same(ops.apply_filter(f, 1, ops.FilterConfig(af), pinned=pin, periodic=True),
                        wd.apply_filter(f, 1, af, pinned=pin, periodic=True))
        assert same(ops.fourth_derivative(f, 1, periodic=True), wd.d4(f, 1, periodic=True))


def test_line_too_short_and_bad_scheme():
    from paper_2111_09859_b200.errors import LineTooShortError
    for s, k in (("E2", 3), ("E4", 5), ("C4", 7), ("C6", 7), ("E6", 7)):
        with pytest.raises(LineTooShortError):
            ops.central_derivative(np.zeros(k - 1), s)
    with pytest.raises(ValueError):
        ops.central_derivative(np.zeros(9), "UW")
    with pytest.raises(LineTooShortError):
        ops.fourth_derivative(np.zeros(4))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 12, 40])
def test_tridiagonal_vs_oracle(n):
    from paper_2111_09859_b200.errors import ZeroPivotError
    rng = np.random.default_rng(100 + n)
    for trial in range(6):
        lower = rng.uniform(-2, 2, n)
        upper = rng.uniform(-2, 2, n)
        diag = rng.uniform(-2, 2, n) + (4.0 if trial % 2 else 0.0)
        rhs = rng.standard_normal((n, 5))
        try:
            r = wd.solve_tridiagonal(lower, diag, upper, rhs)
        except wd.ZeroPivotError:
            with pytest.raises(ZeroPivotError):
                ops.solve_tridiagonal(lower, diag, upper, rhs)
            continue
        assert same(ops.solve_tridiagonal(lower, diag, upper, rhs), r)
    with pytest.raises(ZeroPivotError):
        ops.solve_tridiagonal(np.zeros(1), np.zeros(1), np.zeros(1), np.ones(1))


# ------------------------------------------------------------- metrics
def test_compute_metrics_vs_reference():
    z = goldens.load("residuals")
    for s in ("E2", "E4", "C4", "C6"):
        g = G.CurvilinearGrid(coords=z["coords"].copy())
        G.compute_metrics(g, s)
        assert same(g.metrics, z[f"metrics_{s}"]), s


def test_compute_metrics_3d_and_periodic_vs_oracle():
    og = wd.cylinder(12, 9, 10, scheme="C6")
    pg = G.build_cylinder(12, 9, 10, scheme="C6")
    assert same(pg.metrics, og.metrics)
    assert same(pg.jacobian, og.jacobian)
    oa = wd.annulus(17, 9, scheme="E6")
    pa = G.build_annulus(17, 9, scheme="E6")
    assert same(pa.metrics, oa.metrics)
    ob = wd.sinusoidal_bump(33, 17, scheme="E6")
    pb = G.build_sinusoidal_bump(33, 17, scheme="E6")
    assert same(pb.metrics, ob.metrics)
    assert np.all(pa.jacobian > 0) and np.all(pg.jacobian > 0)


def test_singular_metric():
    from paper_2111_09859_b200.errors import SingularMetricError
    x = np.zeros((9, 9))
    y = np.repeat(np.linspace(0, 1, 9)[None, :], 9, axis=0)
    with pytest.raises(SingularMetricError):
        G.compute_metrics(G.CurvilinearGrid(coords=np.stack([x, y])), "E2")


# ----------------------------------------------------------- residuals
KINDS = ("eikonal", "hj", "hj_lad", "hj_curvature", "poisson")
SCHEMES = ("UW", "E2", "E4", "C4", "C6")


def test_tendency_and_timestep_vs_reference():
    z = goldens.load("residuals")
    g = G.CurvilinearGrid(z["coords"], z["metrics"], z["jacobian"])
    for kind in KINDS:
        fc = forms.FormulationConfig(kind=kind)
        for s in SCHEMES:
            k = forms.tendency(z["phi"], g, s, fc)
            assert same(k, z[f"k_{kind}_{s}"]), (kind, s, maxdiff(k, z[f"k_{kind}_{s}"]))
            dt = slv.local_timestep(z["phi"], g, fc, 0.5, s)
            assert same(dt, z[f"dt_{kind}_{s}"]), (kind, s)
    for s in ("E2", "E4", "C4", "C6"):
        assert same(forms.poisson_postprocess(z["pp"], g, s), z[f"post_{s}"]), s


def test_uniform_path_matches_metric_path():
    """The analytic-Cartesian path equals the (d,d,N)-metrics path."""
    gu = G.build_cartesian(23, 19, Lx=2.0, Ly=1.0)
    gm = G.CurvilinearGrid(gu.coords.copy(), gu.metrics.copy(), gu.jacobian.copy())
    rng = np.random.default_rng(1)
    phi = rng.random(gu.dims)
    for kind in KINDS:
        for s in SCHEMES + ("E6",):
            fc = forms.FormulationConfig(kind=kind)
            assert same(forms.tendency(phi, gu, s, fc), forms.tendency(phi, gm, s, fc)), (kind, s)


def test_negative_radicand():
    from paper_2111_09859_b200.errors import NegativeRadicandError
    g = G.build_cartesian(21, 21)
    with pytest.raises(NegativeRadicandError):
        forms.poisson_postprocess(np.full(g.dims, -0.5), g, "E2")


def test_apply_bc_vs_oracle():
    rng = np.random.default_rng(8)
    for kinds in (("farfield", "farfield", "wall", "farfield"),
                  ("wall", "farfield", "farfield", "wall"),
                  ("farfield", "wall", "wall", "wall")):
        faces = dict(zip(goldens.FACES, kinds))
        phi = rng.standard_normal((9, 7))
        mask = rng.random((9, 7)) < 0.1
        a = slv.apply_boundary_conditions(phi.copy(), slv.BoundarySpec(faces, mask))
        b = wd.apply_bc(phi.copy(), wd.Boundary(faces, mask))
        assert same(a, b)


# -------------------------------------------------------------- solves
def _product_case(z, uniform_from=None):
    g = G.CurvilinearGrid(z["coords"], z["metrics"], z["jacobian"])
    faces = goldens.case_faces(z)
    af = goldens.case_alpha(z)
    cfg = slv.SolveConfig(formulation=forms.FormulationConfig(kind=str(z["kind"])),
                          scheme=str(z["scheme"]),
                          filter_config=None if af is None else ops.FilterConfig(af),
                          cfl=float(z["cfl"]), tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                          arith="exact")
    return g, slv.BoundarySpec(faces, z.get("solid_mask")), cfg


@pytest.mark.parametrize("case", goldens.solve_cases())
def test_solve_vs_reference(case):
    z = goldens.load("solve_" + case)
    g, bnd, cfg = _product_case(z)
    from paper_2111_09859_b200.errors import DivergenceError
    if int(z["diverged"]) > 0:
        with pytest.raises(DivergenceError, match=f"iteration {int(z['diverged'])}"):
            slv.solve_steady(g, bnd, cfg)
        return
    rep = slv.solve_steady(g, bnd, cfg)
    assert rep.iters == int(z["iters"])
    assert rep.converged == bool(z["converged"])
    assert same(rep.residual_history, z["residual_history"])
    assert same(rep.phi, z["phi"])
    if "phi_prime" in z:
        assert same(rep.phi_prime, z["phi_prime"])
    assert rep.wall_seconds.shape == (rep.iters,)


def test_solve_uniform_cartesian_c1_prefix():
    """C1 through the analytic-Cartesian path (build_cartesian)."""
    z = goldens.load("solve_c1_plate_hj_E4")
    g = G.build_cartesian(201, 101, Lx=2.0, Ly=1.0)
    cfg = slv.SolveConfig(formulation=forms.FormulationConfig(kind="hj"), scheme="E4",
                          filter_config=ops.FilterConfig(0.49), tol=1e-8, max_iters=50000,
                          arith="exact")
    rep = slv.solve_steady(g, slv.BoundarySpec(goldens.case_faces(z)), cfg)
    assert rep.iters == int(z["iters"]) == 18440
    assert same(rep.residual_history, z["residual_history"])
    assert same(rep.phi, z["phi"])
    # HJ (eps = 0.2) is accurate near the wall (sec. 5.1)
    near = g.y <= 0.3
    assert maxdiff(rep.phi[near], g.y[near]) < 1e-2


def test_divergence_plate():
    z = goldens.load("diverge_plate_E4")
    from paper_2111_09859_b200.errors import DivergenceError
    g = G.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    cfg = slv.SolveConfig(formulation=forms.FormulationConfig(kind="hj"), scheme="E4",
                          tol=1e-12, max_iters=5000, arith="exact")
    faces = dict(zip(goldens.FACES, ("farfield", "farfield", "wall", "farfield")))
    with pytest.raises(DivergenceError, match=f"iteration {int(z['diverged_at'])}"):
        slv.solve_steady(g, slv.BoundarySpec(faces), cfg)


# --------------------------------------------------- extension solves
def _ext_solve(og, pg, faces, kind, scheme, af, iters, cfl=0.5):
    cfg_o = wd.Config(wd.Formulation(kind=kind), scheme, af, cfl, 1e-14, iters)
    ro = wd.solve(og, wd.Boundary(faces), cfg_o)
    cfg_p = slv.SolveConfig(formulation=forms.FormulationConfig(kind=kind), scheme=scheme,
                            filter_config=None if af is None else ops.FilterConfig(af),
                            cfl=cfl, tol=1e-14, max_iters=iters, arith="exact")
    rp = slv.solve_steady(pg, slv.BoundarySpec(faces), cfg_p)
    return ro, rp


def test_periodic_channel3d_e6_vs_oracle():
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    og = wd.cartesian(8, 17, 9, Lx=8 / 32, Ly=1.0, Lz=9 / 32, periodic=(True, False, True))
    pg = G.build_cartesian(8, 17, 9, Lx=8 / 32, Ly=1.0, Lz=9 / 32, periodic=(True, False, True))
    ro, rp = _ext_solve(og, pg, faces, "hj", "E6", 0.49, 25)
    assert same(rp.residual_history, ro.residual_history)
    assert same(rp.phi, ro.phi)


def test_annulus_curvature_c6_vs_oracle():
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
    og = wd.annulus(33, 17, scheme="C6")
    pg = G.build_annulus(33, 17, scheme="C6")
    ro, rp = _ext_solve(og, pg, faces, "hj_curvature", "C6", 0.48, 40)
    assert same(rp.residual_history, ro.residual_history)
    assert same(rp.phi, ro.phi)


def test_annulus_divergence_iteration_matches_oracle():
    """Too coarse an annulus diverges; the iteration must match the oracle."""
    from paper_2111_09859_b200.errors import DivergenceError
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
    og = wd.annulus(24, 13, scheme="C6")
    ro = wd.solve(og, wd.Boundary(faces), wd.Config(wd.Formulation("hj_curvature"), "C6", 0.48,
                                                   0.5, 1e-14, 40), raise_on_divergence=False)
    assert ro.diverged_at == 10
    pg = G.build_annulus(24, 13, scheme="C6")
    cfg = slv.SolveConfig(formulation=forms.FormulationConfig(kind="hj_curvature"), scheme="C6",
                          filter_config=ops.FilterConfig(0.48), tol=1e-14, max_iters=40)
    with pytest.raises(DivergenceError, match="iteration 10"):
        slv.solve_steady(pg, slv.BoundarySpec(faces), cfg)


def test_cylinder_poisson_c6_vs_oracle():
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
             "kmin": "periodic", "kmax": "periodic"}
    og = wd.cylinder(12, 9, 6, scheme="C6")
    pg = G.build_cylinder(12, 9, 6, scheme="C6")
    ro, rp = _ext_solve(og, pg, faces, "poisson", "C6", None, 10)
    assert same(rp.residual_history, ro.residual_history)
    assert same(rp.phi_prime, ro.phi_prime)
    assert same(rp.phi, ro.phi)
