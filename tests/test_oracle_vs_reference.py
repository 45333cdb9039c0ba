"""Pin the CPU oracle (oracle/wd.py) to the reference implementation.

Runs only where /root/reference exists (this container); on the GPU box the
same pins are carried by tests/test_oracle_golden.py and the committed
fixtures.  Comparisons are bit-exact (np.array_equal: equal values, NaN ==
NaN, +0 == -0).
"""
import numpy as np
import pytest

from oracle import wd
from helpers import same

CENTRAL = ["E2", "E4", "C4", "C6"]
ALL = ["UW", "E2", "E4", "C4", "C6"]


def _ogrid(rg):
    return wd.Grid(rg.coords.copy(), rg.metrics.copy(), rg.jacobian.copy(),
                   rg.ref_length, (False,) * rg.ndim, None)


def _bump(ref, ni=41, nj=23, scheme="E4"):
    return ref.grid.build_bump_grid(ni, nj, scheme=scheme)


@pytest.mark.parametrize("scheme", CENTRAL)
@pytest.mark.parametrize("shape,axis", [((37,), 0), ((9, 13), 0), ((9, 13), 1),
                                        ((6, 7, 8), 0), ((6, 7, 8), 1),
                                        ((6, 7, 8), 2)])
def test_central_derivative_bitwise(ref, scheme, shape, axis):
    rng = np.random.default_rng(hash((scheme, shape, axis)) % 2**32)
    f = rng.standard_normal(shape)
    if shape[axis] < wd.MIN_LINE[scheme]:
        pytest.skip("short")
    assert same(wd.deriv(f, scheme, axis), ref.ops.central_derivative(f, scheme, axis))


@pytest.mark.parametrize("scheme", CENTRAL)
@pytest.mark.parametrize("n", [7, 8, 12, 33, 129, 257])
def test_derivative_line_lengths(ref, scheme, n):
    rng = np.random.default_rng(n)
    f = rng.standard_normal((3, n)) * 10.0 ** rng.integers(-3, 3)
    assert same(wd.deriv(f, scheme, 1), ref.ops.central_derivative(f, scheme, 1))


def test_line_too_short(ref):
    for s in CENTRAL:
        with pytest.raises(wd.LineTooShortError):
            wd.deriv(np.zeros(wd.MIN_LINE[s] - 1), s)


@pytest.mark.parametrize("n", [2, 3, 5, 12, 40, 129])
def test_gtsv_transcription_bitwise(ref, n):
    rng = np.random.default_rng(100 + n)
    for trial in range(10):
        lower = rng.uniform(-2, 2, n)
        upper = rng.uniform(-2, 2, n)
        diag = rng.uniform(-2, 2, n) + (4.0 if trial % 2 else 0.0)
        rhs = rng.standard_normal((n, 4))
        try:
            r = ref.ops.solve_tridiagonal(lower, diag, upper, rhs)
        except ref.errors.ZeroPivotError:
            with pytest.raises(wd.ZeroPivotError):
                wd.solve_tridiagonal(lower, diag, upper, rhs)
            continue
        assert same(wd.solve_tridiagonal(lower, diag, upper, rhs), r)


def test_gtsv_pivot_decisions():
    """C6 swaps at steps 1 and n-2; C4 ties at step 1
    (no swap) and swaps at n-2; the filter never swaps."""
    n = 65
    c6 = wd.compact_factor("C6", n)
    assert list(np.nonzero(c6.swap)[0]) == [1, n - 2]
    c4 = wd.compact_factor("C4", n)
    assert list(np.nonzero(c4.swap)[0]) == [n - 2]
    assert not wd.filter_factor(0.49, n).swap.any()


def test_fourth_derivative(ref):
    rng = np.random.default_rng(4)
    f = rng.standard_normal((8, 11, 6))
    for ax in range(3):
        assert same(wd.d4(f, ax), ref.ops.fourth_derivative(f, ax))


@pytest.mark.parametrize("af", [0.40, 0.47, 0.48, 0.49, 0.495, 0.5])
@pytest.mark.parametrize("n", [3, 4, 5, 7, 11, 12, 13, 30, 64, 281])
def test_filter_bitwise(ref, af, n):
    rng = np.random.default_rng(int(af * 1000) + n)
    f = rng.standard_normal((4, n))
    pin = rng.random((4, n)) < 0.1
    cfg = ref.ops.FilterConfig(alpha_f=af)
    assert same(wd.apply_filter(f, 1, af, pinned=pin),
                ref.ops.apply_filter(f, 1, cfg, pinned=pin))
    g = rng.standard_normal((n, 5))
    assert same(wd.apply_filter(g, 0, af), ref.ops.apply_filter(g, 0, cfg))


def test_filter_short(ref):
    for n in (1, 2):
        f = np.arange(float(n))
        assert same(wd.apply_filter(f, 0, 0.49),
                    ref.ops.apply_filter(f, 0, ref.ops.FilterConfig()))


def test_uw_helpers(ref):
    rng = np.random.default_rng(5)
    f = rng.standard_normal((7, 9))
    for ax in range(2):
        B, F = wd.one_sided(f, ax)
        rB, rF = ref.ops.one_sided_differences(f, ax)
        assert same(B, rB) and same(F, rF)
        assert same(wd.front_derivative(B, F), ref.ops.front_derivative_from_bf(rB, rF))
        u = rng.standard_normal(f.shape)
        assert same(wd.upwind_flux(u, B, F), ref.ops.flux_from_bf(u, rB, rF))


@pytest.mark.parametrize("scheme", CENTRAL)
def test_compute_metrics_2d_bitwise(ref, scheme):
    rg = _bump(ref, 45, 21, scheme)
    og = wd.Grid(rg.coords.copy())
    wd.compute_metrics(og, scheme)
    assert same(og.metrics, rg.metrics)
    assert same(og.jacobian, rg.jacobian)
    assert same(og.min_spacing(), rg.min_spacing())
    for l in range(2):
        assert same(og.row_sumsq(l), rg.metric_row_sumsq(l))


def test_compute_metrics_3d_close(ref):
    n = 9
    i, j, k = np.meshgrid(np.arange(n), np.arange(n + 1), np.arange(n + 2),
                          indexing="ij")
    x = 0.1 * i + 0.01 * j * j
    y = 0.12 * j + 0.02 * np.sin(i)
    z = 0.09 * k + 0.01 * i * j
    rg = ref.grid.CurvilinearGrid(coords=np.stack([x, y, z]))
    ref.grid.compute_metrics(rg, "E4")
    og = wd.compute_metrics(wd.Grid(np.stack([x, y, z])), "E4")
    np.testing.assert_allclose(og.metrics, rg.metrics, rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(og.jacobian, rg.jacobian, rtol=1e-13)
    assert same(og.row_sumsq(2), np.sum(og.metrics[2] ** 2, axis=0))


def _fields(rg, seed):
    rng = np.random.default_rng(seed)
    y = rg.coords[1]
    yield np.abs(y - y.min()) + 1e-3 * rng.standard_normal(rg.dims)
    yield rng.random(rg.dims)
    yield np.zeros(rg.dims)


KINDS = ["eikonal", "hj", "hj_lad", "hj_curvature", "poisson"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("scheme", ALL)
def test_residual_and_timestep_bitwise(ref, kind, scheme):
    rg = _bump(ref, 31, 17, "E4")
    og = _ogrid(rg)
    rfc = ref.forms.FormulationConfig(kind=kind, epsilon=0.2, lad_c=0.1)
    ofc = wd.Formulation(kind=kind, epsilon=0.2, lad_c=0.1)
    for phi in _fields(rg, 11):
        assert same(wd.tendency(phi, og, scheme, ofc),
                    ref.forms.tendency(phi, rg, scheme, rfc))
        assert same(wd.local_timestep(phi, og, ofc, 0.5, scheme),
                    ref.solver.local_timestep(phi, rg, rfc, 0.5, scheme))


def test_residual_3d_bitwise(ref):
    rg = ref.grid.build_cartesian(7, 8, 9, Lx=1.0, Ly=1.3, Lz=0.7)
    og = _ogrid(rg)
    rng = np.random.default_rng(3)
    phi = rng.random(rg.dims)
    for kind in KINDS:
        for scheme in ALL:
            rfc = ref.forms.FormulationConfig(kind=kind)
            ofc = wd.Formulation(kind=kind)
            assert same(wd.tendency(phi, og, scheme, ofc),
                        ref.forms.tendency(phi, rg, scheme, rfc)), (kind, scheme)


def test_poisson_post_bitwise(ref):
    rg = ref.grid.build_cartesian(21, 17)
    og = _ogrid(rg)
    y = rg.coords[1]
    pp = 0.5 * y * (1.0 - y)
    pp[3, 4] = -1e-13
    for s in CENTRAL:
        assert same(wd.poisson_post(pp, og, s), ref.forms.poisson_postprocess(pp, rg, s))
    with pytest.raises(wd.NegativeRadicandError):
        wd.poisson_post(np.full(rg.dims, -0.5), og, "E2")


def _faces(rs, kinds):
    return dict(zip(("imin", "imax", "jmin", "jmax", "kmin", "kmax"), kinds))


@pytest.mark.parametrize("kinds", [("farfield", "farfield", "wall", "farfield"),
                                   ("wall", "farfield", "farfield", "wall"),
                                   ("farfield", "wall", "wall", "wall")])
def test_bc_bitwise(ref, kinds):
    rng = np.random.default_rng(8)
    phi = rng.standard_normal((9, 7))
    mask = rng.random((9, 7)) < 0.1
    faces = _faces(None, kinds)
    a = wd.apply_bc(phi.copy(), wd.Boundary(faces, mask))
    b = ref.solver.apply_boundary_conditions(phi.copy(), ref.solver.BoundarySpec(faces, mask))
    assert same(a, b)
    assert same(wd.Boundary(faces, mask).pinned((9, 7)),
                ref.solver.BoundarySpec(faces, mask).pinned_mask((9, 7)))


CASES = [
    # (grid builder, faces, kind, scheme, alpha_f, cfl, iters)
    ("plate", ("farfield", "farfield", "wall", "farfield"), "hj", "E4", 0.49, 0.5, 40),
    ("channel", ("farfield", "farfield", "wall", "wall"), "hj", "C6", 0.48, 0.5, 30),
    ("channel", ("farfield", "farfield", "wall", "wall"), "hj", "C4", 0.49, 0.5, 20),
    ("bump", ("farfield", "farfield", "wall", "farfield"), "hj_curvature", "E4", 0.495, 0.5, 25),
    ("bump", ("farfield", "farfield", "wall", "farfield"), "hj_lad", "E4", 0.49, 0.1, 25),
    ("bump", ("farfield", "farfield", "wall", "farfield"), "eikonal", "E2", 0.49, 0.5, 25),
    ("bump", ("farfield", "farfield", "wall", "farfield"), "poisson", "C6", None, 0.5, 25),
    ("plate", ("farfield", "farfield", "wall", "farfield"), "hj", "UW", None, 0.5, 30),
    ("plate", ("farfield", "farfield", "wall", "farfield"), "eikonal", "UW", None, 0.5, 30),
]


def _case_grid(ref, name):
    if name == "plate":
        return ref.grid.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    if name == "channel":
        return ref.grid.build_cartesian(25, 25)
    return ref.grid.build_bump_grid(41, 21, scheme="E4")


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}-{c[3]}")
def test_short_solve_bitwise(ref, case):
    name, kinds, kind, scheme, af, cfl, iters = case
    rg = _case_grid(ref, name)
    og = _ogrid(rg)
    faces = _faces(None, kinds)
    rcfg = ref.solver.SolveConfig(
        formulation=ref.forms.FormulationConfig(kind=kind), scheme=scheme,
        filter_config=None if af is None else ref.ops.FilterConfig(af),
        cfl=cfl, tol=1e-12, max_iters=iters)
    ocfg = wd.Config(wd.Formulation(kind=kind), scheme, af, cfl, 1e-12, iters)
    rr = ref.solver.solve_steady(rg, ref.solver.BoundarySpec(faces), rcfg)
    orep = wd.solve(og, wd.Boundary(faces), ocfg)
    assert orep.iters == rr.iters
    assert same(orep.residual_history, rr.residual_history)
    assert same(orep.phi, rr.phi)


def test_solid_mask_solve_bitwise(ref):
    rg = ref.grid.build_cartesian(21, 21)
    og = _ogrid(rg)
    mask = np.zeros(rg.dims, bool)
    mask[8:12, 6:10] = True
    faces = _faces(None, ("farfield",) * 4)
    rcfg = ref.solver.SolveConfig(formulation=ref.forms.FormulationConfig(kind="hj"),
                                  scheme="E4", filter_config=ref.ops.FilterConfig(0.49),
                                  tol=1e-12, max_iters=20)
    rr = ref.solver.solve_steady(rg, ref.solver.BoundarySpec(faces, mask), rcfg)
    orep = wd.solve(og, wd.Boundary(faces, mask),
                    wd.Config(wd.Formulation("hj"), "E4", 0.49, 0.5, 1e-12, 20))
    assert same(orep.residual_history, rr.residual_history)
    assert same(orep.phi, rr.phi)


def test_divergence_matches(ref):
    """HJ-E4 without the filter diverges on the flat plate (App. C)."""
    rg = ref.grid.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    og = _ogrid(rg)
    faces = _faces(None, ("farfield", "farfield", "wall", "farfield"))
    rcfg = ref.solver.SolveConfig(formulation=ref.forms.FormulationConfig(kind="hj"),
                                  scheme="E4", tol=1e-12, max_iters=3000)
    it_ref = None
    try:
        ref.solver.solve_steady(rg, ref.solver.BoundarySpec(faces), rcfg)
    except ref.errors.DivergenceError:
        it_ref = "diverged"
    orep = wd.solve(og, wd.Boundary(faces),
                    wd.Config(wd.Formulation("hj"), "E4", None, 0.5, 1e-12, 3000),
                    raise_on_divergence=False)
    if it_ref == "diverged":
        assert orep.diverged_at is not None
    else:
        assert orep.diverged_at is None
