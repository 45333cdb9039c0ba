"""Fast-arithmetic compact derivatives on the generic path
(csrc/wd_deriv_scan.cuh: segmented-scan solve of the no-pivoting C4/C6
factor with the derivative epilogue fused).  arith='fast' differs from the
reference's dgtsv solve in the last bits only, so every comparison here is
against the oracle (exact restatement of the reference) within round-off
tolerances; arith='exact' never takes this path (test_gpu_parity.py stays
bit-for-bit).  Lines of up to 512 nodes run 16-line tiles, up to 1024
nodes 8-line tiles; longer axes fall back to the exact line solve inside
the same run (covered by the 1100-node case)."""
import numpy as np
import pytest

from oracle import wd

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2111_09859_b200")
from paper_2111_09859_b200 import grid as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_09859_b200 import _native
    _native.lib()


def _pair(og, pg, faces, kind, scheme, af, iters, phi0=None, tol=1e-15, arith="fast"):
    bnd_o = wd.Boundary({k: v for k, v in faces.items() if v != "periodic"})
    ro = wd.solve(og, bnd_o, wd.Config(wd.Formulation(kind), scheme, af, 0.5, tol, iters),
                  phi0=phi0, raise_on_divergence=False)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=kind), scheme=scheme,
                        filter_config=None if af is None else W.FilterConfig(af), tol=tol,
                        max_iters=iters, arith=arith)
    rp = W.solve_steady(pg, W.BoundarySpec(faces), cfg, phi0=phi0)
    return ro, rp


def _close(ro, rp, atol_rel=1e-11, hist_rtol=1e-8):
    assert rp.iters == ro.iters
    np.testing.assert_allclose(rp.residual_history, ro.residual_history, rtol=hist_rtol,
                               atol=1e-14)
    scale = max(1.0, float(np.abs(ro.phi).max()))
    np.testing.assert_allclose(rp.phi, ro.phi, rtol=0, atol=atol_rel * scale)


CYL_FACES = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
             "kmin": "periodic", "kmax": "periodic"}


def _cyl_exact(og):
    x, y = og.coords[0], og.coords[1]
    return np.sqrt(x * x + y * y) - 0.5


def test_cylinder_curvature_c6_fast_vs_oracle():
    """BASELINE config 5's formulation (HJ + curvature, C6, F0.48) on a
    small cylinder: theta (periodic, cyclic scan), r (closures, Thomas
    factor), z (periodic, stride-1 tiles); metric epilogues (acc + M D)."""
    og = wd.cylinder(24, 16, 12, scheme="C6")
    pg = G.build_cylinder(24, 16, 12, scheme="C6")
    phi0 = _cyl_exact(og)
    ro, rp = _pair(og, pg, CYL_FACES, "hj_curvature", "C6", 0.48, 12, phi0=phi0)
    _close(ro, rp)


def test_cylinder_poisson_c6_fast_vs_oracle():
    og = wd.cylinder(16, 20, 12, scheme="C6")
    pg = G.build_cylinder(16, 20, 12, scheme="C6")
    ro, rp = _pair(og, pg, CYL_FACES, "poisson", "C6", None, 10)
    _close(ro, rp)
    np.testing.assert_allclose(rp.phi_prime, ro.phi_prime, rtol=0,
                               atol=1e-11 * max(1.0, np.abs(ro.phi_prime).max()))


@pytest.mark.parametrize("scheme", ["C4", "C6"])
def test_annulus_hj_fast_vs_oracle(scheme):
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
    og = wd.annulus(33, 17, scheme=scheme)
    pg = G.build_annulus(33, 17, scheme=scheme)
    x, y = og.coords[0], og.coords[1]
    phi0 = np.sqrt(x * x + y * y) - 0.5
    ro, rp = _pair(og, pg, faces, "hj", scheme, 0.48, 30, phi0=phi0)
    _close(ro, rp)


def test_channel3d_uniform_c6_fast_vs_oracle():
    """Uniform Cartesian (scalar metric epilogue), every axis on the scan,
    tiles with partial line groups (13 and 20 lines per plane)."""
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    dims = (14, 20, 13)
    og = wd.cartesian(*dims, Lx=14 / 40, Ly=1.0, Lz=13 / 40, periodic=(True, False, True))
    pg = G.build_cartesian(*dims, Lx=14 / 40, Ly=1.0, Lz=13 / 40, periodic=(True, False, True))
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.48, 25)
    _close(ro, rp)


def test_600_node_axis_eight_line_tiles():
    """n = 600 > 512 on axis 0: 8-line tiles, 32 segments of 19 rows."""
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    og = wd.cartesian(600, 16, Lx=4.0, Ly=1.0)
    pg = G.build_cartesian(600, 16, Lx=4.0, Ly=1.0)
    ro, rp = _pair(og, pg, faces, "hj", "C4", 0.49, 15)
    _close(ro, rp)


def test_bump_c6_curvilinear_fast_vs_oracle():
    """Non-periodic curvilinear axes (closures at both ends of both axes;
    the bump's M[0,1] is identically zero, so its divergence term is
    skipped)."""
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    og = wd.sinusoidal_bump(65, 33, scheme="C6")
    pg = G.build_sinusoidal_bump(65, 33, scheme="C6")
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.49, 20)
    _close(ro, rp)


def test_channel_c6_converges_like_oracle():
    """North-star tolerance: converged field within 1e-10 of max wall
    distance and the iteration count to the same residual within 1."""
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall"}
    og = wd.cartesian(16, 41, Lx=16 / 40, Ly=1.0, periodic=(True, False))
    pg = G.build_cartesian(16, 41, Lx=16 / 40, Ly=1.0, periodic=(True, False))
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.48, 20000, tol=1e-8)
    assert ro.converged and rp.converged
    assert abs(rp.iters - ro.iters) <= 1
    assert np.abs(rp.phi - ro.phi).max() <= 1e-10 * np.abs(ro.phi).max()


# full-segment instantiations (n = 256 -> 16 rows, n = 512 -> 32 rows per
# segment, compile-time row loops), strided and stride-1, both schemes
def test_annulus_256_full_segments():
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield"}
    og = wd.annulus(256, 24, scheme="C6")
    pg = G.build_annulus(256, 24, scheme="C6")
    x, y = og.coords[0], og.coords[1]
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.48, 8, phi0=np.sqrt(x * x + y * y) - 0.5)
    _close(ro, rp)


def test_plate_512_contiguous_c4():
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    og = wd.cartesian(20, 512, Lx=0.5, Ly=1.0)
    pg = G.build_cartesian(20, 512, Lx=0.5, Ly=1.0)
    ro, rp = _pair(og, pg, faces, "hj", "C4", 0.49, 8)
    _close(ro, rp)


def test_channel3d_256_contiguous_periodic():
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    dims = (16, 24, 256)
    og = wd.cartesian(*dims, Lx=16 / 24, Ly=1.0, Lz=256 / 24, periodic=(True, False, True))
    pg = G.build_cartesian(*dims, Lx=16 / 24, Ly=1.0, Lz=256 / 24, periodic=(True, False, True))
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.48, 6)
    _close(ro, rp)


def test_block3d_512_strided_closures():
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield",
             "kmin": "farfield", "kmax": "farfield"}
    dims = (512, 12, 16)
    og = wd.cartesian(*dims, Lx=4.0, Ly=1.0, Lz=1.0)
    pg = G.build_cartesian(*dims, Lx=4.0, Ly=1.0, Lz=1.0)
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.49, 4)
    _close(ro, rp)


def test_long_axis_falls_back_to_exact_solve():
    """n = 1100 > 1024 on axis 0 runs the exact line solve, axis 1 the scan."""
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    og = wd.cartesian(1100, 12, Lx=4.0, Ly=1.0)
    pg = G.build_cartesian(1100, 12, Lx=4.0, Ly=1.0)
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.49, 6)
    _close(ro, rp)


def test_ring_1024_periodic_strided():
    """C5's theta axis: n = 1024, periodic, strided (8-line tiles, 32 rows)."""
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "farfield",
             "kmin": "periodic", "kmax": "periodic"}
    og = wd.cylinder(1024, 12, 12, scheme="C6")
    pg = G.build_cylinder(1024, 12, 12, scheme="C6")
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.48, 4, phi0=_cyl_exact(og))
    _close(ro, rp)


def test_plate_1024_contiguous_closures():
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    og = wd.cartesian(12, 1024, Lx=0.1, Ly=1.0)
    pg = G.build_cartesian(12, 1024, Lx=0.1, Ly=1.0)
    ro, rp = _pair(og, pg, faces, "hj", "C6", 0.49, 6)
    _close(ro, rp)


def test_fused_fast_256_last_axis_filter_reduction():
    """Fused 3-D fast path with a 256-node last axis: the scan filter's
    16-row full-segment instantiation with the convergence reduction."""
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    dims = (12, 40, 256)
    og = wd.cartesian(*dims, Lx=12 / 40, Ly=1.0, Lz=256 / 40, periodic=(True, False, True))
    pg = G.build_cartesian(*dims, Lx=12 / 40, Ly=1.0, Lz=256 / 40, periodic=(True, False, True))
    ro, rp = _pair(og, pg, faces, "hj", "E6", 0.49, 6)
    _close(ro, rp)
