"""The fused 3-D stage kernels (wd_fused3d.cuh) against the oracle and the
generic kernels, bit-for-bit, across schemes, face kinds, periodicity,
non-multiple-of-tile sizes and i-chunked launches."""
import numpy as np
import pytest

from helpers import same
from oracle import wd

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2111_09859_b200")
from paper_2111_09859_b200 import _context  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")

CASES = [
    # dims, periodic, faces (non-periodic axes), kind, scheme, alpha_f, iters
    ((8, 17, 9), (True, False, True), ("wall", "wall"), "hj", "E6", 0.49, 12),
    ((64, 20, 40), (True, False, True), ("wall", "wall"), "hj", "E6", 0.49, 6),
    ((13, 21, 35), (False, False, False), ("wall",) * 6, "hj", "E4", 0.49, 8),
    ((19, 18, 33), (False, True, False), ("wall", None, "wall", "wall"), "hj", "E2", 0.48, 8),
    ((70, 11, 12), (False, False, True), ("wall", "wall", "wall", None), "eikonal", "E6", 0.49, 6),
    ((12, 40, 37), (True, True, False), (None, "wall"), "hj", "E4", None, 8),
    # many interior tiles (fast mode: cp.async-pipelined k_f3_fast3, scan filter)
    ((40, 64, 96), (True, False, True), ("wall", "wall"), "hj", "E6", 0.49, 6),
    ((30, 56, 64), (True, False, True), ("wall", "wall"), "eikonal", "E6", 0.49, 5),
]


def _faces(periodic, kinds):
    it = iter(kinds)
    faces = {}
    for ax, p in enumerate(periodic):
        for f in FACES[2 * ax:2 * ax + 2]:
            if p:
                faces[f] = "periodic"
            else:
                k = next(it)
                if k is not None:
                    faces[f] = k
    return faces


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"-{c[4]}-{c[3]}")
def test_fused_vs_oracle(case):
    dims, per, kinds, kind, scheme, af, iters = case
    faces = _faces(per, kinds)
    L = [0.9, 1.0, 1.1]
    og = wd.cartesian(*dims, Lx=L[0], Ly=L[1], Lz=L[2], periodic=per)
    pg = W.build_cartesian(*dims, Lx=L[0], Ly=L[1], Lz=L[2], periodic=per)
    rng = np.random.default_rng(sum(dims))
    phi0 = 1e-3 * rng.random(dims)
    bnd_o = wd.Boundary({k: v for k, v in faces.items() if v != "periodic"})
    ro = wd.solve(og, bnd_o, wd.Config(wd.Formulation(kind), scheme, af, 0.5, 1e-15, iters),
                  phi0=phi0, raise_on_divergence=False)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=kind), scheme=scheme,
                        filter_config=None if af is None else W.FilterConfig(af), tol=1e-15,
                        max_iters=iters, arith="exact")
    ctx = _context.NativeSolver(pg, faces, None, scheme, cfg.formulation, cfg.filter_config)
    assert ctx.fused, "fused path expected"
    ctx.close()
    rp = W.solve_steady(pg, W.BoundarySpec(faces), cfg, phi0=phi0)
    assert rp.iters == ro.iters
    assert same(rp.residual_history, ro.residual_history)
    assert same(rp.phi, ro.phi)


def test_fused_matches_generic(monkeypatch):
    dims, per = (40, 33, 48), (True, False, True)
    faces = _faces(per, ("wall", "wall"))
    pg = W.build_cartesian(*dims, periodic=per)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E6",
                        filter_config=W.FilterConfig(0.49), tol=1e-15, max_iters=10,
                        arith="exact")
    a = W.solve_steady(pg, W.BoundarySpec(faces), cfg)
    monkeypatch.setenv("WD_DISABLE_FUSED", "1")
    ctx = _context.NativeSolver(pg, faces, None, "E6", cfg.formulation, cfg.filter_config)
    assert not ctx.fused
    ctx.close()
    b = W.solve_steady(pg, W.BoundarySpec(faces), cfg)
    assert same(a.residual_history, b.residual_history)
    assert same(a.phi, b.phi)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "fast-" + "x".join(map(str, c[0])) + f"-{c[4]}")
def test_fast_mode_close_to_oracle(case):
    """arith='fast' (FMA + composite Laplacian) stays within round-off of
    the exact oracle over the same steps."""
    dims, per, kinds, kind, scheme, af, iters = case
    faces = _faces(per, kinds)
    og = wd.cartesian(*dims, Lx=0.9, Ly=1.0, Lz=1.1, periodic=per)
    pg = W.build_cartesian(*dims, Lx=0.9, Ly=1.0, Lz=1.1, periodic=per)
    rng = np.random.default_rng(sum(dims))
    phi0 = 1e-3 * rng.random(dims)
    bnd_o = wd.Boundary({k: v for k, v in faces.items() if v != "periodic"})
    ro = wd.solve(og, bnd_o, wd.Config(wd.Formulation(kind), scheme, af, 0.5, 1e-15, iters),
                  phi0=phi0, raise_on_divergence=False)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=kind), scheme=scheme,
                        filter_config=None if af is None else W.FilterConfig(af), tol=1e-15,
                        max_iters=iters, arith="fast")
    rp = W.solve_steady(pg, W.BoundarySpec(faces), cfg, phi0=phi0)
    assert rp.iters == ro.iters
    np.testing.assert_allclose(rp.residual_history, ro.residual_history, rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(rp.phi, ro.phi, rtol=0, atol=1e-12 * max(1.0, np.abs(ro.phi).max()))


# ---------------------------------------------------------------- C4 strips
# BASELINE config 4 (walls y = 0, 1; periodic x, z; HJ E6 F0.49) has an
# x/z-invariant solution, so the oracle's 5 x ny x 5 strip
# (tests/golden/make_strip_golden.py) gives its iteration count and profile.
# The same 5 x ny x 5 grid on the GPU must match bit for bit; wider slabs
# differ at round-off only (the periodic filter of a constant line depends on
# the line length), which the fast-mode tolerance test covers.
import goldens  # noqa: E402


def _strip_case(ny, arith, width):
    z = goldens.load(f"strip_c4_ny{ny}")
    n = int(z["n"])
    faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
             "kmin": "periodic", "kmax": "periodic"}
    g = W.build_cartesian(width, ny, width, Lx=width / n, Ly=1.0, Lz=width / n,
                          periodic=(True, False, True))
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj", epsilon=0.2), scheme="E6",
                        filter_config=W.FilterConfig(0.49), cfl=0.5, tol=float(z["tol"]),
                        max_iters=300000, arith=arith)
    rep = W.solve_steady(g, W.BoundarySpec(faces), cfg)
    return z, rep


@pytest.mark.parametrize("ny", [129, 512])
def test_c4_strip_exact_converged(ny):
    z, rep = _strip_case(ny, "exact", 5)
    assert rep.converged and rep.iters == int(z["iters"])
    assert same(rep.residual_history, z["residual_history"])
    assert same(rep.phi, z["phi"])


@pytest.mark.parametrize("ny", [129, 512])
def test_c4_strip_fast_converged(ny):
    """North-star tolerance: converged field within 1e-10 of max wall
    distance, iteration count within 1."""
    z, rep = _strip_case(ny, "fast", 40)
    assert rep.converged and abs(rep.iters - int(z["iters"])) <= 1
    prof = z["profile"]
    err = np.max(np.abs(rep.phi - prof[None, :, None])) / np.max(prof)
    assert err <= 1e-10, err


def test_c1_plate_fast_converges_like_the_reference():
    """BASELINE config 1 in fast arithmetic (2-D: the exact stage kernels,
    the scan filter sweeps): iteration count within 1 of the reference's
    18,440 and the converged field within 1e-10 * max|phi| (north_star)."""
    import goldens
    z = goldens.load("solve_c1_plate_hj_E4")
    g = W.build_cartesian(201, 101, Lx=2.0, Ly=1.0)
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E4",
                        filter_config=W.FilterConfig(0.49), tol=1e-8, max_iters=30000,
                        arith="fast")
    rep = W.solve_steady(g, W.BoundarySpec(faces), cfg)
    assert rep.converged and abs(rep.iters - int(z["iters"])) <= 1, rep.iters
    ref = z["phi"]
    assert np.max(np.abs(rep.phi - ref)) <= 1e-10 * float(np.max(np.abs(ref)))
