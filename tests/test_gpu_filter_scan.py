"""Fast-arithmetic filter sweep (csrc/wd_filter_scan.cuh: segmented affine
scan of the dgtsv factor) against the oracle's apply_filter
(operators.py:305-352; cyclic extension), one sweep at a time through the
C ABI (wd_fused_filter on an arbitrary (n0, n1, n2) array), plus the fused
convergence reduction it carries on the last axis.

Tolerance: the scan solves the same linear system in a different operation
order, so results agree to round-off: |x - x_oracle| <= 1e-13 * max|u|."""
import ctypes

import numpy as np
import pytest

from oracle import wd

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2111_09859_b200")
from paper_2111_09859_b200 import _context, _native as nat  # noqa: E402

FACES = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
         "kmin": "periodic", "kmax": "periodic"}
AF = 0.49


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


def _ctx(torch, arith="fast"):
    g = W.build_cartesian(16, 16, 16, periodic=(True, False, True))
    ctx = _context.NativeSolver(g, FACES, None, "E6", W.FormulationConfig(kind="hj"),
                                W.FilterConfig(AF), 0.5, 1e-15, 10, arith=arith)
    assert ctx.fused
    phi = torch.zeros((16, 16, 16), dtype=torch.float64, device="cuda")
    hist = torch.zeros(16, dtype=torch.float64, device="cuda")
    nat.check(ctx.lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
    ctx._bound = (phi, hist)
    return ctx


def _sweep(torch, ctx, u, axis, periodic, A=None):
    dev = torch.from_numpy(u).cuda()
    out = torch.empty_like(dev)
    a_dev = torch.from_numpy(A).cuda() if A is not None else None
    nat.check(ctx.lib.wd_fused_filter(ctx.ptr, axis, dev.data_ptr(), out.data_ptr(), *u.shape,
                                     int(periodic), a_dev.data_ptr() if a_dev is not None else None))
    torch.cuda.synchronize()
    return out.cpu().numpy()


CASES = [
    # shape, axis, periodic -- n = 512 exercises the full-segment kernel
    ((512, 3, 20), 0, True),
    ((512, 3, 20), 0, False),
    ((3, 512, 24), 1, False),
    ((3, 512, 17), 1, True),
    ((5, 18, 512), 2, True),
    ((5, 18, 512), 2, False),
    # n = 256: the 16-row full-segment instantiation
    ((256, 3, 20), 0, True),
    ((3, 256, 24), 1, False),
    ((5, 18, 256), 2, True),
    ((5, 18, 256), 2, False),
    ((100, 3, 17), 0, False),
    ((3, 7, 37), 2, True),
    ((2, 45, 33), 1, False),
    ((4, 5, 12), 2, False),
]


@pytest.mark.parametrize("shape,axis,periodic", CASES,
                         ids=lambda c: "x".join(map(str, c)) if isinstance(c, tuple) else str(c))
def test_scan_filter_vs_oracle(torch, shape, axis, periodic):
    rng = np.random.default_rng(sum(shape) + axis)
    u = rng.standard_normal(shape)
    ctx = _ctx(torch)
    try:
        got = _sweep(torch, ctx, u, axis, periodic)
    finally:
        ctx.close()
    ref = wd.apply_filter(u, axis, AF, periodic=periodic)
    err = np.max(np.abs(got - ref))
    assert err <= 1e-13 * np.max(np.abs(u)), err


def test_scan_filter_smooth_field(torch):
    """A smooth periodic mode passes almost unchanged (filter transfer ~1)."""
    n = 512
    x = np.arange(n) / n
    u = np.broadcast_to(np.sin(2 * np.pi * 3 * x)[None, None, :], (4, 16, n)).copy()
    ctx = _ctx(torch)
    try:
        got = _sweep(torch, ctx, u, 2, True)
    finally:
        ctx.close()
    ref = wd.apply_filter(u, 2, AF, periodic=True)
    assert np.max(np.abs(got - ref)) <= 1e-14
    assert np.max(np.abs(got - u)) < 1e-6


def test_scan_filter_reduction(torch):
    """Last-axis sweep also reduces max|x - A|, max|x| into the status word
    (read through wd_status_maxima)."""
    shape = (6, 20, 512)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(shape)
    A = rng.standard_normal(shape)
    ctx = _ctx(torch)
    try:
        got = _sweep(torch, ctx, u, 2, True, A=A)
        stats = torch.zeros(3, dtype=torch.int64, device="cuda")
        nat.check(ctx.lib.wd_status_maxima(ctx.ptr, stats.data_ptr()))
        s = stats.cpu().numpy()
    finally:
        ctx.close()
    md = np.int64(s[0]).view(np.float64)
    ma = np.int64(s[1]).view(np.float64)
    assert md == np.max(np.abs(got - A))
    assert ma == np.max(np.abs(got))
    assert s[2] == 0


def test_exact_ctx_keeps_dgtsv_sweep(torch):
    """arith='exact' never uses the scan: bit-identical to the oracle."""
    shape = (3, 512, 24)
    u = np.random.default_rng(1).standard_normal(shape)
    ctx = _ctx(torch, arith="exact")
    try:
        got = _sweep(torch, ctx, u, 1, False)
    finally:
        ctx.close()
    assert np.array_equal(got, wd.apply_filter(u, 1, AF, periodic=False))
