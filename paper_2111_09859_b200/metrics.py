"""Validation metrics (drop-in for ``walldist/metrics.py``).

The expensive pieces run on the GPU: the brute-force wall-distance oracle
(O(n m) fp64, bit-identical to the reference's numpy evaluation), the
1/J-weighted L2 error norm (deterministic reduction) and |grad phi|.  The
histogram helpers are host bookkeeping over those results, as in the
reference.  The case registry (``cases.py``) is out of scope, so the
case-id helpers take the exact field directly (``exact_field`` raises).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import _context
from .errors import TooFewIterationsError
from .formulations import FormulationConfig


def _torch():
    import torch
    return torch


def _dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=float))).to("cuda")


def sampled_wall_distance(points, wall_points) -> np.ndarray:
    """Minimum Euclidean distance from each query point (n, d) to a dense wall
    sampling (m, d) (metrics.py:20-34)."""
    torch = _torch()
    host = not isinstance(points, torch.Tensor)
    pts = _dev(np.atleast_2d(np.asarray(points, dtype=float)) if host else points)
    if pts.ndim == 1:
        pts = pts[None, :]
    wall = _dev(wall_points)
    n, d = int(pts.shape[0]), int(pts.shape[1])
    if wall.ndim != 2 or int(wall.shape[1]) != d:
        raise ValueError("wall_points must be (m, d) with the points' d")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    lib = nat.lib()
    torch.cuda.synchronize()
    nat.check(lib.wd_sampled_wall_distance(pts.data_ptr(), n, wall.data_ptr(), int(wall.shape[0]),
                                           d, out.data_ptr(), None))
    torch.cuda.synchronize()
    return out.cpu().numpy() if host else out


def l2_norm(phi, phi_exact, grid) -> float:
    """Area/volume-weighted L2 error, weight 1/J per node (metrics.py:54-66)."""
    import ctypes
    torch = _torch()
    shp = tuple(phi.shape)
    if shp != tuple(phi_exact.shape) or shp != tuple(grid.dims):
        raise ValueError(f"shape mismatch: {shp} vs {tuple(phi_exact.shape)} vs {grid.dims}")
    p, e = _dev(phi), _dev(phi_exact)
    jac = _dev(grid.jacobian)
    out = ctypes.c_double(0.0)
    torch.cuda.synchronize()
    nat.check(nat.lib().wd_l2_norm(p.data_ptr(), e.data_ptr(), jac.data_ptr(), 0.0, p.numel(),
                                   ctypes.byref(out), None))
    return float(out.value)


def exact_distance(case_id: str, point, time: float | None = None) -> float:
    raise NotImplementedError("the case registry (walldist/cases.py) is out of scope")


def exact_field(case_id: str, grid, time: float | None = None):
    raise NotImplementedError("the case registry (walldist/cases.py) is out of scope")


@dataclass
class ErrorHistogram:
    """Percentage-error histogram over the counted (non-wall) nodes."""

    bin_edges: np.ndarray
    counts: np.ndarray
    mean_pct: float
    total: int

    def fraction_within(self, lo_pct: float, hi_pct: float) -> float:
        centers = 0.5 * (self.bin_edges[:-1] + self.bin_edges[1:])
        inside = (centers >= lo_pct) & (centers <= hi_pct)
        return float(np.sum(self.counts[inside]) / self.total)


HIST_BIN_PCT_HJ = 0.5
HIST_BIN_PCT_EIKONAL = 0.05


def percentage_errors(phi, exact, exclude=None) -> np.ndarray:
    """(d_act - d) / d_act * 100 over nodes with d_act > 0 (metrics.py:90-101)."""
    phi = np.asarray(phi, dtype=float)
    exact = np.asarray(exact, dtype=float)
    keep = exact > 0.0
    if exclude is not None:
        keep &= ~np.asarray(exclude, dtype=bool)
    return (exact[keep] - phi[keep]) / exact[keep] * 100.0


def error_histogram_from_exact(phi, exact, bin_width_pct: float = HIST_BIN_PCT_HJ,
                               exclude=None) -> ErrorHistogram:
    """metrics.py:104-118 with the exact field given instead of a case id."""
    errs = percentage_errors(phi, exact, exclude=exclude)
    lo = np.floor(errs.min() / bin_width_pct) * bin_width_pct
    hi = np.ceil(errs.max() / bin_width_pct) * bin_width_pct
    if hi <= lo:
        hi = lo + bin_width_pct
    nbins = int(round((hi - lo) / bin_width_pct))
    counts, edges = np.histogram(errs, bins=nbins, range=(lo, hi))
    return ErrorHistogram(bin_edges=edges, counts=counts, mean_pct=float(np.mean(errs)),
                          total=errs.size)


def gradient_magnitude(phi, grid, scheme: str):
    """|grad phi| (metrics.py:121-124): sqrt(sum_m U_m^2), U from the scheme's
    derivatives and the grid metrics, on the GPU."""
    torch = _torch()
    ctx, cached = _context.acquire(grid, scheme=scheme,
                                   formulation=FormulationConfig(kind="eikonal"))
    try:
        p = ctx.field(phi)
        out = ctx.empty()
        nat.check(ctx.lib.wd_gradient_magnitude(ctx.ptr, p.data_ptr(), out.data_ptr()))
        return out if isinstance(phi, torch.Tensor) else out.cpu().numpy()
    finally:
        _context.release(ctx, cached)


def timing_probe(report) -> float:
    """Seconds per 100 pseudo iterations (metrics.py:127-132)."""
    if report.iters < 100:
        raise TooFewIterationsError(f"timing needs >= 100 iterations, got {report.iters}")
    return report.wall_time_per_100_iters


def summary_record(case: str, formulation: str, scheme: str, grid_dims, report,
                   l2: float | None = None, max_pct_err: float | None = None) -> dict:
    return {"case": case, "formulation": formulation, "scheme": scheme,
            "grid": "x".join(str(n) for n in grid_dims), "iters": report.iters,
            "converged": report.converged, "l2": l2, "max_pct_err": max_pct_err,
            "sec_per_100": report.wall_time_per_100_iters}
