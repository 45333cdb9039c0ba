"""Pseudo-time steady solver (drop-in for ``walldist/solver.py:1-293``).

``solve_steady`` keeps the reference signature and SolveReport, and runs the
whole pseudo-time loop on the GPU: local time step, 4 RK stages with fused
boundary conditions, the implicit filter, the convergence/divergence
reduction and the stop test all execute as sm_100a kernels replayed from a
CUDA graph in chunks of k steps.  A device status word freezes the state
at the reference's stopping iteration, so the host polls once per chunk
instead of once per step.  Results (iteration count, residual history,
field) are bit-identical to the reference's on its own paths.
"""
from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import _context
from ._context import FACE_NAMES, NativeSolver
from .errors import DivergenceError
from .formulations import FormulationConfig
from .operators import FilterConfig

_FACE_NAMES = FACE_NAMES
WALL = "wall"
FARFIELD = "farfield"
PERIODIC = "periodic"  # EXTENSION


@dataclass
class BoundarySpec:
    """Per-face boundary kinds plus an optional solid mask (solver.py:32-70).
    EXTENSION: kind "periodic" (on both faces of a periodic grid axis)."""

    faces: dict
    solid_mask: np.ndarray | None = None

    def __post_init__(self):
        for name, kind in self.faces.items():
            if name not in _FACE_NAMES:
                raise ValueError(f"unknown face {name!r}")
            if kind not in (WALL, FARFIELD, PERIODIC):
                raise ValueError(f"unknown boundary kind {kind!r}")

    def ndim(self) -> int:
        return len(self.faces) // 2

    def has_wall(self) -> bool:
        if any(kind == WALL for kind in self.faces.values()):
            return True
        return self.solid_mask is not None and bool(np.any(np.asarray(self.solid_mask)))

    def pinned_mask(self, dims) -> np.ndarray:
        pinned = np.zeros(dims, dtype=bool)
        nd = len(dims)
        for axis in range(nd):
            idx = [slice(None)] * nd
            if self.faces.get(_FACE_NAMES[2 * axis]) == WALL:
                idx[axis] = 0
                pinned[tuple(idx)] = True
            if self.faces.get(_FACE_NAMES[2 * axis + 1]) == WALL:
                idx[axis] = -1
                pinned[tuple(idx)] = True
        if self.solid_mask is not None:
            pinned |= np.asarray(self.solid_mask, dtype=bool)
        return pinned


def all_wall_faces(ndim: int) -> dict:
    return {name: WALL for name in _FACE_NAMES[:2 * ndim]}


@dataclass
class SolveConfig:
    """Everything a steady solve needs besides grid and boundary
    (solver.py:113-133)."""

    formulation: FormulationConfig = field(default_factory=FormulationConfig)
    scheme: str = "UW"
    filter_config: FilterConfig | None = None
    cfl: float = 0.5
    tol: float = 1e-5
    max_iters: int = 50000
    l2_every: int = 0
    # EXTENSION: "exact" reproduces the reference bit for
    # bit; "fast" lets the kernels reassociate (FMA, composite stencils,
    # scan-form line solves: round-off-level differences, the converged field
    # within 1e-10 and the iteration count within 1 of the reference's --
    # BASELINE's tolerance); "auto" (default) = "fast" for the formulations
    # whose iteration is stable under round-off perturbations (hj, poisson;
    # SURVEY sec. 8c) and "exact" for the chaotic ones (hj_lad, hj_curvature,
    # eikonal), whose parity is only defined bit for bit.
    arith: str = "auto"

    def __post_init__(self):
        if self.cfl <= 0.0:
            raise ValueError("cfl must be positive")
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.arith not in ("auto", "exact", "fast"):
            raise ValueError("arith must be 'auto', 'exact' or 'fast'")

    def uses_filter(self) -> bool:
        return self.filter_config is not None and self.scheme != "UW"

    def resolved_arith(self) -> str:
        if self.arith != "auto":
            return self.arith
        return "fast" if self.formulation.kind in ("hj", "poisson") else "exact"


@dataclass
class SolveReport:
    """Converged field plus convergence/timing histories (solver.py:135-154)."""

    phi: np.ndarray
    iters: int
    residual_history: np.ndarray
    wall_seconds: np.ndarray
    converged: bool
    l2_history: np.ndarray | None = None
    phi_prime: np.ndarray | None = None
    time: float | None = None

    @property
    def loop_seconds(self) -> float:
        return float(self.wall_seconds[-1]) if self.iters else 0.0

    @property
    def wall_time_per_100_iters(self) -> float:
        return 100.0 * self.loop_seconds / max(self.iters, 1)


class _GridShim:
    """Minimal uniform grid for grid-free calls (apply_boundary_conditions)."""

    def __init__(self, dims, periodic):
        self.dims = tuple(dims)
        self.ndim = len(dims)
        self.periodic = periodic
        self.is_uniform = True
        self.inv_spacing = (1.0,) * self.ndim
        self.ref_length = 1.0


def apply_boundary_conditions(phi, boundary: BoundarySpec):
    """Far-field copies, then walls, then the solid mask, in place
    (solver.py:87-110)."""
    import torch
    is_t = isinstance(phi, torch.Tensor)
    dims = tuple(phi.shape)
    per = tuple(boundary.faces.get(_FACE_NAMES[2 * a]) == PERIODIC for a in range(len(dims)))
    ctx, cached = _context.acquire(_GridShim(dims, per), boundary.faces, boundary.solid_mask,
                                   "E2", FormulationConfig(kind="eikonal"),
                                   key_extra=("shim", dims, per))
    try:
        t = ctx.field(phi) if not is_t else phi
        if is_t and (t.dtype != torch.float64 or not t.is_contiguous() or not t.is_cuda):
            raise ValueError("in-place BCs need a contiguous fp64 CUDA tensor")
        nat.check(ctx.lib.wd_apply_bc(ctx.ptr, t.data_ptr()))
        if not is_t:
            phi[...] = t.cpu().numpy()
        return phi
    finally:
        _context.release(ctx, cached)


def local_timestep(phi, grid, config: FormulationConfig, cfl: float, scheme: str = "E2"):
    """Per-node pseudo time step (solver.py:160-180)."""
    ctx, cached = _context.acquire(grid, scheme=scheme, formulation=config, cfl=cfl)
    try:
        p = ctx.field(phi)
        dt = ctx.empty()
        nat.check(ctx.lib.wd_local_timestep(ctx.ptr, p.data_ptr(), dt.data_ptr()))
        import torch
        return dt if isinstance(phi, torch.Tensor) else dt.cpu().numpy()
    finally:
        _context.release(ctx, cached)


def rk4_step(phi, grid, config: SolveConfig, dt_field, boundary: BoundarySpec):
    """One classical RK4 step + filter + BCs + divergence check
    (solver.py:183-218)."""
    ctx, cached = _context.acquire(grid, boundary.faces, boundary.solid_mask, config.scheme,
                                   config.formulation, config.filter_config, config.cfl,
                                   config.tol)
    try:
        p = ctx.field(phi)
        dt = ctx.field(dt_field)
        out = ctx.empty()
        div = ctypes.c_int(0)
        nat.check(ctx.lib.wd_rk4_step(ctx.ptr, p.data_ptr(), dt.data_ptr(), out.data_ptr(),
                                      ctypes.byref(div)))
        if div.value:
            limit = 1e6 * grid.ref_length
            raise DivergenceError(f"pseudo-time iteration diverged (max |phi| > {limit:g})")
        import torch
        return out if isinstance(phi, torch.Tensor) else out.cpu().numpy()
    finally:
        _context.release(ctx, cached)


def _chunk_sizes(n_nodes: int):
    """Steps per graph replay: small grids are launch-bound (long chunks),
    large grids are bandwidth-bound (short chunks waste little on freeze)."""
    if n_nodes >= 8_000_000:
        return 2, 8
    if n_nodes >= 500_000:
        return 4, 64
    return 8, 512


def solve_steady(grid, boundary: BoundarySpec, config: SolveConfig, phi0=None, exact=None,
                 *, device_result: bool = False, chunk: int | None = None,
                 comm=None) -> SolveReport:
    """March to the steady wall-distance field (solver.py:221-286).

    Stops when max |phi - phi_old| / Lref <= tol over non-mask nodes, or at
    max_iters (converged=False).  Raises DivergenceError like the reference.
    ``device_result=True`` (extension) keeps ``report.phi`` as a CUDA tensor.
    ``comm`` (extension): a communicator of
    :mod:`paper_2111_09859_b200.dist` -- the solve is decomposed into slabs of
    the periodic axis 0 over its ranks (one process per GPU); every rank
    passes the same global ``grid`` / ``phi0`` and gets the global field back.
    """
    import torch
    if not boundary.has_wall():
        raise ValueError("boundary spec pins no wall nodes (no Dirichlet anchor)")
    if comm is not None:
        return _solve_steady_dist(grid, boundary, config, phi0, exact, device_result, chunk, comm)
    fc = config.formulation
    ctx = NativeSolver(grid, boundary.faces, boundary.solid_mask, config.scheme, fc,
                       config.filter_config if config.uses_filter() else None, config.cfl,
                       config.tol, config.max_iters, arith=config.resolved_arith())
    try:
        lib = ctx.lib
        if phi0 is None:
            phi = torch.zeros(tuple(grid.dims), dtype=torch.float64, device="cuda")
        else:
            phi = ctx.field(phi0)
            if isinstance(phi0, torch.Tensor) and phi.data_ptr() == phi0.data_ptr():
                phi = phi.clone()  # the caller's device tensor is not to be overwritten
        hist = torch.zeros(max(config.max_iters, 1), dtype=torch.float64, device="cuda")
        nat.check(lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr()))
        stream = ctx.stream()
        n_nodes = int(np.prod(grid.dims))
        k, kmax = _chunk_sizes(n_nodes)
        if chunk is not None:
            k = kmax = int(chunk)
        sample_l2 = exact is not None and config.l2_every > 0
        if sample_l2:
            k = kmax = int(config.l2_every)
        if sample_l2 and tuple(np.shape(exact)) != tuple(grid.dims):
            # metrics.py l2_norm raises on a shape mismatch
            raise ValueError(f"exact field shape {tuple(np.shape(exact))} does not match the "
                             f"grid {tuple(grid.dims)}")
        exact_t = ctx.field(exact) if sample_l2 else None
        st = nat.Status()
        seconds = []
        l2_samples = []
        elapsed = 0.0
        done = 0
        while True:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            nat.check(lib.wd_steps(ctx.ptr, k))
            e1.record(stream)
            nat.check(lib.wd_read_status(ctx.ptr, ctypes.byref(st)))
            ran = st.iters - done
            dt_chunk = e0.elapsed_time(e1) / 1e3
            for j in range(ran):
                seconds.append(elapsed + dt_chunk * (j + 1) / max(ran, 1))
            elapsed += dt_chunk
            done = st.iters
            if sample_l2 and ran > 0 and st.state != nat.STATE_DIVERGED \
                    and done % config.l2_every == 0:
                nat.check(lib.wd_finish(ctx.ptr))
                l2_samples.append((done, _l2_norm(ctx, phi, exact_t, grid, config)))
            if st.state != nat.STATE_RUNNING:
                break
            k = min(2 * k, kmax)
        if st.state == nat.STATE_DIVERGED:
            limit = 1e6 * grid.ref_length
            raise DivergenceError(
                f"pseudo-time iteration diverged (max |phi| > {limit:g}) at iteration "
                f"{st.diverged_iter}")
        nat.check(lib.wd_finish(ctx.ptr))
        iters = st.iters
        res = hist[:iters].cpu().numpy().copy()
        report = SolveReport(phi=phi if device_result else nat.to_host(phi), iters=iters,
                             residual_history=res, wall_seconds=np.asarray(seconds[:iters]),
                             converged=st.state == nat.STATE_CONVERGED,
                             l2_history=np.asarray(l2_samples) if l2_samples else None)
        if fc.kind == "poisson":
            out = ctx.empty()
            nat.check(lib.wd_poisson_post(ctx.ptr, phi.data_ptr(), out.data_ptr()))
            report.phi_prime = report.phi
            report.phi = out if device_result else nat.to_host(out)
        return report
    finally:
        ctx.close()


def _solve_steady_dist(grid, boundary, config, phi0, exact, device_result, chunk, comm):
    """solve_steady on the slabs of ``comm`` (dist.DistributedSolve): the same
    loop, the stop decision taken in-device from all-reduced maxima, so every
    rank leaves it at the same iteration."""
    import torch
    from .dist import DistributedSolve
    fc = config.formulation
    if exact is not None and config.l2_every > 0:
        raise NotImplementedError("l2 sampling against an exact field is a single-GPU diagnostic")
    ds = DistributedSolve(grid, boundary.faces, config, comm, boundary.solid_mask)
    try:
        lo, hi = ds.slab.lo, ds.slab.hi
        local = None
        if phi0 is not None:
            local = phi0[lo:hi] if isinstance(phi0, torch.Tensor) else np.asarray(phi0)[lo:hi]
        ds.bind(local)
        stream = ds.stream()
        k, kmax = _chunk_sizes(int(np.prod(ds.local_dims)))
        if chunk is not None:
            k = kmax = int(chunk)
        seconds, elapsed, done = [], 0.0, 0
        while True:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ds.steps(k)
            e1.record(stream)
            st = ds.status()
            ran = st.iters - done
            dt_chunk = e0.elapsed_time(e1) / 1e3
            for j in range(ran):
                seconds.append(elapsed + dt_chunk * (j + 1) / max(ran, 1))
            elapsed += dt_chunk
            done = st.iters
            if st.state != nat.STATE_RUNNING:
                break
            k = min(2 * k, kmax)
        if st.state == nat.STATE_DIVERGED:
            limit = 1e6 * grid.ref_length
            raise DivergenceError(
                f"pseudo-time iteration diverged (max |phi| > {limit:g}) at iteration "
                f"{st.diverged_iter}")
        phi = ds.gather()
        iters = st.iters
        report = SolveReport(phi=phi if device_result else nat.to_host(phi), iters=iters,
                             residual_history=ds.history(),
                             wall_seconds=np.asarray(seconds[:iters]),
                             converged=st.state == nat.STATE_CONVERGED, l2_history=None)
        if fc.kind == "poisson":
            # the post-map's axis-0 derivatives are collective (pencils)
            out = torch.empty_like(ds.phi)
            nat.check(ds.lib.wd_poisson_post(ds.lib.wd_dist_context(ds.ptr), ds.phi.data_ptr(),
                                             out.data_ptr()))
            full = comm.allgather(out.reshape(-1)).view(tuple(grid.dims))
            report.phi_prime = report.phi
            report.phi = full if device_result else nat.to_host(full)
        return report
    finally:
        ds.close()


def _l2_norm(ctx, phi, exact_t, grid, config):
    """metrics.py:54-66 L2 error weighted by 1/J (diagnostic, outside timing;
    wd_l2_norm kernel)."""
    import torch
    p = phi
    if config.formulation.kind == "poisson":
        p = ctx.empty()
        # _l2_vs_exact (solver.py:289-293) post-maps WITHOUT re-applying BCs
        nat.check(ctx.lib.wd_poisson_map(ctx.ptr, phi.data_ptr(), p.data_ptr(), 0))
    if getattr(ctx, "_jac_dev", None) is None:
        ctx._jac_dev = torch.from_numpy(np.ascontiguousarray(grid.jacobian)).to("cuda")
    out = ctypes.c_double(0.0)
    torch.cuda.synchronize()
    nat.check(ctx.lib.wd_l2_norm(p.data_ptr(), exact_t.data_ptr(), ctx._jac_dev.data_ptr(), 0.0,
                                 p.numel(), ctypes.byref(out), None))
    return float(out.value)
