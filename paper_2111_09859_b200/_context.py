"""Owner of a native solver context (wd_ctx) and the device buffers it reads."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

FACE_NAMES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


def face_codes(grid, faces: dict | None):
    """WD_FACE_* per face; periodic axes come from the grid (EXTENSION)."""
    codes = [nat.FACE_IDS[None]] * 6
    faces = faces or {}
    for ax in range(grid.ndim):
        lo, hi = FACE_NAMES[2 * ax], FACE_NAMES[2 * ax + 1]
        per = bool(grid.periodic[ax]) if grid.periodic else False
        klo, khi = faces.get(lo), faces.get(hi)
        if per:
            for k in (klo, khi):
                if k not in (None, "periodic"):
                    raise ValueError(f"axis {ax} is periodic but face kind {k!r} was given")
            codes[2 * ax] = codes[2 * ax + 1] = nat.FACE_IDS["periodic"]
        else:
            for k in (klo, khi):
                if k == "periodic":
                    raise ValueError(f"face of axis {ax} is 'periodic' but the grid is not")
            codes[2 * ax] = nat.FACE_IDS[klo]
            codes[2 * ax + 1] = nat.FACE_IDS[khi]
    return codes


class NativeSolver:
    """wd_ctx for (grid, faces, mask, scheme, formulation, filter, cfl, tol)."""

    def __init__(self, grid, faces=None, solid_mask=None, scheme="E2", formulation=None,
                 filter_config=None, cfl=0.5, tol=1e-5, max_iters=1, arith="exact"):
        import torch
        from .formulations import FormulationConfig
        self.torch = torch
        self.lib = nat.lib()
        fc = formulation or FormulationConfig()
        if scheme not in nat.SCHEME_IDS:
            raise ValueError(f"unknown scheme {scheme!r}")
        self.grid = grid
        gd = nat.GridDesc()
        gd.ndim = grid.ndim
        for a, n in enumerate(grid.dims):
            gd.dims[a] = int(n)
        for i, c in enumerate(face_codes(grid, faces)):
            gd.face[i] = c
        self._keep = []
        if grid.is_uniform:
            gd.uniform = 1
            for a, c in enumerate(grid.inv_spacing):
                gd.inv_spacing[a] = c
            gd.metrics_dev = None
        else:
            gd.uniform = 0
            met = grid.device_metrics()
            self._keep.append(met)
            gd.metrics_dev = met.data_ptr()
        if solid_mask is not None:
            m = solid_mask if isinstance(solid_mask, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(solid_mask, dtype=bool)))
            m = m.to(device="cuda", dtype=torch.uint8).contiguous()
            if tuple(m.shape) != tuple(grid.dims):
                raise ValueError("solid_mask shape does not match the grid")
            self._keep.append(m)
            gd.solid_mask_dev = m.data_ptr()
        gd.ref_length = float(grid.ref_length)
        sd = nat.SolverDesc()
        sd.scheme = nat.SCHEME_IDS[scheme]
        sd.kind = nat.KIND_IDS[fc.kind]
        sd.epsilon = float(fc.epsilon)
        sd.lad_c = float(fc.lad_c)
        sd.eps0 = float(fc.eps0) if fc.eps0 is not None else 1e-12 / grid.ref_length
        sd.use_filter = 1 if (filter_config is not None and scheme != "UW") else 0
        sd.alpha_f = float(filter_config.alpha_f) if filter_config is not None else 0.0
        sd.cfl = float(cfl)
        sd.tol = float(tol)
        sd.max_iters = int(max_iters)
        sd.arith = {"exact": 0, "fast": 1}[arith]
        self.gd, self.sd = gd, sd
        ptr = ctypes.c_void_p()
        torch.cuda.synchronize()
        nat.check(self.lib.wd_create(ctypes.byref(gd), ctypes.byref(sd), None, ctypes.byref(ptr)))
        self.ptr = ptr

    @property
    def fused(self) -> bool:
        return bool(self.lib.wd_fused_active(self.ptr))

    def stream(self):
        return self.torch.cuda.ExternalStream(self.lib.wd_get_stream(self.ptr))

    def close(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            self.lib.wd_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
    def field(self, values):
        torch = self.torch
        if isinstance(values, torch.Tensor):
            return values.to(device="cuda", dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(values, dtype=float))).to("cuda")

    def empty(self):
        return self.torch.empty(tuple(self.grid.dims), dtype=self.torch.float64, device="cuda")


# ---------------------------------------------------------------------------
# Operator-level calls (tendency, local_timestep, rk4_step, gradient_magnitude,
# poisson_postprocess ...) each need a context for (grid, scheme, formulation);
# building and destroying one per call costs a workspace allocation, the host
# factorisation and a device synchronisation.  A few
# contexts are kept, keyed by the grid OBJECT (held alive by the entry, its
# device metrics tensor checked for identity) and the configuration; grids
# above _CACHE_MAX_NODES and calls with a solid mask build a private context.
from collections import OrderedDict  # noqa: E402
import dataclasses  # noqa: E402

_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_SLOTS = 4
_CACHE_MAX_NODES = 4_000_000


def acquire(grid, faces=None, solid_mask=None, scheme="E2", formulation=None,
            filter_config=None, cfl=0.5, tol=1e-5, max_iters=1, arith="exact", key_extra=None):
    """(context, cached): a context for this configuration; release() it."""
    n_nodes = int(np.prod(grid.dims))
    if solid_mask is not None or n_nodes > _CACHE_MAX_NODES:
        return NativeSolver(grid, faces, solid_mask, scheme, formulation, filter_config, cfl,
                            tol, max_iters, arith=arith), False
    fc = dataclasses.astuple(formulation) if formulation is not None else None
    gkey = key_extra if key_extra is not None else id(grid)
    key = (gkey, tuple(sorted((faces or {}).items())), scheme, fc,
           None if filter_config is None else float(filter_config.alpha_f), float(cfl),
           float(tol), int(max_iters), arith)
    ent = _CACHE.get(key)
    if ent is not None:
        ctx, kept_grid, met = ent
        same_grid = key_extra is not None or kept_grid is grid
        same_met = grid.is_uniform or grid.device_metrics() is met
        if same_grid and same_met and ctx.ptr is not None:
            _CACHE.move_to_end(key)
            return ctx, True
        _CACHE.pop(key)
        ctx.close()
    ctx = NativeSolver(grid, faces, None, scheme, formulation, filter_config, cfl, tol,
                       max_iters, arith=arith)
    _CACHE[key] = (ctx, grid, None if grid.is_uniform else grid.device_metrics())
    while len(_CACHE) > _CACHE_SLOTS:
        _, (old, _g, _m) = _CACHE.popitem(last=False)
        old.close()
    return ctx, True


def release(ctx, cached):
    if not cached:
        ctx.close()


def drop_cached():
    """Close every cached context (tests, interpreter shutdown)."""
    while _CACHE:
        _, (ctx, _g, _m) = _CACHE.popitem()
        ctx.close()
