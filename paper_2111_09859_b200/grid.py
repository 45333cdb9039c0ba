"""Structured curvilinear grids: coordinates, metric terms, Jacobian.

Drop-in for the reference ``walldist/grid.py`` (same names, conventions and
errors): arrays are node-based ``(ni, nj[, nk])``, axis 0 = xi, unit
computational spacing, ``metrics[l, m] = d xi_l / d x_m``, J > 0
(grid.py:1-12).

B200 layout: coordinates, metrics and Jacobian live on the GPU as fp64
C-order tensors (``grid.device_metrics()``); the numpy views the reference
API exposes are materialised lazily.  Uniform Cartesian grids
(``build_cartesian``) are analytic: the solver uses the diagonal constants
and never stores d^2 metric fields (the reference fills them with exact
constants, grid.py:116-120, so the arithmetic is identical).

EXTENSIONS: periodic axes (``periodic=`` flags, ``periods`` = coordinate
jump per period for differencing) and the BASELINE grid generators
``build_channel3d``, ``build_annulus``, ``build_cylinder``,
``build_sinusoidal_bump``.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import DegenerateMappingError, DimensionTooSmallError

MIN_NODES = 5  # grid.py:24


def _torch():
    import torch
    return torch


class CurvilinearGrid:
    """Node coordinates plus metric terms for a structured (i,j[,k]) mesh
    (grid.py:27-80)."""

    def __init__(self, coords=None, metrics=None, jacobian=None, ref_length=1.0,
                 periodic=None, periods=None):
        self._coords = None if coords is None else np.asarray(coords, dtype=float)
        self._metrics = None if metrics is None else np.asarray(metrics, dtype=float)
        self._jacobian = None if jacobian is None else np.asarray(jacobian, dtype=float)
        self.ref_length = float(ref_length)
        self._uniform = None          # (origin, spacing, dims) for analytic grids
        self._dims = None if self._coords is None else tuple(self._coords.shape[1:])
        nd = len(self._dims) if self._dims else 0
        self.periodic = tuple(bool(p) for p in (periodic or (False,) * nd))
        self.periods = None if periods is None else np.asarray(periods, dtype=float)
        self._dev = {}

    # -- construction helpers -------------------------------------------
    @classmethod
    def _analytic(cls, origin, spacing, dims, ref_length, periodic, extents):
        g = cls.__new__(cls)
        g._coords = g._metrics = g._jacobian = None
        g.ref_length = float(ref_length)
        g._uniform = (tuple(float(o) for o in origin), tuple(float(s) for s in spacing),
                      tuple(int(n) for n in dims), tuple(float(e) for e in extents))
        g._dims = tuple(int(n) for n in dims)
        g.periodic = tuple(bool(p) for p in periodic)
        nd = len(dims)
        g.periods = np.zeros((nd, nd))
        for d in range(nd):
            if g.periodic[d]:
                g.periods[d, d] = spacing[d] * dims[d]
        g._dev = {}
        return g

    # -- reference attributes ---------------------------------------------
    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def dims(self) -> tuple:
        return self._dims

    @property
    def is_uniform(self) -> bool:
        return self._uniform is not None

    @property
    def inv_spacing(self):
        return tuple(1.0 / s for s in self._uniform[1])

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None and self._uniform is not None:
            origin, spacing, dims, extents = self._uniform
            axes = []
            for d, n in enumerate(dims):
                if self.periodic[d]:
                    axes.append(origin[d] + spacing[d] * np.arange(n))
                else:
                    axes.append(np.linspace(origin[d], origin[d] + extents[d], n))
            self._coords = np.stack(np.meshgrid(*axes, indexing="ij"))
        return self._coords

    @coords.setter
    def coords(self, value):
        self._coords = np.asarray(value, dtype=float)
        self._dims = tuple(self._coords.shape[1:])
        self._uniform = None
        self._dev.clear()

    @property
    def metrics(self):
        if self._metrics is None:
            if self._uniform is not None:
                nd = self.ndim
                m = np.zeros((nd, nd) + self.dims)
                for d in range(nd):
                    m[d, d] = 1.0 / self._uniform[1][d]
                self._metrics = m
            elif "metrics" in self._dev:
                self._metrics = self._dev["metrics"].cpu().numpy()
        return self._metrics

    @metrics.setter
    def metrics(self, value):
        self._metrics = None if value is None else np.asarray(value, dtype=float)
        self._uniform_drop()
        self._dev.pop("metrics", None)

    @property
    def jacobian(self):
        if self._jacobian is None:
            if self._uniform is not None:
                self._jacobian = np.full(self.dims, float(np.prod(
                    [1.0 / s for s in self._uniform[1]])))
            elif "jacobian" in self._dev:
                self._jacobian = self._dev["jacobian"].cpu().numpy()
        return self._jacobian

    @jacobian.setter
    def jacobian(self, value):
        self._jacobian = None if value is None else np.asarray(value, dtype=float)
        self._dev.pop("jacobian", None)

    def _uniform_drop(self):
        if self._uniform is not None:
            _ = self.coords
            self._uniform = None

    @property
    def x(self):
        return self.coords[0]

    @property
    def y(self):
        return self.coords[1]

    @property
    def z(self):
        return self.coords[2]

    def metric(self, l: int, m: int) -> np.ndarray:
        return self.metrics[l, m]

    def metric_row_sumsq(self, l: int) -> np.ndarray:
        """S_l = sum_m (d xi_l / d x_m)^2 (grid.py:60-63)."""
        return np.sum(self.metrics[l] ** 2, axis=0)

    def local_spacing(self, l: int) -> np.ndarray:
        return 1.0 / np.sqrt(self.metric_row_sumsq(l))

    def min_spacing(self) -> np.ndarray:
        return np.min(np.stack([self.local_spacing(l) for l in range(self.ndim)]), axis=0)

    def new_field(self, fill: float = 0.0) -> np.ndarray:
        return np.full(self.dims, fill, dtype=float)

    def validate(self) -> None:
        if self.jacobian is not None and np.any(self.jacobian <= 0.0):
            raise DegenerateMappingError("Jacobian is not positive everywhere")

    # -- device views -------------------------------------------------------
    def device_metrics(self):
        """(d, d, N) fp64 CUDA tensor (None for analytic uniform grids)."""
        if self._uniform is not None:
            return None
        if "metrics" not in self._dev:
            if self._metrics is None:
                raise ValueError("grid has no metrics; call compute_metrics first")
            torch = _torch()
            self._dev["metrics"] = torch.from_numpy(
                np.ascontiguousarray(self._metrics)).to("cuda")
        return self._dev["metrics"]

    def device_coords(self):
        if "coords" not in self._dev:
            torch = _torch()
            self._dev["coords"] = torch.from_numpy(np.ascontiguousarray(self.coords)).to("cuda")
        return self._dev["coords"]


def _check_dims(dims, extents):
    """grid.py:83-90."""
    for n in dims:
        if n < MIN_NODES:
            raise DimensionTooSmallError(
                f"need at least {MIN_NODES} nodes per direction, got {dims}")
    for ext in extents:
        if ext <= 0.0:
            raise ValueError(f"extents must be positive, got {extents}")


def build_cartesian(ni, nj, nk=None, Lx=1.0, Ly=1.0, Lz=None,
                    origin=(0.0, 0.0, 0.0), ref_length=1.0, periodic=None) -> CurvilinearGrid:
    """Uniform axis-aligned Cartesian grid with analytic metrics
    (grid.py:93-122).  EXTENSION: a periodic axis has spacing L/n (its last
    node is one cell short of the period)."""
    if nk is None:
        dims, extents = (ni, nj), (Lx, Ly)
    else:
        dims, extents = (ni, nj, nk), (Lx, Ly, 1.0 if Lz is None else Lz)
    _check_dims(dims, extents)
    nd = len(dims)
    per = tuple(bool(p) for p in (periodic or (False,) * nd))
    spacing = [extents[d] / (dims[d] if per[d] else dims[d] - 1) for d in range(nd)]
    return CurvilinearGrid._analytic(origin[:nd], spacing, dims, ref_length, per, extents)


@dataclass(frozen=True)
class BumpParams:
    """Flat plate with a circular-arc bump on the lower wall (grid.py:125-156)."""

    length: float = 3.0
    domain_height: float = 1.0
    chord: float = 1.0
    height: float = 0.3
    center_x: float = 1.5

    def wall_y(self, x):
        x = np.asarray(x, dtype=float)
        y = np.zeros_like(x)
        if self.height <= 0.0:
            return y
        R = (0.25 * self.chord**2 + self.height**2) / (2.0 * self.height)
        yc = self.height - R
        dx = x - self.center_x
        on = np.abs(dx) <= 0.5 * self.chord
        y[on] = yc + np.sqrt(R**2 - dx[on] ** 2)
        return y

    def wall_polyline(self, n_samples: int = 20001) -> np.ndarray:
        xs = np.linspace(0.0, self.length, n_samples)
        return np.column_stack([xs, self.wall_y(xs)])


def build_bump_grid(ni: int, nj: int, params: BumpParams = BumpParams(),
                    scheme: str = "E4", ref_length: float = 1.0) -> CurvilinearGrid:
    """Body-fitted bump grid (grid.py:159-177); metrics on the GPU."""
    _check_dims((ni, nj), (params.length, params.domain_height))
    xs = np.linspace(0.0, params.length, ni)
    yw = params.wall_y(xs)
    if np.any(yw >= params.domain_height):
        raise DegenerateMappingError("bump reaches the upper boundary")
    s = np.linspace(0.0, 1.0, nj)
    x2 = np.repeat(xs[:, None], nj, axis=1)
    y2 = yw[:, None] * (1.0 - s[None, :]) + params.domain_height * s[None, :]
    grid = CurvilinearGrid(coords=np.stack([x2, y2]), ref_length=ref_length)
    compute_metrics(grid, scheme)
    if np.any(grid.jacobian <= 0.0):
        raise DegenerateMappingError("bump grid mapping is degenerate (J <= 0)")
    return grid


def compute_metrics(grid: CurvilinearGrid, scheme: str = "E2") -> CurvilinearGrid:
    """Metric terms and Jacobian by differencing the coordinates on the GPU
    (grid.py:180-217; kernel wd_compute_metrics).  2-D uses the reference's
    closed-form inverse (bit-identical); 3-D the closed-form cofactor inverse
    (the reference's LAPACK inverse agrees to round-off)."""
    torch = _torch()
    lib = nat.lib()
    if scheme not in nat.SCHEME_IDS:
        raise ValueError(f"unknown scheme {scheme!r}")
    grid._uniform_drop()
    nd = grid.ndim
    coords = grid.device_coords()
    N = int(np.prod(grid.dims))
    met = torch.empty((nd, nd) + tuple(grid.dims), dtype=torch.float64, device="cuda")
    jac = torch.empty(tuple(grid.dims), dtype=torch.float64, device="cuda")
    per = nat.int_array([1 if p else 0 for p in grid.periodic] + [0] * (3 - nd))
    periods = None
    if grid.periods is not None:
        periods = nat.double_array(np.asarray(grid.periods, dtype=float).ravel())
    stream = torch.cuda.current_stream().cuda_stream
    nat.check(lib.wd_compute_metrics(coords.data_ptr(), met.data_ptr(), jac.data_ptr(), nd,
                                     nat.int_array(grid.dims), nat.SCHEME_IDS[scheme], per,
                                     periods, stream))
    assert N == jac.numel()
    grid._dev["metrics"] = met
    grid._dev["jacobian"] = jac
    grid._metrics = None
    grid._jacobian = None
    return grid


# ------------------------------------------------------------------ EXTENSIONS
def tanh_stretch(n: int, beta: float) -> np.ndarray:
    """t in [0, 1] clustered at t = 0: 1 + tanh(beta (s - 1)) / tanh(beta)."""
    s = np.linspace(0.0, 1.0, n)
    return 1.0 + np.tanh(beta * (s - 1.0)) / np.tanh(beta)


def build_channel3d(n=512, L=1.0, ref_length=1.0) -> CurvilinearGrid:
    """BASELINE config 4: [0,1]^3 channel, walls at y = 0, 1, periodic x, z
    (dx = dz = L/n)."""
    return build_cartesian(n, n, n, Lx=L, Ly=L, Lz=L, ref_length=ref_length,
                           periodic=(True, False, True))


def build_sinusoidal_bump(ni=1025, nj=513, beta=1.069082, amp=0.1, length=4.0,
                          top=1.0, scheme="E6") -> CurvilinearGrid:
    """BASELINE config 3: wall y_w = amp sin(2 pi x), tanh wall-normal
    stretching (first cell ~1e-3 at beta = 1.069082), flat top."""
    x = np.linspace(0.0, length, ni)
    yw = amp * np.sin(2.0 * np.pi * x)
    t = tanh_stretch(nj, beta)
    X = np.repeat(x[:, None], nj, axis=1)
    Y = yw[:, None] * (1.0 - t[None, :]) + top * t[None, :]
    g = CurvilinearGrid(coords=np.stack([X, Y]))
    return compute_metrics(g, scheme)


def build_annulus(ntheta=257, nr=129, r0=0.5, r1=5.0, beta=3.041018,
                  scheme="C6") -> CurvilinearGrid:
    """BASELINE config 2: O-grid, theta clockwise (J > 0) and periodic."""
    th = -2.0 * np.pi * np.arange(ntheta) / ntheta
    r = r0 + (r1 - r0) * tanh_stretch(nr, beta)
    T, R = np.meshgrid(th, r, indexing="ij")
    g = CurvilinearGrid(coords=np.stack([R * np.cos(T), R * np.sin(T)]),
                        periodic=(True, False), periods=np.zeros((2, 2)))
    return compute_metrics(g, scheme)


def build_cylinder(ntheta=1024, nr=512, nz=256, r0=0.5, r1=10.0, lz=4.0,
                   beta=2.643022, scheme="C6") -> CurvilinearGrid:
    """BASELINE config 5: (theta periodic clockwise, r tanh-stretched, z
    periodic)."""
    th = -2.0 * np.pi * np.arange(ntheta) / ntheta
    r = r0 + (r1 - r0) * tanh_stretch(nr, beta)
    z = lz * np.arange(nz) / nz
    T, R, Z = np.meshgrid(th, r, z, indexing="ij")
    periods = np.zeros((3, 3))
    periods[2, 2] = lz
    g = CurvilinearGrid(coords=np.stack([R * np.cos(T), R * np.sin(T), Z]),
                        periodic=(True, False, True), periods=periods)
    return compute_metrics(g, scheme)


def write_grid_csv(grid: CurvilinearGrid, path) -> None:
    """Plain-text grid dump, one row per node: i,j[,k],x,y[,z],J (grid.py:220-231)."""
    ndim = grid.ndim
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["i", "j", "k"][:ndim] + ["x", "y", "z"][:ndim] + ["J"])
        coords, jac = grid.coords, grid.jacobian
        for idx in np.ndindex(*grid.dims):
            w.writerow(list(idx) + [coords[(d,) + idx] for d in range(ndim)] + [jac[idx]])


def read_grid_csv(path):
    with open(path, newline="") as fh:
        r = csv.reader(fh)
        header = next(r)
        ndim = sum(1 for name in header if name in ("x", "y", "z"))
        rows = [[float(v) for v in row] for row in r]
    data = np.asarray(rows)
    return data[:, :ndim].astype(int), data[:, ndim:2 * ndim], data[:, 2 * ndim]
