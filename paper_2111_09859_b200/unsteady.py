"""Moving-body re-solves (drop-in for ``walldist/solver.py:296-410``:
``MotionSpec`` and ``solve_unsteady``).

The caller of the hot path: at every physical step the solid mask of the
prescribed body is rebuilt on the host and ``solve_steady`` runs again,
warm-started from the previous field.  Here the warm start stays on the
device (``solve_steady(..., device_result=True)``), so a physical step
costs one mask upload and the pseudo-time iterations; the reports carry
host copies like the reference's.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import BodyOutsideDomainError
from .solver import (FARFIELD, WALL, _FACE_NAMES, BoundarySpec, SolveConfig, SolveReport,
                     all_wall_faces, solve_steady)

_MOTIONS = ("none", "piston_sinusoid", "bouncing_cube")


@dataclass(frozen=True)
class MotionSpec:
    """Prescribed body motion (solver.py:296-389).

    ``piston_sinusoid``: solid for x <= x0 + amplitude sin(2 pi t / period)
    in an all-wall chamber.  ``bouncing_cube``: a square of side ``size``
    dropped from rest at ``y_start`` under ``gravity`` between walls at the
    bottom and top, each floor impact keeping a fraction 1 - energy_loss of
    the kinetic energy, parked once the rebound apex is negligible.
    ``physical_dt`` is the physical time between re-solves.
    """

    kind: str = "none"
    physical_dt: float = 0.05
    x0: float = 0.3
    amplitude: float = 0.15
    period: float = 1.0
    size: float = 0.2
    x_center: float = 0.5
    y_start: float = 0.7
    gravity: float = 2.0
    energy_loss: float = 0.2

    def __post_init__(self):
        if self.kind not in _MOTIONS:
            raise ValueError(f"unknown motion kind {self.kind!r}")
        if self.physical_dt <= 0.0:
            raise ValueError("physical_dt must be positive")

    def default_faces(self, ndim: int) -> dict:
        """All walls, except the cube case: walls at jmin/jmax only."""
        if self.kind != "bouncing_cube":
            return all_wall_faces(ndim)
        faces = {name: FARFIELD for name in _FACE_NAMES[:2 * ndim]}
        faces["jmin"] = faces["jmax"] = WALL
        return faces

    def piston_position(self, t: float) -> float:
        return self.x0 + self.amplitude * math.sin(2.0 * math.pi * t / self.period)

    def cube_center_y(self, t: float, floor_y: float) -> float:
        """Centre height at time t: ballistic arcs between floor impacts
        (solver.py:343-367, same operation order)."""
        rest = floor_y + 0.5 * self.size
        g = self.gravity
        keep = math.sqrt(1.0 - self.energy_loss)
        y, v, t_arc = self.y_start, 0.0, 0.0
        for _ in range(10000):
            # first root of y + v s - g s^2 / 2 = rest (the impact)
            qa, qb, qc = -0.5 * g, v, y - rest
            s_hit = (-qb - math.sqrt(max(qb * qb - 4.0 * qa * qc, 0.0))) / (2.0 * qa)
            if t - t_arc < s_hit:
                s = t - t_arc
                return y + v * s - 0.5 * g * s * s
            t_arc += s_hit
            v = -(v - g * s_hit) * keep
            y = rest
            if v * v / (2.0 * g) < 1e-4 * self.size:
                return rest
        return rest

    def body_mask(self, grid, t: float) -> np.ndarray | None:
        """Solid nodes at time t, nearest-node quantised (solver.py:369-389)."""
        if self.kind == "none":
            return None
        x, y = grid.x, grid.y
        hx = 0.5 * (x.max() - x.min()) / (grid.dims[0] - 1)
        hy = 0.5 * (y.max() - y.min()) / (grid.dims[1] - 1)
        if self.kind == "piston_sinusoid":
            xp = self.piston_position(t)
            if not x.min() < xp < x.max():
                raise BodyOutsideDomainError(
                    f"piston face x={xp:.4f} leaves the domain at t={t:.4f}")
            return x <= xp + hx
        yc = self.cube_center_y(t, floor_y=y.min())
        half = 0.5 * self.size
        if (yc + half > y.max() or self.x_center - half < x.min()
                or self.x_center + half > x.max()):
            raise BodyOutsideDomainError(f"cube leaves the domain at t={t:.4f}")
        return (np.abs(x - self.x_center) <= half + hx) & (np.abs(y - yc) <= half + hy)


def solve_unsteady(grid, motion: MotionSpec, config: SolveConfig, n_steps: int,
                   faces: dict | None = None) -> list[SolveReport]:
    """Re-solve the wall distance at t = step * physical_dt, each solve
    warm-started from the previous field (solver.py:392-410)."""
    if faces is None:
        faces = motion.default_faces(grid.ndim)
    reports = []
    phi = None  # device tensor between physical steps
    for step in range(n_steps):
        t = step * motion.physical_dt
        bnd = BoundarySpec(faces=dict(faces), solid_mask=motion.body_mask(grid, t))
        rep = solve_steady(grid, bnd, config, phi0=phi, device_result=True)
        phi = rep.phi
        rep.phi = nat.to_host(phi)
        if rep.phi_prime is not None:
            rep.phi_prime = nat.to_host(rep.phi_prime)
        rep.time = t
        reports.append(rep)
    return reports
