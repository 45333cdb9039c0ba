"""Residual evaluators (drop-in for ``walldist/formulations.py``).

The five formulations (eikonal, hj, hj_lad, hj_curvature, poisson) are
evaluated by the libwd_b200 kernels (wd_tendency), bit-identical to the
reference.  ``FormulationConfig`` keeps the reference's validation
(formulations.py:39-63).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import _context

FORMULATIONS = ("eikonal", "hj", "hj_lad", "hj_curvature", "poisson")


@dataclass(frozen=True)
class FormulationConfig:
    """Formulation choice plus its coefficients (formulations.py:39-63)."""

    kind: str = "eikonal"
    epsilon: float = 0.2
    lad_c: float = 0.1
    eps0: float | None = None

    def __post_init__(self):
        if self.kind not in FORMULATIONS:
            raise ValueError(f"unknown formulation {self.kind!r}; expected {FORMULATIONS}")
        if self.epsilon < 0.0:
            raise ValueError("epsilon must be non-negative")
        if self.lad_c < 0.0:
            raise ValueError("lad_c must be non-negative")
        if self.eps0 is not None and self.eps0 <= 0.0:
            raise ValueError("eps0 must be positive")


def _as_out(values, t):
    import torch
    return t if isinstance(values, torch.Tensor) else t.cpu().numpy()


def tendency(phi, grid, scheme: str, config: FormulationConfig):
    """Pseudo-time derivative d(phi)/dt* (formulations.py:244-252)."""
    ctx, cached = _context.acquire(grid, scheme=scheme, formulation=config)
    try:
        p = ctx.field(phi)
        k = ctx.empty()
        nat.check(ctx.lib.wd_tendency(ctx.ptr, p.data_ptr(), k.data_ptr()))
        return _as_out(phi, k)
    finally:
        _context.release(ctx, cached)


def residual(phi, grid, scheme: str, config: FormulationConfig):
    """formulations.py:232-241 (the Poisson residual is -tendency)."""
    k = tendency(phi, grid, scheme, config)
    return -k if config.kind == "poisson" else k


def eikonal_residual(phi, grid, scheme: str):
    return tendency(phi, grid, scheme, FormulationConfig(kind="eikonal"))


def hj_residual(phi, grid, scheme: str, config: FormulationConfig):
    kind = config.kind if config.kind in ("hj", "hj_lad") else "hj"
    cfg = FormulationConfig(kind=kind, epsilon=config.epsilon, lad_c=config.lad_c,
                            eps0=config.eps0)
    return tendency(phi, grid, scheme, cfg)


def hj_curvature_residual(phi, grid, scheme: str, config: FormulationConfig):
    cfg = FormulationConfig(kind="hj_curvature", epsilon=config.epsilon, lad_c=config.lad_c,
                            eps0=config.eps0)
    return tendency(phi, grid, scheme, cfg)


def poisson_residual(phi_prime, grid, scheme: str):
    return residual(phi_prime, grid, scheme, FormulationConfig(kind="poisson"))


def gamma_standard(phi, epsilon: float):
    """Gamma = eps * phi (formulations.py:159-161)."""
    return epsilon * np.asarray(phi, dtype=float)


def poisson_postprocess(phi_prime, grid, scheme: str):
    """phi = -|grad phi'| + sqrt(|grad phi'|^2 + 2 phi') (formulations.py:255-270)."""
    ctx, cached = _context.acquire(grid, scheme=scheme,
                                   formulation=FormulationConfig(kind="poisson"))
    try:
        p = ctx.field(phi_prime)
        out = ctx.empty()
        nat.check(ctx.lib.wd_poisson_post(ctx.ptr, p.data_ptr(), out.data_ptr()))
        return _as_out(phi_prime, out)
    finally:
        _context.release(ctx, cached)
