"""B200-native pseudo-time wall-distance solver (arXiv 2111.09859 hot path).

Drop-in for the reference package ``walldist`` (``__init__.py:9-29``):
same names, signatures, dataclasses and exceptions, with every hot-path
operation executed by hand-written sm_100a CUDA kernels in libwd_b200.so
(C ABI: include/walldist_b200.h).  There is no CPU fallback: compute calls
raise ``NativeUnavailableError`` when the library or a CUDA device is
missing.
"""

from .grid import (BumpParams, CurvilinearGrid, build_annulus, build_bump_grid,
                   build_cartesian, build_channel3d, build_cylinder,
                   build_sinusoidal_bump, compute_metrics)
from .operators import FilterConfig
from .formulations import FormulationConfig
from .solver import BoundarySpec, SolveConfig, SolveReport, solve_steady
from .unsteady import MotionSpec, solve_unsteady
from ._native import NativeUnavailableError

__all__ = [
    "CurvilinearGrid",
    "build_cartesian",
    "build_bump_grid",
    "compute_metrics",
    "FilterConfig",
    "FormulationConfig",
    "BoundarySpec",
    "MotionSpec",
    "SolveConfig",
    "SolveReport",
    "solve_steady",
    "solve_unsteady",
    "BumpParams",
    "build_channel3d",
    "build_annulus",
    "build_cylinder",
    "build_sinusoidal_bump",
    "NativeUnavailableError",
]

__version__ = "0.1.0"
