"""Line operators on the GPU (drop-in for ``walldist/operators.py``).

Every function runs the sm_100a kernels of libwd_b200.so; inputs may be
numpy arrays (copied to the device, result returned as numpy, like the
reference) or CUDA tensors (result stays a CUDA tensor).  Arithmetic is
bit-identical to the reference.

EXTENSIONS: scheme "E6" and ``periodic=True`` lines.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import LineTooShortError

CENTRAL_SCHEMES = ("E2", "E4", "E6", "C4", "C6")
SCHEMES = ("UW",) + CENTRAL_SCHEMES
_MIN_LEN = {"UW": 3, "E2": 3, "E4": 5, "E6": 7, "C4": 7, "C6": 7}

# interior relation alpha d[i-1] + d[i] + alpha d[i+1] = a (w+1 - w-1)/2
#   + b (w+2 - w-2)/4 [+ c (w+3 - w-3)/6]   (operators.py:27-34)
_SCHEME_COEFFS = {
    "E2": (0.0, 1.0, 0.0),
    "E4": (0.0, 4.0 / 3.0, -1.0 / 3.0),
    "C4": (0.25, 1.5, 0.0),
    "C6": (1.0 / 3.0, 14.0 / 9.0, 1.0 / 9.0),
    "E6": (0.0, 1.5, -0.6, 0.1),
}


def scheme_order(scheme: str) -> int:
    return {"UW": 1, "E2": 2, "E4": 4, "E6": 6, "C4": 4, "C6": 6}[scheme]


def _check_scheme(scheme: str) -> None:
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}; expected one of {SCHEMES}")


class _Dev:
    """numpy/torch <-> contiguous fp64 CUDA tensor."""

    def __init__(self, values):
        import torch
        self.torch = torch
        self.was_numpy = not isinstance(values, torch.Tensor)
        if self.was_numpy:
            arr = np.ascontiguousarray(np.asarray(values, dtype=float))
            self.t = torch.from_numpy(arr).to("cuda")
        else:
            self.t = values.to(device="cuda", dtype=torch.float64).contiguous()

    def out(self, t):
        return t.cpu().numpy() if self.was_numpy else t


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def central_derivative(line_values, scheme: str, axis: int = 0, periodic: bool = False):
    """First derivative along ``axis`` (operators.py:94-148) on the GPU."""
    _check_scheme(scheme)
    if scheme == "UW":
        raise ValueError("use upwind_front_derivative for the UW scheme")
    lib = nat.lib()
    d = _Dev(line_values)
    t = d.t
    if t.dim() == 0:
        raise ValueError("need at least a 1-D array")
    axis = axis % t.dim()
    n = t.shape[axis]
    need = 5 if periodic else _MIN_LEN[scheme]
    if n < need:
        raise LineTooShortError(f"{scheme} derivative needs at least {need} points, got {n}")
    shape = tuple(t.shape)
    # collapse to <= 3 dims around the axis: (before, n, after)
    before = int(np.prod(shape[:axis])) if axis else 1
    after = int(np.prod(shape[axis + 1:])) if axis + 1 < len(shape) else 1
    dims = (before, n, after)
    out = d.torch.empty_like(t)
    nat.check(lib.wd_derivative(t.data_ptr(), out.data_ptr(), 3, nat.int_array(dims), 1,
                                nat.SCHEME_IDS[scheme], 1 if periodic else 0, 0.0, _stream()))
    return d.out(out)


def fourth_derivative(line_values, axis: int = 0, periodic: bool = False):
    """Centered 5-point 4th derivative, boundary copy (operators.py:236-250)."""
    lib = nat.lib()
    d = _Dev(line_values)
    t = d.t
    axis = axis % t.dim()
    n = t.shape[axis]
    if n < 5:
        raise LineTooShortError(f"fourth derivative needs at least 5 points, got {n}")
    shape = tuple(t.shape)
    dims = (int(np.prod(shape[:axis])) if axis else 1, n,
            int(np.prod(shape[axis + 1:])) if axis + 1 < len(shape) else 1)
    out = d.torch.empty_like(t)
    nat.check(lib.wd_fourth_derivative(t.data_ptr(), out.data_ptr(), 3, nat.int_array(dims), 1,
                                       1 if periodic else 0, _stream()))
    return d.out(out)


@dataclass(frozen=True)
class FilterConfig:
    """Implicit filter setup (operators.py:253-266): alpha_f in [0.40, 0.5]."""

    alpha_f: float = 0.49

    def __post_init__(self):
        if not 0.40 <= self.alpha_f <= 0.5:
            raise ValueError(f"alpha_f must lie in [0.40, 0.5], got {self.alpha_f}")


def apply_filter(field, axis: int, filter_config: FilterConfig, pinned=None,
                 periodic: bool = False):
    """10th-order implicit filter along ``axis`` (operators.py:305-352)."""
    lib = nat.lib()
    d = _Dev(field)
    t = d.t
    axis = axis % t.dim()
    shape = tuple(t.shape)
    n = shape[axis]
    dims = (int(np.prod(shape[:axis])) if axis else 1, n,
            int(np.prod(shape[axis + 1:])) if axis + 1 < len(shape) else 1)
    pin = None
    if pinned is not None:
        torch = d.torch
        pm = pinned if isinstance(pinned, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(pinned, dtype=bool)))
        pin = pm.to(device="cuda", dtype=torch.uint8).contiguous()
    out = d.torch.empty_like(t)
    nat.check(lib.wd_filter(t.data_ptr(), out.data_ptr(), None if pin is None else pin.data_ptr(),
                            3, nat.int_array(dims), 1, float(filter_config.alpha_f),
                            1 if periodic else 0, _stream()))
    return d.out(out)


def solve_tridiagonal(lower, diag, upper, rhs):
    """Batched tridiagonal solve in LAPACK dgtsv order (operators.py:53-78).
    rhs (n,) or (n, m); the same matrix for every column."""
    lib = nat.lib()
    diag = np.ascontiguousarray(np.asarray(diag, dtype=float))
    lower = np.ascontiguousarray(np.asarray(lower, dtype=float))
    upper = np.ascontiguousarray(np.asarray(upper, dtype=float))
    n = diag.shape[0]
    d = _Dev(rhs)
    t = d.t.clone()
    m = 1 if t.dim() == 1 else int(np.prod(t.shape[1:]))
    import ctypes
    dp = ctypes.POINTER(ctypes.c_double)
    nat.check(lib.wd_solve_tridiagonal(lower.ctypes.data_as(dp), diag.ctypes.data_as(dp),
                                       upper.ctypes.data_as(dp), t.data_ptr(), n, m, _stream()))
    return d.out(t)
