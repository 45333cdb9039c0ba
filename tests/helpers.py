"""Shared test helpers (no oracle logic here)."""
import numpy as np


def same(a, b):
    """Bit-identical up to the sign of zero (np.array_equal semantics),
    NaNs matching."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.array_equal(a, b, equal_nan=True))


def maxdiff(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b))) if a.size else 0.0
