"""Loading of the committed golden fixtures (made by tests/golden/make_golden.py
from the reference implementation)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


def load(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        import pytest
        pytest.skip(f"golden {name} not generated")
    return dict(np.load(path, allow_pickle=False))


def solve_cases():
    return sorted(os.path.basename(p)[len("solve_"):-4]
                  for p in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


def case_faces(z):
    return dict(zip(FACES, [str(f) for f in z["faces"]]))


def case_alpha(z):
    a = float(z["alpha_f"])
    return None if np.isnan(a) else a
