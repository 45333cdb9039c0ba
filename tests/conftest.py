import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def ref():
    """The reference package, imported read-only (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not present (GPU box)")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import walldist  # noqa: F401
    from walldist import operators, formulations, solver, grid, errors
    return type("Ref", (), dict(ops=operators, forms=formulations, solver=solver,
                                grid=grid, errors=errors))
