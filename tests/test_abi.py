"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"^\s*(?:int|void\*|const char\*)\s+(wd_\w+)\(", src, re.M))
    return names


def test_header_declares_api():
    names = _declared()
    assert {"wd_create", "wd_steps", "wd_bind", "wd_derivative", "wd_filter",
            "wd_compute_metrics", "wd_tendency"} <= names


def test_library_exports_all_symbols():
    from paper_2111_09859_b200 import _native
    try:
        lib = _native.load()
    except _native.NativeUnavailableError as exc:
        pytest.fail(str(exc))
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_native.SIGNATURES) >= _declared()
    assert lib.wd_version() >= 100
    assert lib.wd_device_count() >= 0


def test_compute_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2111_09859_b200 import _native, operators
    import numpy as np
    with pytest.raises(_native.NativeUnavailableError):
        operators.central_derivative(np.zeros(9), "E4")
