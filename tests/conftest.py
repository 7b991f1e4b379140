import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        idx = json.load(f)
    out = {}
    for name, meta in idx.items():
        arr = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        out[name] = (meta, {k: arr[k] for k in arr.files})
    return out


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.restated()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.reference()


@pytest.fixture(scope="session")
def gpu():
    """The product library on a real device; skips (CPU suite) when absent."""
    from paper_1902_01829_b200 import _lib
    lib = _lib.load()
    if lib.h2b_device_count() == 0:
        pytest.skip("no sm_100 device")
    return lib


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
