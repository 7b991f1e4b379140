"""GPU: the C++ drop-in shim (include/h2kit_b200.hpp) against the reference's
own C++ API, via the compiled tests/cpp/test_shim binary."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp", "test_shim")


def test_cpp_shim_suite(gpu):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_shim not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_shim_suite_strict_fingerprint(gpu):
    """The same suite with full-content fingerprints (H2KIT_B200_STRICT=1)."""
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_shim not built (needs the reference headers at build time)")
    env = dict(os.environ, H2KIT_B200_STRICT="1")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
