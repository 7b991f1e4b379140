"""CPU: the C-ABI library loads, exports every symbol include/h2b.h declares,
and fails loudly (no CPU fallback) without a device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "h2b.h")).read()
    return sorted(set(re.findall(r"\b(h2b_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1902_01829_b200 import _lib
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 19
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}$", out, re.M), name
    assert set(_lib.EXPORTED_SYMBOLS) <= set(names)


def test_library_is_sm100a_only():
    from paper_1902_01829_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_oracle_in_product():
    """The product library never links or loads the oracle."""
    from paper_1902_01829_b200 import _lib
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "h2ref" not in out
    for f in os.listdir(os.path.join(ROOT, "paper_1902_01829_b200")):
        if f.endswith(".py"):
            assert "import oracle" not in open(os.path.join(ROOT, "paper_1902_01829_b200", f)).read()


def test_compute_fails_loudly_without_device():
    from paper_1902_01829_b200 import _lib, H2Matrix, H2bNoDevice
    lib = _lib.load()
    if lib.h2b_device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(H2bNoDevice):
        H2Matrix.construct(2, 1024)
    import oracle
    hm = oracle.restated().construct(2, 1024).to_host()
    with pytest.raises(H2bNoDevice):
        H2Matrix.from_host(hm)


def test_invalid_arguments_before_device():
    """Argument validation mirrors the reference's require() messages."""
    from paper_1902_01829_b200 import H2Matrix, H2bInvalidArgument
    with pytest.raises(H2bInvalidArgument, match="dim must be 2 or 3"):
        H2Matrix.construct(4, 1024)
    with pytest.raises(H2bInvalidArgument, match="eta must be positive"):
        H2Matrix.construct(2, 1024, eta=0.0)
    with pytest.raises(ValueError):
        H2Matrix.construct(2, 900)


def test_hostmatrix_validate_rejects_bad_sizes(orc):
    """api.H2Matrix.from_host validates every pool size before the C call
    (the C side copies exactly the sizes implied by n, ranks and row_ptr)."""
    import numpy as np
    import pytest
    hm = orc.construct(2, 1024).to_host()
    hm.validate()
    bad = hm.copy()
    bad.leaf = bad.leaf[:-1]
    with pytest.raises(ValueError):
        bad.validate()
    bad = hm.copy()
    bad.perm = bad.perm.astype(np.int64)
    with pytest.raises(ValueError):
        bad.validate()
    bad = hm.copy()
    bad.cpl_values = np.zeros(3)
    with pytest.raises(ValueError):
        bad.validate()
