"""GPU: the reference's OWN test programs, unmodified, run on the B200 through
the H2KIT_USE_B200 binding (include/h2kit_b200_bind.hpp: explicit
specializations of hmv / upsweep / tree_multiply / downsweep / block_sparse_mv /
compress / orthogonalize_basis / project_coupling / generate_weight_tree /
truncate_basis -> libh2b.so).  Built by tests/cpp/Makefile from
/root/reference/proj/tests/{test_hmv,test_compression,test_bsr,acceptance_test}.cpp
with tests/cpp/doctest/doctest.h for the absent vendor/doctest.h."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp")


def _run(name, timeout=1200):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd="/tmp")
    print(r.stdout[-4000:])
    return r


@pytest.mark.parametrize("suite", ["ref_test_hmv", "ref_test_compression", "ref_test_bsr"])
def test_reference_doctest_suite_through_binding(gpu, suite):
    r = _run(suite)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[doctest] Status: SUCCESS!" in r.stdout
    assert " 0 failed" in r.stdout


def test_reference_acceptance_suite_through_binding(gpu):
    r = _run("ref_acceptance_test", timeout=3000)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 8 and "[FAIL]" not in r.stdout
