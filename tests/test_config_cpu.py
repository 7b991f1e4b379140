"""The config-scale goldens (tests/golden/config/, written by the real reference
on the GPU host) pinned against the CPU restatement where it runs in seconds:
C1 / C1k64 construct + hmv bit for bit, compress ranks / bytes / error.  Also
checks every golden file is complete (what test_config_gpu.py reads)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR

CONFIG_DIR = os.path.join(GOLDEN_DIR, "config")
CASES = ["C1", "C1k64", "C2", "C2alt", "C3", "C4"]


def load_case(name):
    with open(os.path.join(CONFIG_DIR, name + ".json")) as f:
        meta = json.load(f)
    arr = np.load(os.path.join(CONFIG_DIR, name + ".npz"))
    return meta, {k: arr[k] for k in arr.files}


@pytest.mark.parametrize("case", CASES)
def test_config_golden_complete(case):
    meta, arr = load_case(case)
    assert meta["case"] == case
    assert len(arr["idx"]) == min(meta["n"], 1 << 16) == len(arr["y"])
    assert np.all(np.diff(arr["idx"]) > 0) and arr["idx"][-1] < meta["n"]
    assert meta["footprint"] > 0 and meta["hmv_time"]["reps"] >= 1
    if meta["eps"] is not None:
        assert len(meta["compress"]["new_ranks"]) == len(meta["ranks"])
        assert len(arr["yc"]) == len(arr["idx"])


@pytest.mark.parametrize("case", ["C1", "C1k64"])
def test_config_golden_vs_restatement(orc, case):
    meta, arr = load_case(case)
    O = orc.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
    assert O.footprint() == meta["footprint"]
    x = orc.random_vector(meta["n"], 1)
    y = O.hmv(x)
    assert np.array_equal(y[arr["idx"]], arr["y"])  # the restatement is bit-identical
    rep = O.compress(meta["eps"])
    g = meta["compress"]
    assert rep["new_ranks"] == g["new_ranks"]
    assert int(rep["bytes_after"]) == int(g["bytes_after"])
    assert rep["frobenius_error"] == g["frobenius_error"]
    assert np.array_equal(O.hmv(x)[arr["idx"]], arr["yc"])
