"""GPU: the C++ host driver examples/part_hmv_nccl.cpp (no Python on its data
path): P partitions emulated on one GPU (host-staged all-gathers between the
rank threads) and the NCCL communicator at one rank, each checked against the
whole-matrix h2b_hmv on the same x (max relative error <= 1e-12)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "part_hmv_nccl")


def run(*args):
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True)
    out = subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("P,nvec", [(1, 1), (2, 1), (4, 1), (8, 1), (4, 16), (2, 20)])
def test_cpp_driver_emulated(gpu, P, nvec):
    r = run("--dim", 2, "--n", 1 << 14, "--order", 8, "--emulate", P, "--nvec", nvec, "--steps", 3,
            "--warmup", 1, "--check")
    assert r["ranks"] == P and 0 <= r["check_rel_err"] <= 1e-12


def test_cpp_driver_emulated_3d_owned(gpu):
    r = run("--dim", 3, "--n", 1 << 14, "--order", 4, "--emulate", 8, "--owned", "--steps", 2, "--warmup", 1)
    assert r["y_mode"] == "owned" and r["ms_per_step"] > 0


def test_cpp_driver_nccl_one_rank(gpu):
    r = run("--dim", 2, "--n", 1 << 14, "--order", 8, "--gpus", 1, "--steps", 3, "--warmup", 1, "--check")
    assert r["comm"] == "nccl" and 0 <= r["check_rel_err"] <= 1e-12
