"""The bench.py contract: one JSON line on stdout with the keys the driver
reads.  CPU: the reference arm (`--impl reference`, the reference's own CPU
path from oracle/_ref).  GPU: our arm at a small n."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout  # exactly one line, and it is JSON
    return json.loads(lines[0])


def test_reference_arm_line(ref):
    # (the default n = 2^22 needs ~90 GB of host RAM: the GPU host has 196 GB,
    # this container 62 GB -- the CPU suite runs the same code at n = 2^16)
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--n", str(1 << 16)], timeout=600)
    assert KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["n"] == 1 << 16 and d["config"]["same_config"] is True
    assert d["omp"]["OMP_PROC_BIND"] == "close" and d["one_thread"]["ms_per_step"] > 0
    assert d["host"]["logical_cpus"] >= 1


def test_cpu_baseline_child(ref):
    """Our arm's cpu_baseline leg: the reference on the same workload in a child process."""
    sys.path.insert(0, ROOT)
    import bench
    cb = bench.cpu_baseline_subprocess(dict(bench.WORKLOAD, n=1 << 14), timeout_s=300)
    assert cb["kind"] == "reference" and cb["value"] > 0 and cb["reps"] >= 5
    assert cb["omp"] == {"OMP_PROC_BIND": "close", "OMP_PLACES": "cores"}


@pytest.mark.gpu
def test_our_arm_line(gpu):
    d = _run(["--steps", "3", "--warmup", "3", "--no-compress", "--no-cpu-baseline", "--n", str(1 << 16)],
             timeout=900)
    assert KEYS | {"roofline", "gpu_launches", "clocks"} <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * (1 << 16) and d["e2e"]["value"] > 0
