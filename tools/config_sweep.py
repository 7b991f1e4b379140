"""Every BASELINE config on one B200 next to the reference's CPU times recorded
on the same host (tests/golden/config/*.json, 16 pinned threads): mat-vec
device time (CUDA events, 20 steps after 3 warm-ups, device x / y), the same
through the public API with pinned host x / y (synchronous), and compress
device / wall time at the config's eps.  One JSON line per config.
    python tools/config_sweep.py [C1 C2 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1902_01829_b200 as h2

GOLD = os.path.join("tests", "golden", "config")


def events(fn, steps, st):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run(name):
    meta = json.load(open(os.path.join(GOLD, name + ".json")))
    A = h2.H2Matrix.construct(meta["dim"], meta["n"], leaf_size=meta["leaf_size"], grid_order=meta["grid_order"])
    n, fp = meta["n"], A.memory_footprint()
    st = torch.cuda.current_stream()
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    for _ in range(3):
        h2.hmv(A, x, y)
    ms = events(lambda: h2.hmv(A, x, y), 20, st)
    xh = torch.rand(n, dtype=torch.float64).pin_memory()
    yh = torch.zeros(n, dtype=torch.float64).pin_memory()
    h2.hmv(A, xh.numpy(), yh.numpy())
    t0 = time.perf_counter()
    for _ in range(10):
        h2.hmv(A, xh.numpy(), yh.numpy())
    e2e = (time.perf_counter() - t0) * 100.0
    out = {"config": name, "n": n, "footprint_bytes": fp, "hmv_ms": round(ms, 4), "hmv_GBs": round(fp / ms / 1e6, 1),
           "hmv_e2e_ms": round(e2e, 4), "ref_hmv_ms_16t": round(meta["hmv_time"]["mean_ms"], 2),
           "hmv_speedup_vs_ref": round(meta["hmv_time"]["mean_ms"] / ms, 1)}
    if meta.get("eps") is not None:
        h2.compress(A, meta["eps"])  # warm: the workspace of this size is mapped once, then cached
        A.close()
        A = h2.H2Matrix.construct(meta["dim"], meta["n"], leaf_size=meta["leaf_size"],
                                  grid_order=meta["grid_order"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = h2.compress(A, meta["eps"])
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        g = meta["compress"]
        out.update({"compress_ms": round(rep.total_ms(), 2), "compress_wall_ms": round(wall, 2),
                    "compress_model_gflops": round(rep.total_flops() / rep.total_ms() / 1e6, 1),
                    "ref_compress_wall_ms_16t": round(1e3 * g["wall_s"], 1),
                    "compress_speedup_vs_ref": round(1e3 * g["wall_s"] / wall, 1),
                    "ranks_equal_reference": rep.new_ranks == g["new_ranks"]})
    A.close()
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C2alt", "C3", "C4"]
    # a first compress pays one-time workspace set-up: warm up on a small case
    w = h2.H2Matrix.construct(2, 1 << 14)
    h2.compress(w, 1e-7)
    w.close()
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
