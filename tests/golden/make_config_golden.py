"""Config-scale golden values from the REAL reference (oracle/_ref), run on the
GPU host (196 GB RAM, enough for C3 / C4), plus the reference's CPU timings on
that host's cores (the bench's CPU baseline).  TEST INFRASTRUCTURE ONLY.

    python tests/golden/make_config_golden.py --case C4 --out DIR

One case per process (the matrices are 10-80 GB).  tools/run_config_golden.sh
runs every case on a gpurun box; the JSON/NPZ it writes are copied into
tests/golden/config/ and committed.  Recorded per case:

* the reference's construct() (h2kit.cpp:28-57 parameters: perturbation 0.25,
  seed 1, eta 2.0, leaf 64, ell 0.1 / 0.2), its footprint and hmv flop model;
* y = hmv(A, x) for x = random_vector(n, 1) (hmv.hpp:175-188): ||y||_2, sum(y)
  and y at 65 536 fixed indices (all of y when n <= 2^16);
* compress(A, eps) (compression.hpp:466-551): per-level ranks, frobenius
  error / norm, bytes before / after, model flops per phase, and y after
  compression at the same indices;
* timings: hmv with one HmvContext (the CLI matvec loop, h2kit.cpp:104-141),
  OMP_PROC_BIND=close OMP_PLACES=cores, all host threads (mean of >= 5) and 1
  thread; construct and compress wall time; the host's CPU model, cores, RAM.
"""
import argparse
import json
import os
import sys
import time

# OpenMP pinning must be in the environment before libgomp is loaded.
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import numpy as np  # noqa: E402

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import oracle  # noqa: E402

# name: (dim, n, grid_order, eps, one_thread_compress)
CASES = {
    "C1": (2, 1 << 14, 4, 1e-7, True),       # 2D 2^14 k16
    "C1k64": (2, 1 << 14, 8, 1e-7, True),    # 2D 2^14 k64 (SURVEY §8c golden)
    "C2": (2, 1 << 20, 6, 1e-7, False),      # 2D 2^20 k36
    "C2alt": (2, 1 << 20, 8, 1e-7, False),   # 2D 2^20 k64
    "C3": (3, 1 << 20, 4, 1e-6, False),      # 3D 2^20 k64
    "C4": (2, 1 << 22, 8, None, False),      # 2D 2^22 k64 (hmv only)
}
NSAMPLE = 1 << 16


def sample_index(n):
    """Fixed indices: all of them for n <= 2^16, else one per stride, jittered
    inside the stride (every leaf of the tree is hit)."""
    if n <= NSAMPLE:
        return np.arange(n, dtype=np.int64)
    stride = n // NSAMPLE
    i = np.arange(NSAMPLE, dtype=np.int64)
    return i * stride + (i * 7919) % stride


def host_info():
    model, mem = "unknown", 0
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    mem = int(ln.split()[1]) * 1024
                    break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "mem_total_bytes": mem,
            "omp_proc_bind": os.environ.get("OMP_PROC_BIND"), "omp_places": os.environ.get("OMP_PLACES")}


def time_hmv(R, A, x, threads, min_reps, budget_s):
    """Mean seconds per hmv with one HmvContext (ref_hmv_reps), after 1 warm-up."""
    R.set_threads(threads)
    y = np.zeros_like(x)
    fn = R.lib.ref_hmv_reps
    R.check(fn(A.h, x.ctypes.data, y.ctypes.data, 1))
    times = []
    t_all = time.time()
    while len(times) < min_reps or (time.time() - t_all < budget_s and len(times) < 50):
        t = time.perf_counter()
        R.check(fn(A.h, x.ctypes.data, y.ctypes.data, 1))
        times.append(time.perf_counter() - t)
        if time.time() - t_all > 4 * budget_s:
            break
    return times


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True, choices=sorted(CASES))
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    dim, n, order, eps, one_thread_compress = CASES[args.case]
    R = oracle.reference()
    threads = os.cpu_count() or 1
    R.set_threads(threads)
    rec = {"case": args.case, "dim": dim, "n": n, "grid_order": order, "leaf_size": 64, "eta": 2.0,
           "ell": 0.1 if dim == 2 else 0.2, "perturbation": 0.25, "seed": 1, "eps": eps,
           "host": host_info(), "threads": R.max_threads()}
    t0 = time.time()
    A = R.construct(dim, n, grid_order=order)
    rec["construct_s"] = time.time() - t0
    ranks, nb, nd = A.layout()
    rec["ranks"] = [int(r) for r in ranks]
    rec["cpl_blocks"] = [int(v) for v in nb]
    rec["dense_blocks"] = nd
    rec["footprint"] = A.footprint()
    x = R.random_vector(n, 1)
    R.fn("flops_reset")()
    y = A.hmv(x)
    rec["hmv_flops"] = float(R.fn("flops_total")())
    idx = sample_index(n)
    rec["y_norm2"] = float(np.linalg.norm(y))
    rec["y_sum"] = float(y.sum())
    arrays = {"idx": idx, "y": y[idx]}
    print(args.case, "built", rec["construct_s"], "s; ranks", rec["ranks"], flush=True)

    t_all = time_hmv(R, A, x, threads, 5, 10.0)
    t_one = time_hmv(R, A, x, 1, 1, 20.0)
    R.set_threads(threads)
    rec["hmv_time"] = {
        "threads": threads, "reps": len(t_all), "mean_ms": 1e3 * float(np.mean(t_all)),
        "min_ms": 1e3 * float(np.min(t_all)), "GBs": rec["footprint"] / float(np.mean(t_all)) / 1e9,
        "one_thread_reps": len(t_one), "one_thread_mean_ms": 1e3 * float(np.mean(t_one)),
        "one_thread_GBs": rec["footprint"] / float(np.mean(t_one)) / 1e9}
    print(args.case, "hmv", rec["hmv_time"], flush=True)

    if eps is not None:
        B = A.clone() if one_thread_compress else None
        t0 = time.time()
        rep = A.compress(eps)
        wall = time.time() - t0
        rec["compress"] = {k: rep[k] for k in ("new_ranks", "old_ranks", "frobenius_error", "frobenius_norm",
                                               "bytes_before", "bytes_after", "total_flops", "total_ms",
                                               "time_orthogonalize_ms", "time_project_orth_ms",
                                               "time_weights_ms", "time_truncate_ms", "time_project_trunc_ms",
                                               "flops_orthogonalize", "flops_project_orth", "flops_weights",
                                               "flops_truncate", "flops_project_trunc")}
        rec["compress"]["wall_s"] = wall
        rec["compress"]["model_GFLOPs"] = rep["total_flops"] / wall / 1e9
        yc = A.hmv(x)
        arrays["yc"] = yc[idx]
        rec["yc_norm2"] = float(np.linalg.norm(yc))
        print(args.case, "compress", rec["compress"]["new_ranks"], rep["frobenius_error"], wall, "s", flush=True)
        if B is not None:
            R.set_threads(1)
            t0 = time.time()
            B.compress(eps)
            rec["compress"]["one_thread_wall_s"] = time.time() - t0
            R.set_threads(threads)
            del B
    os.makedirs(args.out, exist_ok=True)
    np.savez_compressed(os.path.join(args.out, args.case + ".npz"), **arrays)
    with open(os.path.join(args.out, args.case + ".json"), "w") as f:
        json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
