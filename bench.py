#!/usr/bin/env python
"""Benchmark of the B200 H^2 mat-vec hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one single-vector H^2 mat-vec y = A x (hmv.hpp:175-188) over the
n = 2^22 2D exponential-covariance matrix (leaf 64, Chebyshev order 8 -> rank
64, eta 2, ell 0.1, perturbation 0.25, seed 1; BASELINE.json configs[3], the
"n=2^22" the metric is quoted at), built directly in HBM (76.98 GB, > L2).

value  = reference bytes (memory_footprint(A).total(), h2kit.cpp:131-132) / device
         time per step, whole job (sum over ranks of bytes / max-over-ranks time).
e2e    = the same metric through the public API with pinned HOST x/y: each step
         copies x H2D and y D2H inside h2b_hmv (counted in the timed region),
         one synchronous call at a time; e2e.pipelined: two calls in flight
         (H2B_PTR_HOST_ASYNC, one HmvContext and stream each) so one step's
         PCIe copies overlap another's kernels.
roofline = the dominant kernel (k_bsr: coupling + dense blocks) from per-phase
         CUDA events recorded on the launching stream during the timed region.
cpu_baseline = the unmodified reference (oracle/_ref, OpenMP pinned
         close/cores, all host threads) on the SAME workload: its own
         construct() of the n=2^22 matrix (~32 s, 77 GB host RAM) and >= 5
         hmv steps with one HmvContext (the CLI matvec loop, h2kit.cpp:104-141),
         in a child process so its OpenMP pinning and memory stay out of ours.
--impl reference = the same, K timed steps after W warm-ups, plus one
         1-thread step; same config, metric and unit as our arm.

N > 1 (torchrun): the same n=2^22 matrix is partitioned by top-level subtrees
across the ranks (1/N of the matrix per GPU) and one mat-vec exchanges x^ and
the y slices with NCCL all-gathers; scaling "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H2 mat-vec GB/s (% of HBM peak) & ms at n=2^22; compression GFLOP/s"
WORKLOAD = dict(workload="H2 single-vector mat-vec, 2D exponential covariance", dim=2,
                n=1 << 22, leaf_size=64, grid_order=8, rank=64, eta=2.0, ell=0.1,
                perturbation=0.25, seed=1)
CONFIG_GOLDEN = os.path.join(ROOT, "tests", "golden", "config")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_pipes():
    """FP64 / DMMA pipe utilisation of the compression and 16-vector kernels
    from the committed ncu captures (profiles/tensor_pipe.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "tensor_pipe.json")) as f:
            return json.load(f)
    except Exception:
        return None


def load_traffic():
    """dram bytes per k_bsr launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("workload_n") == WORKLOAD["n"]:
            return float(d["k_bsr_dram_bytes"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


_JSON_OUT = None  # the bench line's stream once stdout is handed to the libraries


def emit(line: dict):
    """Print THE bench line: on the saved stdout when dist_setup redirected
    file descriptor 1 (NCCL and the CUDA libraries write banners such as
    "NCCL version ..." to fd 1, which must not precede the JSON line)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def dist_setup(force: bool = False):
    global _JSON_OUT
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or force:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)  # library output on fd 1 goes to stderr
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def host_cpu_info():
    """CPU model / family / cores / RAM of this host (the CPU baseline's machine)."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                k, _, v = ln.partition(":")
                k = k.strip()
                if k in ("model name", "cpu family", "model", "stepping") and k not in info:
                    info[k] = v.strip()
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    info["mem_total_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return info


def pin_openmp():
    """OMP_PROC_BIND=close OMP_PLACES=cores (unpinned reference runs
    vary 10-100x); must be set before libgomp is loaded."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")


def cpu_reference_sample(cfg, steps: int = 5, warmup: int = 1, one_thread: bool = False):
    """The unmodified reference on the full workload: construct() of the same
    matrix, then `steps` timed hmv calls with one HmvContext (ref_hmv_reps:
    the CLI matvec loop) after `warmup`, all host threads, OpenMP pinned."""
    import numpy as np

    import oracle
    kind = "reference" if oracle.reference_available() else "port"
    be = oracle.best()
    cores = os.cpu_count() or 1
    be.set_threads(cores)
    n = cfg["n"]
    t0 = time.time()
    A = be.construct(cfg["dim"], n, leaf_size=cfg["leaf_size"], grid_order=cfg["grid_order"], eta=cfg["eta"],
                     ell=cfg["ell"], perturbation=cfg["perturbation"], seed=cfg["seed"])
    build_s = time.time() - t0
    x = be.random_vector(n, 1)
    y = np.zeros_like(x)
    fp = A.footprint()

    def step():
        if kind == "reference":
            be.check(be.lib.ref_hmv_reps(A.h, x.ctypes.data, y.ctypes.data, 1))
        else:
            A.hmv(x)

    for _ in range(max(0, warmup)):
        step()
    times = []
    for _ in range(max(1, steps)):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
    mean = sum(times) / len(times)
    out = {"value": fp / mean / 1e9, "unit": "GB/s", "cores": be.max_threads(), "kind": kind,
           "ms_per_step": mean * 1e3, "ms_min": min(times) * 1e3, "reps": len(times),
           "footprint_bytes": fp, "construct_s": round(build_s, 1), "host": host_cpu_info(),
           "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")},
           "sample": f"the full workload: reference construct() of the 2D n=2^{n.bit_length() - 1} k=64 matrix "
                     f"({fp / 1e9:.2f} GB) + {len(times)} timed hmv steps (one HmvContext) after {warmup} "
                     f"warm-up, OpenMP {be.max_threads()} threads pinned close/cores"}
    if one_thread and kind == "reference":
        be.set_threads(1)
        t = time.perf_counter()
        step()
        dt = time.perf_counter() - t
        be.set_threads(cores)
        out["one_thread"] = {"ms_per_step": round(dt * 1e3, 1), "value": round(fp / dt / 1e9, 3), "reps": 1}
    return out


def cpu_baseline_subprocess(cfg, timeout_s: float = 900.0):
    """cpu_reference_sample in a child process (its OpenMP pinning and the
    77 GB host matrix stay out of the GPU process)."""
    env = dict(os.environ)
    env.setdefault("OMP_PROC_BIND", "close")
    env.setdefault("OMP_PLACES", "cores")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-json", "--n", str(cfg["n"])],
                       capture_output=True, text=True, timeout=timeout_s, env=env)
    if r.returncode != 0:
        raise RuntimeError((r.stderr or r.stdout).strip().splitlines()[-1] if (r.stderr or r.stdout) else "failed")
    return json.loads(r.stdout.strip().splitlines()[-1])


def recorded_reference_compress():
    """The reference's compress() of C3 on this pool's GPU host (16 threads,
    pinned), recorded by tests/golden/make_config_golden.py (136.98 s; the
    parity goldens come from the same run)."""
    try:
        with open(os.path.join(CONFIG_GOLDEN, "C3.json")) as f:
            d = json.load(f)
        c = d["compress"]
        return {"wall_ms": round(1e3 * c["wall_s"], 0), "model_flops": c["total_flops"],
                "model_gflops": round(c["model_GFLOPs"], 2), "threads": d["threads"], "kind": "reference",
                "host": d["host"], "source": "tests/golden/config/C3.json (recorded by "
                "tests/golden/make_config_golden.py on the GPU host; not re-run by bench.py)"}
    except Exception:  # noqa: BLE001
        return None


FP64_PEAK_TFLOPS = 37.1  # DMMA m8n8k4 measured on this pool's B200 (tools/fp64_peak.cu: 37.07); DFMA 36.4
READ_STREAM_PEAK_GBS = 7440.0  # recorded: tools/microbench/tma_stream.cu on the pool's B200
COMPRESS_CFG = dict(dim=3, n=1 << 20, grid_order=4, eps=1e-6)


def compression_run(h2, torch, device, reps):
    """compress() of the C3 matrix (3D exponential covariance n=2^20, rank 64,
    eps 1e-6): model GFLOP/s = reference analytic flops (flops.hpp) / device time."""
    warm = h2.H2Matrix.construct(2, 1 << 14, device=device)
    h2.compress(warm, 1e-7)
    warm.close()
    times, dev, rep = [], [], None
    for _ in range(max(1, reps)):
        A = h2.H2Matrix.construct(COMPRESS_CFG["dim"], COMPRESS_CFG["n"],
                                  grid_order=COMPRESS_CFG["grid_order"], device=device)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = h2.compress(A, COMPRESS_CFG["eps"])
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        dev.append(r.total_ms())
        if rep is None or r.total_ms() <= rep.total_ms():
            rep = r
        A.close()
    dev_ms = rep.total_ms()  # best rep: the first one also pays the memory pool's growth
    gflops = rep.total_flops() / (dev_ms * 1e-3) / 1e9
    return {"config": "3D exponential covariance n=2^20, leaf 64, order 4 (rank 64), eps 1e-6 (C3)",
            "ms": round(dev_ms, 1), "ms_all_reps": [round(v, 1) for v in dev],
            "wall_ms": round(min(times), 1), "reps": len(times),
            "model_flops": rep.total_flops(), "gflops": round(gflops, 1),
            "pct_fp64_peak": round(100 * gflops / 1e3 / FP64_PEAK_TFLOPS, 2),
            "fp64_peak_tflops": FP64_PEAK_TFLOPS,
            "phase_ms": {"orthogonalize": round(rep.time_orthogonalize_ms, 1),
                         "project_orth": round(rep.time_project_orth_ms, 1),
                         "weights": round(rep.time_weights_ms, 1),
                         "truncate": round(rep.time_truncate_ms, 1),
                         "project_trunc": round(rep.time_project_trunc_ms, 1)},
            "new_ranks": rep.new_ranks, "frobenius_error": rep.frobenius_error,
            "bytes": [rep.bytes_before, rep.bytes_after],
            "executed": executed_compress(dev_ms),
            "pipe_utilisation_ncu_recorded": (load_pipes() or {}).get("compression_C3")}


def executed_compress(dev_ms):
    """Executed FP64 flops of one C3 compress (ncu SASS counters: 2 DFMA + DADD
    + DMUL + 512 DMMA.8x8x4, tools/compress_exec_flops.py), RECORDED in
    profiles/r02_compress_exec_flops_c3.json -- not measured by this run -- over
    this run's device time.  The kernels execute ~79% of the reference model's
    flops: unpadded weight stacks, upper blocks of symmetric levels, skipped
    triangular fragments, ~6 Jacobi sweeps (but also the dead-lane FMAs)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_compress_exec_flops_c3.json")) as f:
            ex = json.load(f)["executed_flops"]
    except Exception:
        return None
    g = ex / (dev_ms * 1e-3) / 1e9
    return {"flops": ex, "gflops": round(g, 1), "pct_fp64_peak": round(100 * g / 1e3 / FP64_PEAK_TFLOPS, 2),
            "source": "profiles/r02_compress_exec_flops_c3.json (ncu, recorded)"}


def compression_run_dist(torch, device, reps, world):
    """Subtree-partitioned compress() of C3 across the ranks (h2b_part_compress,
    NCCL all-gathers of the projection trees): device time = max over ranks of
    the per-rank phase times (collective waits included)."""
    import paper_1902_01829_b200 as h2
    from paper_1902_01829_b200.dist import DistributedH2Matrix
    warm = DistributedH2Matrix(2, 1 << 14, device=device)
    warm.compress(1e-7)
    warm.close()
    best, rep = None, None
    for _ in range(max(1, reps)):
        D = DistributedH2Matrix(COMPRESS_CFG["dim"], COMPRESS_CFG["n"], grid_order=COMPRESS_CFG["grid_order"],
                                device=device)
        torch.cuda.synchronize()
        barrier(world)
        rep = D.compress(COMPRESS_CFG["eps"])
        ms = max_over_ranks(rep.total_ms(), world)
        best = ms if best is None else min(best, ms)
        D.close()
    h2.release_cached_memory(device)
    gflops = rep.total_flops() / (best * 1e-3) / 1e9
    return {"config": "3D exponential covariance n=2^20, leaf 64, order 4 (rank 64), eps 1e-6 (C3), "
                      f"subtree-partitioned over {world} GPUs",
            "ms": round(best, 1), "reps": reps, "model_flops": rep.total_flops(), "gflops": round(gflops, 1),
            "pct_fp64_peak_per_gpu": round(100 * gflops / 1e3 / FP64_PEAK_TFLOPS / world, 2),
            "fp64_peak_tflops": FP64_PEAK_TFLOPS, "new_ranks": rep.new_ranks,
            "frobenius_error": rep.frobenius_error, "bytes": [rep.bytes_before, rep.bytes_after]}


def multi16_run(A, torch, steps):
    """16 right-hand sides per pass through h2b_hmv_multi (device pointers):
    every block is read once per 16 vectors and multiplied on the FP64 tensor
    cores (mma.sync m8n8k4, k_hmv_mv.cu)."""
    import ctypes as C

    from paper_1902_01829_b200 import _lib
    n = A.info().n
    fp = A.memory_footprint()
    flops = A.info().hmv_flops
    X = torch.rand(16, n, dtype=torch.float64, device="cuda")
    Y = torch.zeros_like(X)
    s = torch.cuda.current_stream()
    lib = _lib.load()

    def run():
        _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()),
                                     n, 1.0, 0.0, _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream or 1)))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        run()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"vectors": 16, "ms_per_pass": round(ms, 3), "ms_per_vector": round(ms / 16, 4),
            "effective_GBs": round(16 * fp / ms / 1e6, 1),
            "matrix_stream_GBs": round(fp / ms / 1e6, 1),
            "model_tflops": round(16 * flops / ms / 1e9, 2),
            "pct_fp64_peak": round(100 * 16 * flops / ms / 1e9 / FP64_PEAK_TFLOPS, 2),
            "byte_bound": mv16_byte_bound(A, n, fp, ms),
            "pipe_utilisation_ncu_recorded": (load_pipes() or {}).get("multi16_C4")}


def mv16_byte_bound(A, n, fp, ms):
    """Compulsory HBM bytes of one 16-vector pass: every matrix entry once, the
    (symmetric) basis a second time in the downsweep, the 16-column panels of
    x (read), y (written), xc / yc (written + read) and x^ / y^ (written +
    read), over the measured copy peak."""
    inf = A.info()
    k = list(inf.ranks[:inf.depth + 1])
    basis = 8 * (n * k[-1] + sum((1 << l) * k[l] * k[l - 1] for l in range(1, len(k))))
    vec = sum((1 << l) * k[l] for l in range(len(k)))
    byts = fp + basis + 128 * n * 6 + 128 * vec * 4
    peak, _ = load_peaks()
    bound = byts / (peak * 1e6)
    return {"bytes": byts, "ms": round(bound, 3), "frac": round(bound / ms, 3), "peak_GBs": peak}


def run_reference(args):
    """--impl reference: the unmodified reference (oracle/_ref) on the host
    cores, same workload / metric / unit as our arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pin_openmp()
    cfg = dict(WORKLOAD, n=args.n)
    cb = cpu_reference_sample(cfg, steps=max(1, args.steps), warmup=args.warmup, one_thread=True)
    line = {"metric": METRIC, "value": round(cb["value"], 3), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(cb["ms_per_step"], 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": dict(cfg, parallelism=f"OpenMP {cb['cores']} threads (host)", same_config=True,
                           construct_s=cb["construct_s"]),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "host": cb["host"], "omp": cb["omp"], "one_thread": cb.get("one_thread"),
            "e2e": {"value": round(cb["value"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "compression_recorded": recorded_reference_compress()}
    emit(line)


def run_distributed(args, cfg, world, rank, local):
    """N > 1: subtree-partitioned mat-vec of the SAME n=2^22 matrix (strong
    scaling): every rank holds 1/N of the matrix (its top-level subtree plus
    the replicated levels above the split) and exchanges x^ / y slices with
    NCCL all-gathers (paper_1902_01829_b200/dist.py)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1902_01829_b200 import _lib
    from paper_1902_01829_b200.dist import DistributedH2Matrix
    import ctypes as C

    t0 = time.time()
    D = DistributedH2Matrix(cfg["dim"], cfg["n"], leaf_size=cfg["leaf_size"],
                            grid_order=cfg["grid_order"], eta=cfg["eta"], ell=cfg["ell"],
                            perturbation=cfg["perturbation"], seed=cfg["seed"], device=local)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    n = D.n
    fp = D.footprint_global
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    gen = torch.Generator(device="cuda").manual_seed(1)  # same x on every rank
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        D.hmv(x, y)
    torch.cuda.synchronize()
    lib = _lib.load()
    _lib.check(lib.h2b_set_phase_timing(D._h, 1))
    buf = (C.c_double * 4)()
    lib.h2b_last_hmv_timing(D._h, buf)
    sampler = ClockSampler(local) if rank == 0 else None
    barrier(world)
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        D.hmv(x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop() if sampler else None
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    _lib.check(lib.h2b_last_hmv_timing(D._h, buf))
    phases = list(buf)
    _lib.check(lib.h2b_set_phase_timing(D._h, 0))
    value = fp / (ms * 1e-3) / 1e9

    # e2e: pinned host x -> device, mat-vec, full y -> pinned host, every rank
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    xd = torch.empty_like(x)

    def e2e_step():
        xd.copy_(xh, non_blocking=True)
        D.hmv(xd, y)
        yh.copy_(y, non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    # parity spot check against the replicated-input result
    assert torch.allclose(yh, y.cpu(), rtol=0, atol=0)
    # 16-vector pass on the partitions (h2b_part_hmv_multi, BASELINE configs[3])
    X = torch.rand(16, n, dtype=torch.float64, device="cuda", generator=gen)
    Y = torch.zeros_like(X)
    for _ in range(2):
        D.hmv_multi(X, Y)
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        D.hmv_multi(X, Y)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    mv_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    multi = {"vectors": 16, "ms_per_pass": round(mv_ms, 3), "ms_per_vector": round(mv_ms / 16, 4),
             "effective_GBs": round(16 * fp / mv_ms / 1e6, 1)}
    del X, Y
    inf = D.info
    D.close()
    comp = None
    if not args.no_compress:
        comp = compression_run_dist(torch, local, args.compress_reps, world)
    if rank != 0:
        dist.destroy_process_group()
        return
    peak, peak_src = load_peaks()
    q = inf.depth
    bsr_bytes = 8 * (sum(inf.cpl_blocks[l] * inf.ranks[l] ** 2 for l in range(q + 1))
                     + inf.dense_blocks * inf.m * inf.m)
    achieved = bsr_bytes / (phases[1] * 1e-3) / 1e9 if phases[1] > 0 else None
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(cfg, parallelism=f"subtree{world}", footprint_bytes=fp,
                       footprint_per_gpu=D.footprint_local,
                       l2="inputs larger than L2", build_s=round(build_s, 2)),
        "pct_of_hbm_peak": round(100.0 * value / world / peak, 2),
        "phase_ms_rank0": {"top_upsweep": round(phases[0], 4), "coupling_dense_bsr": round(phases[1], 4),
                           "downsweep": round(phases[2], 4)},
        "roofline": {"bound": "hbm", "kernel": "k_bsr (rank 0 partition)",
                     "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None, "traffic": None,
                     "algorithmic_bytes_per_launch": bsr_bytes},
        "cpu_baseline": None,
        "e2e": {"value": round(fp / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": 8 * n * world,
                "d2h_bytes_per_step": 8 * n * world},
        # ours per step: up_leaf, gather, per-level up (q), bsr, per-level down (q), down_leaf
        "gpu_launches": (2 * q + 4) * args.steps,
        "clocks": clocks,
        "multi16": multi,
        "compression": comp,
    }
    emit(line)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=WORKLOAD["n"], help="override n (testing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compress", action="store_true")
    ap.add_argument("--compress-reps", type=int, default=3)
    ap.add_argument("--dist", action="store_true",
                    help="use the subtree-partitioned path even at N=1 (testing)")
    ap.add_argument("--cpu-baseline-json", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_baseline_json:  # child process of cpu_baseline_subprocess
        pin_openmp()
        print(json.dumps(cpu_reference_sample(dict(WORKLOAD, n=args.n))))
        return
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(3, args.warmup)

    import numpy as np
    import torch

    import paper_1902_01829_b200 as h2

    world, rank, local = dist_setup(force=args.dist)
    torch.cuda.set_device(local)
    cfg = dict(WORKLOAD, n=args.n)
    if world > 1 or args.dist:
        return run_distributed(args, cfg, world, rank, local)
    t0 = time.time()
    A = h2.H2Matrix.construct(cfg["dim"], cfg["n"], leaf_size=cfg["leaf_size"],
                              grid_order=cfg["grid_order"], eta=cfg["eta"], ell=cfg["ell"],
                              perturbation=cfg["perturbation"], seed=cfg["seed"], device=local)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    info = A.info()
    fp = info.footprint_bytes
    n = info.n
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    xt = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen)
    yt = torch.zeros(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.Stream()  # explicit stream: NULL would mean the matrix's own stream
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    # our kernels per step: k_up_leaf, k_up_fused (levels q..1), k_bsr,
    # k_down_fused (levels 1..q), k_down_leaf (plus two 16-byte ticket memsets)
    launches = 5 if info.depth >= 1 else 3
    r = info.ranks

    for _ in range(args.warmup):
        h2.hmv(A, xt, yt, stream=sp)
    torch.cuda.synchronize()

    # ---- device-resident timed region --------------------------------
    A.set_phase_timing(True)
    A.last_hmv_timing()  # reset
    sampler = ClockSampler(local) if rank == 0 else None
    barrier(world)
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        h2.hmv(A, xt, yt, stream=sp)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop() if sampler else None
    ms_local = ev0.elapsed_time(ev1) / args.steps
    phases = A.last_hmv_timing()
    A.set_phase_timing(False)
    ms = max_over_ranks(ms_local, world)
    value = world * fp / (ms * 1e-3) / 1e9

    # ---- end-to-end through the public API with pinned host buffers ----
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh.copy_(xt.cpu())
    xn, yn = xh.numpy(), yh.numpy()
    for _ in range(2):
        h2.hmv(A, xn, yn, stream=sp)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        h2.hmv(A, xn, yn, stream=sp)  # synchronous: H2D x, mat-vec, D2H y, host sync
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_sync_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    # correctness spot check of the e2e result against the device result
    assert np.allclose(yn, yt.cpu().numpy(), rtol=1e-13, atol=0)
    # Pipelined: two calls in flight (one HmvContext, stream and pinned y each,
    # H2B_PTR_HOST_ASYNC), so one call's PCIe copies overlap the other's
    # kernels; every step still copies its x in and its y out.
    ctxs = [h2.HmvContext(A) for _ in range(2)]
    sts = [torch.cuda.Stream() for _ in range(2)]
    yhs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    yns = [t.numpy() for t in yhs]

    def pipelined(steps):
        for st in sts:
            st.wait_stream(stream)
        for i in range(steps):
            k = i & 1
            h2.hmv(A, xn, yns[k], stream=sts[k].cuda_stream, ctx=ctxs[k], asynchronous=True)
        for st in sts:
            stream.wait_stream(st)

    pipelined(2)
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    pipelined(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    e2e_value = world * fp / (e2e_ms * 1e-3) / 1e9
    for yk in yns:
        assert np.allclose(yk, yt.cpu().numpy(), rtol=1e-13, atol=0)
    for c in ctxs:
        c.close()

    # ---- 16-vector FP64-MMA mat-vec on the same matrix (BASELINE configs[3]) ----
    multi = multi16_run(A, torch, args.steps)
    # ---- accuracy of the device-built matrix: exact-kernel sampled validation
    #      (validate.hpp:26-62; acceptance c1 bound 1e-7 in 2D) ----
    t0 = time.time()
    acc = {"sampled_rel_err": h2.validate_sampled(A, 1e-3, 1), "fraction": 1e-3,
           "bound_2d": 1e-7}
    acc["seconds"] = round(time.time() - t0, 2)

    # ---- compression GFLOP/s (metric's second half): C3, 3D n=2^20 k=64, eps 1e-6 ----
    A.close()
    del A
    torch.cuda.synchronize()
    comp = None
    if not args.no_compress:
        comp = compression_run(h2, torch, local, args.compress_reps)
    h2.release_cached_memory(local)

    if rank != 0:
        return
    peak, peak_src = load_peaks()
    bsr_bytes = 8 * (sum(info.cpl_blocks[l] * r[l] * r[l] for l in range(info.depth + 1))
                     + info.dense_blocks * info.m * info.m)
    bsr_ms = phases[1]
    achieved = bsr_bytes / (bsr_ms * 1e-3) / 1e9 if bsr_ms > 0 else None
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cb = cpu_baseline_subprocess(cfg)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu.update(ms_per_step=round(cb["ms_per_step"], 1), host=cb["host"], omp=cb["omp"],
                       same_config=True)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if comp is not None:
        comp["cpu_baseline"] = recorded_reference_compress()
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": dict(cfg, parallelism=f"replicas{world}" if world > 1 else "single",
                       footprint_bytes=fp, l2="inputs larger than L2 (76.98 GB matrix per step)",
                       build_s=round(build_s, 2)),
        "pct_of_hbm_peak": round(100.0 * value / world / peak, 2),
        "phase_ms": {"upsweep": round(phases[0], 4), "coupling_dense_bsr": round(phases[1], 4),
                     "downsweep_scatter": round(phases[2], 4)},
        "roofline": {"bound": "hbm", "kernel": "k_bsr_tma (coupling + dense blocks, TMA-streamed)",
                     "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": load_traffic(), "algorithmic_bytes_per_launch": bsr_bytes,
                     # a read-only stream outruns the read+write copy peak: the same kernel
                     # against the read-stream ceiling measured on this pool's B200s
                     "read_stream_peak_recorded": {
                         "GBs": READ_STREAM_PEAK_GBS,
                         "frac": round(achieved / READ_STREAM_PEAK_GBS, 4) if achieved else None,
                         "source": "tools/microbench/tma_stream.cu: 64 GB f64 stream through a TMA box ring "
                                   "(2 stages x 2 CTAs/SM); 16-byte evict-first loads reach 7.06-7.09 TB/s"}},
        "cpu_baseline": cpu,
        "e2e": {"value": round(world * fp / (e2e_sync_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_sync_ms, 4), "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "mode": "one synchronous h2b_hmv call per step (pinned host x in, y out)",
                "pipelined": {"value": round(e2e_value, 2), "ms_per_step": round(e2e_ms, 4),
                              "mode": "two calls in flight (H2B_PTR_HOST_ASYNC, one HmvContext + stream "
                                      "each): one step's PCIe copies overlap another's kernels"}},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
        "multi16": multi,
        "accuracy": acc,
        "compression": comp,
    }
    emit(line)


if __name__ == "__main__":
    main()
