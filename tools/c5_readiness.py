"""C5 readiness on ONE B200 (SURVEY.md §8 C5 / §8(e) weak-scaling ladder).

  python tools/c5_readiness.py rung1   # 3D n=2^21 k=64 whole matrix (98.2 GB): hmv, compress, validate
  python tools/c5_readiness.py part0   # 3D n=2^24 k=64, partition 0 of 8 (~106 GB): local hmv + compress

part0 runs the rank-0 share of the 8-GPU C5 job with stubbed collectives
(the x^ all-gather is skipped, the projection-tree all-gathers replicate the
local slice, the rank / energy all-reduces are identities): the per-GPU
device time and memory of C5, not a parity run.  Prints one JSON line.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1902_01829_b200 as h2  # noqa: E402
from paper_1902_01829_b200 import _lib  # noqa: E402
from paper_1902_01829_b200.dist import Communicator, DistributedH2Matrix  # noqa: E402

FP64_PEAK = 37.1


def events_ms(fn, steps, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def rung1(steps=10):
    t0 = time.time()
    A = h2.H2Matrix.construct(3, 1 << 21)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    inf = A.info()
    n = inf.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    s = torch.cuda.current_stream()
    for _ in range(3):
        h2.hmv(A, x, y)
    ms = events_ms(lambda: h2.hmv(A, x, y), steps, s)
    free, total = torch.cuda.mem_get_info()
    t0 = time.time()
    err = h2.validate_sampled(A, 1e-4, 1)
    val_s = time.time() - t0
    rep = h2.compress(A, 1e-6)
    for _ in range(3):  # the first calls after compress() re-size the workspace
        h2.hmv(A, x, y)
    ms2 = events_ms(lambda: h2.hmv(A, x, y), steps, s)
    out = {"case": "3D n=2^21 k=64 (C5 ladder rung, 1 GPU)", "build_s": round(build_s, 1),
           "footprint_bytes": inf.footprint_bytes, "device_bytes": inf.device_bytes,
           "hbm_used_gb": round((total - free) / 1e9, 1),
           "hmv_ms": round(ms, 3), "hmv_GBs": round(inf.footprint_bytes / ms / 1e6, 1),
           "validate_sampled": {"fraction": 1e-4, "rel_err": err, "seconds": round(val_s, 2)},
           "compress": {"eps": 1e-6, "ms": round(rep.total_ms(), 1), "model_flops": rep.total_flops(),
                        "pct_fp64_peak": round(100 * rep.total_flops() / rep.total_ms() / 1e9 / FP64_PEAK, 2),
                        "new_ranks": rep.new_ranks, "frobenius_error": rep.frobenius_error,
                        "bytes": [rep.bytes_before, rep.bytes_after]},
           "hmv_after_compress_ms": round(ms2, 3)}
    A.close()
    h2.release_cached_memory(0)
    return out


class StubComm(Communicator):
    """Rank 0 of 8 without peers: all-gathers replicate the local slice (finite
    stand-ins for the remote projection trees), all-reduces are identities."""

    def allgather(self, buf):
        chunk = buf.numel() // self.nparts
        mine = buf[self.part * chunk:(self.part + 1) * chunk].clone()
        for g in range(self.nparts):
            if g != self.part:
                buf[g * chunk:(g + 1) * chunk].copy_(mine)
        torch.cuda.synchronize()

    def allreduce_max(self, t):
        pass

    def allreduce_sum(self, t):
        pass


def part0(steps=10):
    t0 = time.time()
    D = DistributedH2Matrix(3, 1 << 24, nparts=8, part=0, device=0)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    n = D.n
    free, total = torch.cuda.mem_get_info()
    fp_local, fp_global = D.footprint_local, D.footprint_global  # before compress() shrinks them
    lib = _lib.load()
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    st = C.c_void_p(s.cuda_stream or 1)

    def local_hmv():  # x^ / y all-gathers stubbed out (rank-local device work only)
        _lib.check(lib.h2b_part_upsweep(D._h, C.c_void_p(x.data_ptr()), st))
        _lib.check(lib.h2b_part_finish(D._h, C.c_void_p(D.y_slice.data_ptr()), st))

    for _ in range(3):
        local_hmv()
    _lib.check(lib.h2b_set_phase_timing(D._h, 1))
    buf = (C.c_double * 4)()
    lib.h2b_last_hmv_timing(D._h, buf)
    ms = events_ms(local_hmv, steps, s)
    _lib.check(lib.h2b_last_hmv_timing(D._h, buf))
    _lib.check(lib.h2b_set_phase_timing(D._h, 0))
    gather = sum((1 << l) * k for l, k in enumerate(D.ranks) if l >= 3) * 8  # x^ bytes all-gathered per GPU
    t0 = time.time()
    rep = D.compress(1e-6, comm=StubComm(8, 0, 0))
    torch.cuda.synchronize()
    comp_wall = time.time() - t0
    out = {"case": "3D n=2^24 k=64 (C5), partition 0 of 8, collectives stubbed",
           "build_s": round(build_s, 1), "footprint_local_bytes": fp_local,
           "footprint_global_bytes": fp_global, "hbm_used_gb": round((total - free) / 1e9, 1),
           "local_hmv_ms": round(ms, 3), "local_hmv_GBs": round(fp_local / ms / 1e6, 1),
           "phase_ms_after_upsweep": [round(v, 4) for v in list(buf)[:3]],
           "xhat_allgather_bytes_per_gpu": gather,
           "compress_local": {"eps": 1e-6, "ms": round(rep.total_ms(), 1), "wall_s": round(comp_wall, 2),
                              "new_ranks_local": rep.new_ranks, "bytes": [rep.bytes_before, rep.bytes_after]}}
    D.close()
    h2.release_cached_memory(0)
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "rung1"
    print(json.dumps(rung1() if which == "rung1" else part0()))
