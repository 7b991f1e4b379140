"""Compression at scale on one B200 vs the reference's recorded results
(ranks, frob estimates, model flops measured on the CPU)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1902_01829_b200 as h2

REF = {  # BASELINE.md §3 / SURVEY.md §8(c)
    "2d_2^14_k64": dict(dim=2, n=1 << 14, order=8, eps=1e-7, ranks=[0, 0, 0, 22, 32, 35, 38, 38, 32], frob=4.66e-8, flops=2.046e10, cpu_s=1.528),
    "2d_2^20_k36": dict(dim=2, n=1 << 20, order=6, eps=1e-7, ranks=[0, 0, 0, 14, 29, 31, 35, 31, 32, 26, 27, 22, 22, 24, 21], frob=1.98e-7, flops=2.813e11, cpu_s=30.2),
    "2d_2^20_k64": dict(dim=2, n=1 << 20, order=8, eps=1e-7, ranks=[0, 0, 0, 14, 32, 35, 38, 31, 32, 26, 27, 23, 22, 25, 21], frob=1.91e-7, flops=1.267e12, cpu_s=104.9),
    "3d_2^18_k64": dict(dim=3, n=1 << 18, order=4, eps=1e-6, ranks=[0, 0, 0, 0, 37, 51, 60, 60, 58, 59, 50, 54, 46], frob=1.60e-6, flops=7.556e11, cpu_s=72.2),
    "3d_2^20_k64": dict(dim=3, n=1 << 20, order=4, eps=1e-6, ranks=None, frob=None, flops=None, cpu_s=None),
}

names = sys.argv[1:] or list(REF)
for name in names:
    r = REF[name]
    t0 = time.time()
    A = h2.H2Matrix.construct(r["dim"], r["n"], grid_order=r["order"])
    torch.cuda.synchronize()
    tb = time.time() - t0
    x = np.random.default_rng(1).random(r["n"])
    y0 = h2.hmv(A, x)
    t0 = time.time()
    rep = h2.compress(A, r["eps"])
    wall = time.time() - t0
    y1 = h2.hmv(A, x)
    ms = rep.total_ms()
    out = dict(name=name, build_s=round(tb, 2), compress_wall_s=round(wall, 3), device_ms=round(ms, 1),
               phases_ms=[round(v, 1) for v in (rep.time_orthogonalize_ms, rep.time_project_orth_ms,
                                                rep.time_weights_ms, rep.time_truncate_ms,
                                                rep.time_project_trunc_ms)],
               model_flops=rep.total_flops(), gflops=round(rep.total_flops() / ms / 1e6, 1),
               ranks=rep.new_ranks, ref_ranks=r["ranks"], frob=rep.frobenius_error, ref_frob=r["frob"],
               ref_flops=r["flops"], ref_cpu_s=r["cpu_s"],
               op_change=float(np.linalg.norm(y1 - y0) / np.linalg.norm(y0)),
               bytes=[rep.bytes_before, rep.bytes_after])
    print(json.dumps(out), flush=True)
    del A
