"""Device time of compress() at C3 (3D n=2^20, k=64, eps 1e-6) over fresh
matrices: best / all reps, phases, ranks.   python tools/compress_time.py [reps]"""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_1902_01829_b200 as h2

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
warm = h2.H2Matrix.construct(2, 1 << 14)
h2.compress(warm, 1e-7)
warm.close()
out = []
for _ in range(reps):
    A = h2.H2Matrix.construct(3, 1 << 20, grid_order=4)
    torch.cuda.synchronize()
    r = h2.compress(A, 1e-6)
    out.append(r)
    A.close()
best = min(out, key=lambda r: r.total_ms())
print(json.dumps({"ms": [round(r.total_ms(), 1) for r in out],
                  "pct_fp64_peak": round(100 * best.total_flops() / best.total_ms() / 1e9 / 37.1, 2),
                  "phases": [round(v, 1) for v in (best.time_orthogonalize_ms, best.time_project_orth_ms,
                                                   best.time_weights_ms, best.time_truncate_ms,
                                                   best.time_project_trunc_ms)],
                  "ranks": best.new_ranks, "frob": best.frobenius_error}))
