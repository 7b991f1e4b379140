"""compress() of a given config (fresh matrix each rep), phase times; for ncu
launch lists use reps=1.
    python tools/compress_profile.py DIM N ORDER EPS [REPS]"""
import json
import sys

sys.path.insert(0, ".")
import paper_1902_01829_b200 as h2

dim, n, order, eps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
settle = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
for _ in range(reps):
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    if settle:
        import time
        import torch
        torch.cuda.synchronize()
        time.sleep(settle)
    rep = h2.compress(A, eps)
    ph = [rep.time_orthogonalize_ms, rep.time_project_orth_ms, rep.time_weights_ms,
          rep.time_truncate_ms, rep.time_project_trunc_ms]
    print(json.dumps(dict(cfg=f"{dim}d n={n} order={order} eps={eps}", ranks=rep.new_ranks,
                          ms=round(rep.total_ms(), 1), phases=[round(p, 1) for p in ph],
                          tflops_model=round(rep.total_flops() / rep.total_ms() / 1e9, 2))), flush=True)
    A.close()
    del A
