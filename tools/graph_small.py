"""Small matrices: direct mat-vec calls vs a replayed CUDA graph of the same
call (h2b_hmv_graph_*), device time per mat-vec over 200 back-to-back steps.
    python tools/graph_small.py"""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_1902_01829_b200 as h2


def per_step(fn, steps=200):
    st = torch.cuda.current_stream()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for dim, n, order in [(2, 1 << 12, 8), (2, 1 << 14, 4), (2, 1 << 16, 8), (3, 1 << 16, 4)]:
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    direct = per_step(lambda: h2.hmv(A, x, y))
    g = h2.HmvGraph(A, x, y)
    graph = per_step(lambda: g.launch())
    print(json.dumps({"dim": dim, "n": n, "grid_order": order, "footprint_bytes": A.memory_footprint(),
                      "direct_us": round(1e3 * direct, 2), "graph_us": round(1e3 * graph, 2)}), flush=True)
    g.close()
    A.close()
