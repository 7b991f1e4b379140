"""C4 single-vector mat-vec: per-phase device times (3 repetitions)."""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
A = h2.H2Matrix.construct(2, 1 << 22, grid_order=8)
x = torch.rand(1 << 22, dtype=torch.float64, device='cuda')
y = torch.zeros_like(x)
for _ in range(3):
    h2.hmv(A, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record()
    for _ in range(10):
        h2.hmv(A, x, y)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"ms_per_hmv": round(e0.elapsed_time(e1) / 10, 4)}), flush=True)
