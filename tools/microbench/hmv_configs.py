"""Device ms per single-vector mat-vec (20 calls after 3 warm-ups) for C2, C3
and C3 compressed at 1e-6 -- for same-box A/B comparisons of kernel variants."""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
def t(A, n, steps=20):
    x = torch.rand(n, dtype=torch.float64, device='cuda'); y = torch.zeros_like(x)
    for _ in range(3):
        h2.hmv(A, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h2.hmv(A, x, y)
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / steps, 4)
out = {}
A = h2.H2Matrix.construct(2, 1 << 20, grid_order=6); out["C2"] = t(A, 1 << 20); A.close()
A = h2.H2Matrix.construct(3, 1 << 20, grid_order=4); out["C3"] = t(A, 1 << 20)
h2.compress(A, 1e-6); out["C3c"] = t(A, 1 << 20); A.close()
print(json.dumps(out), flush=True)
