"""Mat-vec of a compressed matrix (3D n=2^20 k=64 compressed at 1e-6, C3),
warmed up, events over 20 calls."""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
A = h2.H2Matrix.construct(3, 1 << 20, grid_order=4)
x = torch.rand(1 << 20, dtype=torch.float64, device='cuda')
y = torch.zeros_like(x)
def t(steps=20):
    for _ in range(3):
        h2.hmv(A, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h2.hmv(A, x, y)
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / steps, 4)
before = t()
h2.compress(A, 1e-6)
print(json.dumps({"before_ms": before, "after_ms": t(), "after_ms_2": t(), "footprint": A.memory_footprint()}), flush=True)
