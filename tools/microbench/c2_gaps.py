"""C2 (2D n=2^20, k=36) single-vector mat-vec: per-call host time and device
time back to back, and the kernel timeline of two calls."""
import sys, time
sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1902_01829_b200 as h2
A = h2.H2Matrix.construct(2, 1 << 20, grid_order=6)
x = torch.rand(1 << 20, dtype=torch.float64, device='cuda')
y = torch.zeros_like(x)
for _ in range(3):
    h2.hmv(A, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h0 = time.perf_counter()
for _ in range(20):
    h2.hmv(A, x, y)
h1 = time.perf_counter()
e1.record(); torch.cuda.synchronize()
print(f"device {e0.elapsed_time(e1) / 20:.4f} ms per call, host {1e3 * (h1 - h0) / 20:.4f} ms per call", flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        h2.hmv(A, x, y)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"  {(e.time_range.start - t0) / 1e3:8.3f} {e.time_range.elapsed_us() / 1e3:7.3f}  {e.name.split('(')[0][-30:]}")
