"""Kernel timeline (CUPTI via torch.profiler) of the 16-vector pass at C4
(2D n=2^22, k=64): every launch of REPS passes with start offset and duration,
to compare in-situ kernel times with the serialised ncu launch list.
    python tools/mv16_timeline.py [REPS]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A = h2.H2Matrix.construct(2, 1 << 22, grid_order=8)
n = A.info().n
X = torch.rand(16, n, dtype=torch.float64, device="cuda")
Y = torch.zeros_like(X)
s = torch.cuda.current_stream()
lib = _lib.load()


def run():
    _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n, 1.0, 0.0,
                                 _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream or 1)))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    run()
e1.record(s)
torch.cuda.synchronize()
print(f"events: {e0.elapsed_time(e1) / 10:.3f} ms per pass", flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    k = e.name.replace("h2b::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:34]
    print(f"  {(e.time_range.start - t0) / 1e3:9.3f} {e.time_range.elapsed_us() / 1e3:8.3f}  {k}", flush=True)
