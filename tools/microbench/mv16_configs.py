"""Device ms per 16-vector pass (10 passes after 3 warm-ups, device pointers)
for C2, C3 and C3 compressed at 1e-6 -- same-box A/B of kernel variants."""
import ctypes as C
import json
import sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib
lib = _lib.load()
def t(A, n, steps=10):
    X = torch.rand(16, n, dtype=torch.float64, device='cuda'); Y = torch.zeros_like(X)
    s = torch.cuda.current_stream()
    def run():
        _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n, 1.0, 0.0,
                                     _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream or 1)))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        run()
    e1.record(s); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / steps, 4)
out = {}
A = h2.H2Matrix.construct(2, 1 << 20, grid_order=6); out["C2"] = t(A, 1 << 20); A.close()
A = h2.H2Matrix.construct(3, 1 << 20, grid_order=4); out["C3"] = t(A, 1 << 20)
h2.compress(A, 1e-6); out["C3c"] = t(A, 1 << 20); A.close()
print(json.dumps(out), flush=True)
