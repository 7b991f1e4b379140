"""16-vector pass on a compressed matrix (3D n=2^20 k=64 compressed at 1e-6)."""
import ctypes as C
import json
import sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib
A = h2.H2Matrix.construct(3, 1 << 20, grid_order=4)
n = 1 << 20
X = torch.rand(16, n, dtype=torch.float64, device='cuda')
Y = torch.zeros_like(X)
s = torch.cuda.current_stream()
lib = _lib.load()
def run():
    _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n, 1.0, 0.0,
                                 _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream or 1)))
def t(steps=10):
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        run()
    e1.record(s); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / steps, 4)
before = t()
h2.compress(A, 1e-6)
print(json.dumps({"before_ms": before, "after_ms": t(), "after_ms_2": t()}), flush=True)
