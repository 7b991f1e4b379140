"""16-vector pass time (CUDA events, 20 passes after 3 warm-ups) at n=2^22."""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib
n = 1 << 22
A = h2.H2Matrix.construct(2, n)
X = torch.rand(16, n, dtype=torch.float64, device="cuda")
Y = torch.zeros_like(X)
lib = _lib.load()
s = torch.cuda.current_stream()
def run():
    _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n, 1.0, 0.0,
                                 _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream or 1)))
for _ in range(3): run()
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20): run()
    e1.record(s); torch.cuda.synchronize()
    print("mv16 ms", round(e0.elapsed_time(e1) / 20, 3))
