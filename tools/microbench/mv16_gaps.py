"""16-vector pass at C4: CUDA-event time per pass with and without a host
sync between passes, and the host time per call (is the GPU starved?)."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import torch
import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib
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
for mode in ("back-to-back", "synced", "back-to-back"):
    ts = []
    t_host = 0.0
    for _ in range(10):
        e0.record(s)
        h0 = time.perf_counter()
        run()
        t_host += time.perf_counter() - h0
        e1.record(s)
        if mode == "synced":
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if mode != "synced":
        ts = [e0.elapsed_time(e1)]
    print(mode, "last-pass or per-pass ms:", [round(t, 3) for t in ts], "host ms per call:", round(1e3 * t_host / 10, 3), flush=True)
e0.record(s)
for _ in range(10):
    run()
e1.record(s)
torch.cuda.synchronize()
print("10 back-to-back:", round(e0.elapsed_time(e1) / 10, 3), "ms per pass", flush=True)
