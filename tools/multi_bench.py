"""Time the 16-vector FP64-MMA mat-vec at n = 2^22 (C4) vs 16 single-vector calls."""
import ctypes as C
import json
import sys
sys.path.insert(0, ".")
import torch
import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
A = h2.H2Matrix.construct(2, n)
fp = A.memory_footprint()
flops = A.info().hmv_flops
X = torch.rand(16, n, dtype=torch.float64, device="cuda")
Y = torch.zeros_like(X)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
lib = _lib.load()
def run():
    _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n,
                                 1.0, 0.0, _lib.PTR_DEVICE, C.c_void_p(s.cuda_stream)))
for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
K = 10
for _ in range(K):
    run()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
y1 = h2.hmv(A, X[3].contiguous())
torch.cuda.synchronize()
err = float((Y[3] - y1).norm() / y1.norm())
print(json.dumps(dict(n=n, ms_16vec=round(ms, 3), ms_per_vector=round(ms / 16, 4),
                      effective_GBs=round(16 * fp / ms / 1e6, 1), matrix_pass_GBs=round(fp / ms / 1e6, 1),
                      model_TFLOPs=round(16 * flops / ms / 1e9, 2), col3_rel_err_vs_single=err)))
