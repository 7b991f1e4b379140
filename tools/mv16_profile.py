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
for _ in range(2):
    _lib.check(lib.h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), n, C.c_void_p(Y.data_ptr()), n, 1.0, 0.0, _lib.PTR_DEVICE, None))
torch.cuda.synchronize()
