"""C4 single-vector mat-vec, a few calls (for ncu captures of its kernels)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1902_01829_b200 as h2
A = h2.H2Matrix.construct(2, 1 << 22, grid_order=8)
x = torch.rand(1 << 22, dtype=torch.float64, device='cuda')
y = torch.zeros_like(x)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    h2.hmv(A, x, y)
torch.cuda.synchronize()
