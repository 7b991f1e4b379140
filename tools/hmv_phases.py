"""Per-phase device time of the single-vector mat-vec (upsweep | coupling + dense | downsweep | total)
for 2D rank 36 / 64 at n = 2^20 and 2^22 (h2b_set_phase_timing events)."""
import sys, json
sys.path.insert(0, ".")
import torch
import paper_1902_01829_b200 as h2
for order, n in [(6, 1 << 20), (8, 1 << 20), (8, 1 << 22)]:
    A = h2.H2Matrix.construct(2, n, grid_order=order)
    x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
    for _ in range(3): h2.hmv(A, x, y)
    torch.cuda.synchronize()
    A.set_phase_timing(True)
    for _ in range(20): h2.hmv(A, x, y)
    torch.cuda.synchronize()
    ph = A.last_hmv_timing()
    A.set_phase_timing(False)
    inf = A.info()
    print(json.dumps({"order": order, "n": n, "fp_GB": A.memory_footprint() / 1e9, "phases_ms": [round(v, 4) for v in ph]}))
    A.close()
