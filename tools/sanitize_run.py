"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): device construction, hmv (fused sweeps), 16-vector pass, phase
API, compress (orth / project / weights / truncation / compaction), a
non-symmetric matrix and its compress.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np

import paper_1902_01829_b200 as h2

n = 1 << 12
A = h2.H2Matrix.construct(2, n, grid_order=6)
x = np.random.default_rng(1).random(n)
y = h2.hmv(A, x)
Y = h2.hmv_multi(A, np.random.default_rng(2).random((16, n)))
xh = h2.upsweep(A, x)
yh = h2.tree_multiply(A, xh)
rep = h2.compress(A, 1e-6)
y2 = h2.hmv(A, x)
B = h2.H2Matrix.construct(3, n, grid_order=3)
h2.compress(B, 1e-5)
from nonsym import scaled  # noqa: E402

hm = A.to_host()
N = h2.H2Matrix.from_host(scaled(hm))
h2.hmv(N, x)
h2.compress(N, 1e-5)
print("ok", rep.new_ranks, float(np.linalg.norm(y2 - y) / np.linalg.norm(y)))
