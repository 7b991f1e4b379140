import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1902_01829_b200 as h2
dim, n, order = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = h2.H2Matrix.construct(dim, n, grid_order=order)
inf = A.info()
print(dim, n, order, inf.ranks, inf.cpl_blocks, flush=True)
x = np.random.default_rng(1).random(n)
print(h2.hmv(A, x)[:2], flush=True)
