"""One compress() of a given config, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import paper_1902_01829_b200 as h2
dim, n, order, eps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
A = h2.H2Matrix.construct(dim, n, grid_order=order)
rep = h2.compress(A, eps)
print(rep.new_ranks, rep.total_ms(), rep.total_flops() / rep.total_ms() / 1e9, "TF/s model")
