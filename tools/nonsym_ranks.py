import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, oracle, paper_1902_01829_b200 as h2
from nonsym import scaled, random_cols
ref = oracle.reference()
for dim, n, order, eps, make in [(2, 1 << 13, 8, 1e-7, "scaled"), (3, 1 << 12, 4, 1e-6, "scaled"), (2, 1 << 12, 6, 1e-5, "random"), (2, 1 << 14, 8, 1e-7, "scaled")]:
    base = ref.construct(dim, n, grid_order=order).to_host()
    hm = scaled(base) if make == "scaled" else random_cols(base, drop=0)
    R = ref.from_host(hm); A = h2.H2Matrix.from_host(hm)
    rr = R.compress(eps); rg = h2.compress(A, eps)
    import ctypes as C
    q = R.shape()[2]; cr = np.zeros(q + 1, np.int32)
    R.be.lib.ref_col_ranks.argtypes = [C.c_void_p, C.c_void_p]; R.be.lib.ref_col_ranks(R.h, cr.ctypes.data)
    print(make, dim, n, "row", rg.new_ranks == rr["new_ranks"], "col", list(A.info().col_ranks) == cr.tolist(),
          rg.new_ranks, list(A.info().col_ranks), "frob", rg.frobenius_error, rr["frobenius_error"], "bytes", rg.bytes_after, int(rr["bytes_after"]))
