"""Generate the committed golden fixtures from the REAL reference (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref was
compiled by `make -C oracle`):

    PYTHONPATH=. python tests/golden/make_golden.py

For each case: the reference's construct() parameters, x = random_vector(n, 1),
y = hmv(A, x) (alpha=1, beta=0), y2 = hmv(A, x, y0, 2, 3) for y0 = random_vector(n, 2),
memory_footprint, the analytic hmv flop count, and compress(A, eps): new ranks,
frobenius_error/norm, bytes after, and hmv(A_compressed, x).  A CRC of the
exported matrix arrays pins construct() bit for bit.
"""
import json
import os
import sys
import zlib

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import oracle  # noqa: E402

CASES = [
    # name, dim, n, order, eps
    ("2d_n256_k64", 2, 256, 8, 1e-7),
    ("2d_n1024_k64", 2, 1024, 8, 1e-7),
    ("2d_n4096_k16", 2, 4096, 4, 1e-7),
    ("2d_n4096_k36", 2, 4096, 6, 1e-7),
    ("3d_n4096_k64", 3, 4096, 4, 1e-6),
    ("3d_n2048_k27", 3, 2048, 3, 1e-3),
]


def crc_of(hm):
    c = 0
    for a in hm.arrays():
        c = zlib.crc32(np.ascontiguousarray(a).tobytes(), c)
    return c


def main():
    R = oracle.reference()
    out_dir = os.path.dirname(os.path.abspath(__file__))
    index = {}
    for name, dim, n, order, eps in CASES:
        A = R.construct(dim, n, grid_order=order)
        x = R.random_vector(n, 1)
        y0 = R.random_vector(n, 2)
        y = A.hmv(x)
        y2 = A.hmv(x, y0, 2.0, 3.0)
        hm = A.to_host()
        rep = A.compress(eps)
        yc = A.hmv(x)
        np.savez_compressed(os.path.join(out_dir, name + ".npz"), x=x, y=y, y0=y0, y2=y2, yc=yc)
        index[name] = dict(dim=dim, n=n, grid_order=order, eps=eps, leaf_size=64, eta=2.0,
                           ell=0.1 if dim == 2 else 0.2, perturbation=0.25, seed=1,
                           ranks=[int(r) for r in hm.ranks], footprint=hm.footprint(),
                           hmv_flops=hm.hmv_flops(), crc32=crc_of(hm),
                           cpl_blocks=hm.cpl_blocks(), dense_blocks=int(hm.dense_row_ptr[-1]),
                           compress=dict(new_ranks=rep["new_ranks"],
                                         frobenius_error=rep["frobenius_error"],
                                         frobenius_norm=rep["frobenius_norm"],
                                         bytes_after=int(rep["bytes_after"]),
                                         total_flops=rep["total_flops"]))
        print(name, index[name]["ranks"], "->", rep["new_ranks"], rep["frobenius_error"])
    with open(os.path.join(out_dir, "golden.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
