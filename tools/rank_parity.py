"""Compression parity sweep against the reference (oracle/_ref): per case, are
the per-level ranks identical, the bytes identical, and how close are the error
estimates.  Writes one line per case.
    python tools/rank_parity.py"""
import sys

sys.path.insert(0, ".")
import numpy as np

import oracle
import paper_1902_01829_b200 as h2

ref = oracle.reference()
same = total = 0
for dim, n, order in [(2, 1 << 13, 8), (2, 1 << 14, 6), (3, 1 << 12, 4), (3, 1 << 13, 3), (2, 1 << 12, 4)]:
    for eps in [1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-12]:
        R = ref.construct(dim, n, grid_order=order)
        A = h2.H2Matrix.from_host(R.to_host())
        rr = R.compress(eps)
        rg = h2.compress(A, eps)
        eq = rg.new_ranks == rr["new_ranks"]
        same += eq
        total += 1
        fe = rg.frobenius_error / rr["frobenius_error"] if rr["frobenius_error"] > 0 else float("nan")
        print(f"{dim}D n={n} order={order} eps={eps:g}: ranks {'identical' if eq else 'DIFFER'} "
              f"{rg.new_ranks if eq else (rg.new_ranks, rr['new_ranks'])} bytes "
              f"{'identical' if rg.bytes_after == int(rr['bytes_after']) else 'differ'} "
              f"err ratio {fe:.12f}", flush=True)
print(f"identical ranks in {same} of {total} cases")
