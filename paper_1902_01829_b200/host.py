"""Host-side H^2 matrix in the reference's flat pool layout ("export layout").

This mirrors the reference's ``H2Matrix<double>`` (include/h2kit/h2_matrix.hpp:62-80)
with every per-level ``std::vector`` pool concatenated over levels:

* ``perm[n]``                          -- H2Matrix::perm (cluster position -> point id)
* ``ranks[depth+1]``                   -- BasisTree::ranks
* ``leaf``                             -- BasisTree::leaf_pool, 2^depth blocks of m x ranks[depth]
* ``transfer``                         -- BasisTree::transfer[l], l = 1..depth, 2^l blocks of
                                          ranks[l] x ranks[l-1]
* ``cpl_row_ptr / cpl_col_idx / cpl_values`` -- MatrixTree::levels[l] (BSRLayer, bsr.hpp:13-31)
* ``dense_row_ptr / dense_col_idx / dense_values`` -- H2Matrix::dense
* ``col_ranks / col_leaf / col_transfer`` -- the column basis V / F of a
  non-symmetric matrix (H2Matrix::col_basis_store, h2_matrix.hpp:69,75-78);
  None when symmetric.  Coupling blocks of level l are then
  ranks[l] x col_ranks[l].

All blocks are column-major; values are float64, indices int32 (index_t,
include/h2kit/defs.hpp:15).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class HostMatrix:
    n: int
    m: int
    depth: int
    ranks: np.ndarray
    perm: np.ndarray
    leaf: np.ndarray
    transfer: np.ndarray
    cpl_row_ptr: np.ndarray
    cpl_col_idx: np.ndarray
    cpl_values: np.ndarray
    dense_row_ptr: np.ndarray
    dense_col_idx: np.ndarray
    dense_values: np.ndarray
    meta: dict = field(default_factory=dict)
    col_ranks: np.ndarray | None = None
    col_leaf: np.ndarray | None = None
    col_transfer: np.ndarray | None = None

    @property
    def symmetric(self) -> bool:
        return self.col_ranks is None

    def cranks(self) -> np.ndarray:
        return self.ranks if self.col_ranks is None else self.col_ranks

    # -- layout helpers -------------------------------------------------
    def nodes(self, l: int) -> int:
        return 1 << l

    def cpl_blocks(self) -> list[int]:
        out, o = [], 0
        for l in range(self.depth + 1):
            rp = self.cpl_row_ptr[o:o + self.nodes(l) + 1]
            out.append(int(rp[-1]))
            o += self.nodes(l) + 1
        return out

    def level_row_ptr(self, l: int) -> np.ndarray:
        o = sum(self.nodes(j) + 1 for j in range(l))
        return self.cpl_row_ptr[o:o + self.nodes(l) + 1]

    def level_col_idx(self, l: int) -> np.ndarray:
        nb = self.cpl_blocks()
        o = sum(nb[:l])
        return self.cpl_col_idx[o:o + nb[l]]

    def level_values(self, l: int) -> np.ndarray:
        """Coupling blocks of level l as an array (nb, k, k) in column-major blocks
        (block[b][:, j] is column j)."""
        nb = self.cpl_blocks()
        c = self.cranks()
        k, kc = int(self.ranks[l]), int(c[l])
        o = sum(nb[j] * int(self.ranks[j]) * int(c[j]) for j in range(l))
        v = self.cpl_values[o:o + nb[l] * k * kc]
        return v.reshape(nb[l], kc, k).transpose(0, 2, 1)

    def transfer_level(self, l: int) -> np.ndarray:
        """Transfers of level l as (2^l, k_l, k_{l-1})."""
        o = sum(self.nodes(j) * int(self.ranks[j]) * int(self.ranks[j - 1]) for j in range(1, l))
        kc, kp = int(self.ranks[l]), int(self.ranks[l - 1])
        v = self.transfer[o:o + self.nodes(l) * kc * kp]
        return v.reshape(self.nodes(l), kp, kc).transpose(0, 2, 1)

    def leaves(self) -> np.ndarray:
        k = int(self.ranks[self.depth])
        return self.leaf.reshape(self.nodes(self.depth), k, self.m).transpose(0, 2, 1)

    def vec_offsets(self) -> list[int]:
        off = [0]
        for l in range(self.depth + 1):
            off.append(off[-1] + self.nodes(l) * int(self.ranks[l]))
        return off

    def footprint(self) -> int:
        """memory_footprint(A).total() (h2_matrix.hpp:90-102)."""
        f = self.dense_values.size + self.cpl_values.size + self.leaf.size + self.transfer.size
        if not self.symmetric:
            f += self.col_leaf.size + self.col_transfer.size
        return 8 * int(f)

    def hmv_flops(self) -> float:
        """Reference analytic flop model of one hmv (flops.hpp:29-47)."""
        q, m = self.depth, self.m
        r = [int(v) for v in self.ranks]
        c = [int(v) for v in self.cranks()]
        nbd = int(self.dense_row_ptr[-1])
        f = 2.0 * m * m * nbd + 2.0 * m * (r[q] + c[q]) * self.nodes(q)
        for l in range(1, q + 1):
            f += 2.0 * (r[l] * r[l - 1] + c[l] * c[l - 1]) * self.nodes(l)
        for l, nb in enumerate(self.cpl_blocks()):
            if nb:
                f += 2.0 * r[l] * c[l] * nb
        return f

    def validate(self) -> None:
        """Array dtypes and sizes against n, m, depth, ranks and the block
        counts of the row pointers (ValueError otherwise): the C side reads
        exactly that many entries from every pointer."""
        q, m, n = int(self.depth), int(self.m), int(self.n)
        if q < 0 or q > 30 or m < 1 or (m << q) != n:
            raise ValueError("HostMatrix: n must equal m * 2^depth")

        def arr(a, dt, size, name):
            if not isinstance(a, np.ndarray) or a.dtype != dt:
                raise ValueError(f"HostMatrix.{name}: must be a {np.dtype(dt).name} array")
            if a.size != size:
                raise ValueError(f"HostMatrix.{name}: has {a.size} entries, expected {size}")

        if len(self.ranks) != q + 1:
            raise ValueError(f"HostMatrix.ranks: expected {q + 1} levels")
        r = [int(v) for v in self.ranks]
        c = [int(v) for v in self.cranks()]
        if len(c) != q + 1:
            raise ValueError(f"HostMatrix.col_ranks: expected {q + 1} levels")
        arr(self.perm, np.int32, n, "perm")
        arr(self.leaf, np.float64, (1 << q) * m * r[q], "leaf")
        arr(self.transfer, np.float64, sum((1 << l) * r[l] * r[l - 1] for l in range(1, q + 1)), "transfer")
        arr(self.cpl_row_ptr, np.int32, sum((1 << l) + 1 for l in range(q + 1)), "cpl_row_ptr")
        nb = self.cpl_blocks()
        if any(b < 0 for b in nb):
            raise ValueError("HostMatrix.cpl_row_ptr: negative block count")
        arr(self.cpl_col_idx, np.int32, sum(nb), "cpl_col_idx")
        arr(self.cpl_values, np.float64, sum(b * r[l] * c[l] for l, b in enumerate(nb)), "cpl_values")
        arr(self.dense_row_ptr, np.int32, (1 << q) + 1, "dense_row_ptr")
        nd = int(self.dense_row_ptr[-1])
        arr(self.dense_col_idx, np.int32, nd, "dense_col_idx")
        arr(self.dense_values, np.float64, nd * m * m, "dense_values")
        if not self.symmetric:
            arr(self.col_leaf, np.float64, (1 << q) * m * c[q], "col_leaf")
            arr(self.col_transfer, np.float64, sum((1 << l) * c[l] * c[l - 1] for l in range(1, q + 1)),
                "col_transfer")

    def copy(self) -> "HostMatrix":
        cp = lambda a: None if a is None else np.array(a, copy=True)  # noqa: E731
        return HostMatrix(self.n, self.m, self.depth, *(np.array(a, copy=True) for a in (
            self.ranks, self.perm, self.leaf, self.transfer, self.cpl_row_ptr, self.cpl_col_idx,
            self.cpl_values, self.dense_row_ptr, self.dense_col_idx, self.dense_values)),
            meta=dict(self.meta), col_ranks=cp(self.col_ranks), col_leaf=cp(self.col_leaf),
            col_transfer=cp(self.col_transfer))

    @staticmethod
    def empty(n, m, depth, ranks, cpl_blocks, dense_blocks, col_ranks=None) -> "HostMatrix":
        ranks = np.asarray(ranks, dtype=np.int32)
        c = ranks if col_ranks is None else np.asarray(col_ranks, dtype=np.int32)
        nl = 1 << depth
        ntr = sum((1 << l) * int(ranks[l]) * int(ranks[l - 1]) for l in range(1, depth + 1))
        nrp = sum((1 << l) + 1 for l in range(depth + 1))
        nci = int(sum(cpl_blocks))
        nsv = int(sum(int(b) * int(ranks[l]) * int(c[l]) for l, b in enumerate(cpl_blocks)))
        col = {}
        if col_ranks is not None:
            ctr = sum((1 << l) * int(c[l]) * int(c[l - 1]) for l in range(1, depth + 1))
            col = dict(col_ranks=c, col_leaf=np.zeros(nl * m * int(c[depth]), np.float64),
                       col_transfer=np.zeros(ctr, np.float64))
        return HostMatrix(
            n=n, m=m, depth=depth, ranks=ranks,
            perm=np.zeros(n, np.int32),
            leaf=np.zeros(nl * m * int(ranks[depth]), np.float64),
            transfer=np.zeros(ntr, np.float64),
            cpl_row_ptr=np.zeros(nrp, np.int32),
            cpl_col_idx=np.zeros(nci, np.int32),
            cpl_values=np.zeros(nsv, np.float64),
            dense_row_ptr=np.zeros(nl + 1, np.int32),
            dense_col_idx=np.zeros(int(dense_blocks), np.int32),
            dense_values=np.zeros(int(dense_blocks) * m * m, np.float64),
            **col,
        )

    def arrays(self):
        return (self.perm, self.leaf, self.transfer, self.cpl_row_ptr, self.cpl_col_idx,
                self.cpl_values, self.dense_row_ptr, self.dense_col_idx, self.dense_values)
