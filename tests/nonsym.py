"""Non-symmetric test matrices (H2Matrix::col_basis_store, h2_matrix.hpp:69,75-78).

construct() only produces symmetric matrices and the reference's own tests
never build a non-symmetric one, so these are derived from a constructed
matrix:

* ``scaled``: the same operator with V = U D: per level a positive diagonal
  D_l, V leaves = U D_q, F_c = D_l^-1 E_c D_{l-1}, S'_l = S_l D_l^-1.  Then
  V_parent = [V_c1 F_c1; V_c2 F_c2] = U_parent D_{l-1} and U S' V^T = U S U^T:
  the hmv must equal the symmetric one's.
* ``random_cols``: a column basis of different (smaller) ranks with random
  entries and random coupling blocks of ranks[l] x col_ranks[l] on the same
  block structure -- checked against the reference's own hmv on the imported
  matrix.
"""
from __future__ import annotations

import numpy as np

from paper_1902_01829_b200.host import HostMatrix


def scaled(hm: HostMatrix, seed: int = 7) -> HostMatrix:
    rng = np.random.default_rng(seed)
    q, m = hm.depth, hm.m
    r = [int(v) for v in hm.ranks]
    d = [0.5 + rng.random(k) for k in r]
    out = hm.copy()
    out.col_ranks = np.array(r, np.int32)
    nl = 1 << q
    leaves = hm.leaf.reshape(nl, r[q], m)  # [leaf][column][row]
    out.col_leaf = (leaves * d[q][None, :, None]).reshape(-1).copy()
    parts = []
    for l in range(1, q + 1):
        E = hm.transfer_level(l)  # (2^l, k_l, k_{l-1})
        F = E / d[l][None, :, None] * d[l - 1][None, None, :]
        parts.append(F.transpose(0, 2, 1).reshape(-1))
    out.col_transfer = np.concatenate(parts) if parts else np.zeros(0)
    vals = []
    for l in range(q + 1):
        S = hm.level_values(l)  # (nb, k, k)
        if S.size:
            vals.append((S / d[l][None, None, :]).transpose(0, 2, 1).reshape(-1))
    out.cpl_values = np.concatenate(vals) if vals else np.zeros(0)
    return out


def random_cols(hm: HostMatrix, seed: int = 11, drop: int = 3) -> HostMatrix:
    rng = np.random.default_rng(seed)
    q, m = hm.depth, hm.m
    r = [int(v) for v in hm.ranks]
    c = [max(1, k - drop) if k else 0 for k in r]
    c[q] = min(c[q], m)
    nb = hm.cpl_blocks()
    out = HostMatrix.empty(hm.n, m, q, r, nb, int(hm.dense_row_ptr[-1]), c)
    out.perm[:] = hm.perm
    out.leaf[:] = hm.leaf
    out.transfer[:] = hm.transfer
    out.cpl_row_ptr[:] = hm.cpl_row_ptr
    out.cpl_col_idx[:] = hm.cpl_col_idx
    out.dense_row_ptr[:] = hm.dense_row_ptr
    out.dense_col_idx[:] = hm.dense_col_idx
    out.dense_values[:] = hm.dense_values
    out.col_leaf[:] = rng.standard_normal(out.col_leaf.size) / np.sqrt(m)
    out.col_transfer[:] = rng.standard_normal(out.col_transfer.size) * 0.5
    out.cpl_values[:] = rng.standard_normal(out.cpl_values.size) * 1e-2
    return out
