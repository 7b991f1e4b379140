"""CPU: the host-side model of non-symmetric matrices (column basis V / F,
h2_matrix.hpp:69,75-78) against the reference imported from the same pools:
memory_footprint (h2_matrix.hpp:90-102, column basis counted), the hmv flop
model (flops.hpp over hmv.hpp:175-188) and the export round trip; the
operator-preserving column basis gives the symmetric matrix's hmv in the
reference itself."""
import numpy as np
import pytest

from conftest import rel_err
from nonsym import random_cols, scaled


@pytest.mark.parametrize("dim,n,order", [(2, 1 << 11, 4), (3, 1 << 11, 3)])
def test_host_model_matches_reference(ref, dim, n, order):
    hm = random_cols(ref.construct(dim, n, grid_order=order).to_host())
    R = ref.from_host(hm)
    assert R.shape()[3] == 0
    assert R.footprint() == hm.footprint()
    assert R.hmv_flops() == pytest.approx(hm.hmv_flops(), rel=1e-12)
    back = R.to_host()
    for a in ("col_ranks", "col_leaf", "col_transfer", "cpl_values", "leaf", "transfer"):
        assert np.array_equal(getattr(back, a), getattr(hm, a)), a


def test_scaled_basis_is_the_same_operator_in_the_reference(ref):
    n = 1 << 11
    R = ref.construct(2, n, grid_order=4)
    N = ref.from_host(scaled(R.to_host()))
    x = np.random.default_rng(2).random(n)
    assert rel_err(N.hmv(x), R.hmv(x)) <= 1e-13


def test_reference_column_orthogonalize_binding(ref):
    """oracle binding of orthogonalize_basis(A.col_basis()) (the checker of
    h2b_orthogonalize_col): orthonormal column leaves, the row basis untouched,
    and on a symmetric matrix the row-basis result."""
    base = ref.construct(2, 1 << 11, grid_order=4).to_host()
    R = ref.from_host(random_cols(base))
    before = R.to_host()
    t = R.orthogonalize_col()
    after = R.to_host()
    assert t.size == sum((1 << l) * int(k) ** 2 for l, k in enumerate(before.col_ranks))
    assert np.array_equal(after.leaf, before.leaf) and np.array_equal(after.transfer, before.transfer)
    k, m = int(after.col_ranks[-1]), after.m
    V = after.col_leaf.reshape(-1, k, m).transpose(0, 2, 1)
    assert np.max(np.abs(np.einsum("bij,bik->bjk", V, V) - np.eye(k))) <= 1e-12
    S1, S2 = ref.from_host(base), ref.from_host(base)
    assert np.array_equal(S1.orthogonalize_col(), S2.orthogonalize())
