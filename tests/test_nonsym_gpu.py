"""GPU: non-symmetric matrices (U != V; h2_matrix.hpp:69,75-78, hmv.hpp:175-188:
the upsweep runs on A.col_basis(), the downsweep on A.row_basis).

* an operator-preserving column basis V = U D gives the symmetric matrix's
  hmv (no oracle involved);
* random column bases of other ranks: hmv and the phase entry points equal
  the reference's on the imported matrix; footprint and flop model too;
* containers: byte-identical to the reference's save, both directions;
* compress (both bases orthogonalized, projected, weighted -- the column
  weight tree over the transposed layers -- and truncated,
  compression.hpp:466-551) against the reference's compress of the same
  matrix: row and column ranks, error estimate, bytes, the operator.  The
  reference's weight-tree marshaling (compression.hpp:194-205, 236-243)
  assumes square coupling blocks (ranks[l] x ranks[l]): with row rank !=
  column rank on a level that has blocks it reads past them (undefined
  behaviour: run-to-run different results, NaNs), so reference parity uses
  equal ranks on the levels with blocks; unequal ranks are checked by the
  operator they preserve;
* the 16-vector pass;
* orthogonalize_basis on the row basis and on the column basis (the two
  entry points h2b_orthogonalize / h2b_orthogonalize_col) against the
  reference's orthogonalize_basis(A.row_basis / A.col_basis())."""
import numpy as np
import pytest

from conftest import rel_err
from nonsym import random_cols, scaled

import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib

pytestmark = pytest.mark.gpu

CASES = [(2, 1 << 12, 4), (3, 1 << 12, 3), (2, 1 << 13, 8)]


@pytest.mark.parametrize("dim,n,order", CASES)
def test_scaled_column_basis_is_the_same_operator(gpu, ref, dim, n, order):
    R = ref.construct(dim, n, grid_order=order)
    hm = R.to_host()
    S = h2.H2Matrix.from_host(hm)
    N = h2.H2Matrix.from_host(scaled(hm))
    assert N.info().symmetric == 0 and S.info().symmetric == 1
    x = np.random.default_rng(1).random(n)
    ys, yn = h2.hmv(S, x), h2.hmv(N, x)
    assert rel_err(yn, ys) <= 1e-13
    assert rel_err(yn, R.hmv(x)) <= 1e-12


@pytest.mark.parametrize("dim,n,order", CASES)
def test_random_column_basis_matches_reference(gpu, ref, dim, n, order):
    hm = random_cols(ref.construct(dim, n, grid_order=order).to_host())
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    inf = A.info()
    assert list(inf.col_ranks)[:hm.depth + 1] == hm.col_ranks.tolist()
    assert A.memory_footprint() == R.footprint() == hm.footprint()
    assert inf.hmv_flops == pytest.approx(R.hmv_flops(), rel=1e-12)
    rng = np.random.default_rng(5)
    x = rng.random(n)
    assert rel_err(h2.hmv(A, x), R.hmv(x)) <= 1e-12
    y0 = rng.random(n)
    assert rel_err(h2.hmv(A, x, y0.copy(), 2.0, -0.5), R.hmv(x, y0.copy(), 2.0, -0.5)) <= 1e-12


def test_phase_entry_points_use_the_column_basis(gpu, ref):
    n = 1 << 12
    hm = random_cols(ref.construct(2, n, grid_order=4).to_host())
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    xc = np.random.default_rng(9).random(n)
    xh_ref = R.upsweep(xc)
    xh = h2.upsweep(A, xc)
    assert xh.size == xh_ref.size  # column-rank sized
    assert rel_err(xh, xh_ref) <= 1e-13
    yh_ref = R.tree_multiply(xh_ref)
    yh = h2.tree_multiply(A, xh)
    assert yh.size == yh_ref.size  # row-rank sized
    assert rel_err(yh, yh_ref) <= 1e-13


def test_export_roundtrip(gpu, ref):
    hm = random_cols(ref.construct(3, 1 << 12, grid_order=3).to_host())
    back = h2.H2Matrix.from_host(hm).to_host()
    assert not back.symmetric
    for a in ("ranks", "col_ranks", "perm", "leaf", "transfer", "col_leaf", "col_transfer",
              "cpl_row_ptr", "cpl_col_idx", "cpl_values", "dense_row_ptr", "dense_col_idx",
              "dense_values"):
        assert np.array_equal(getattr(back, a), getattr(hm, a)), a


def test_container_byte_identical_both_ways(gpu, ref, tmp_path):
    n = 1 << 12
    hm = random_cols(ref.construct(2, n, grid_order=4).to_host())
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    ours, theirs = tmp_path / "ours.h2", tmp_path / "ref.h2"
    A.save(ours)
    R.save(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    B = h2.H2Matrix.load(theirs)
    R2 = ref.load(str(ours))
    x = np.random.default_rng(4).random(n)
    assert rel_err(h2.hmv(B, x), R2.hmv(x)) <= 1e-12
    assert B.info().symmetric == 0


def _col_ranks(R):
    import ctypes as C
    q = R.shape()[2]
    cr = np.zeros(q + 1, np.int32)
    R.be.lib.ref_col_ranks.argtypes = [C.c_void_p, C.c_void_p]
    R.be.lib.ref_col_ranks(R.h, cr.ctypes.data)
    return cr.tolist()


@pytest.mark.parametrize("dim,n,order,eps,make", [(2, 1 << 13, 8, 1e-7, "scaled"),
                                                   (3, 1 << 12, 4, 1e-6, "scaled"),
                                                   (2, 1 << 12, 6, 1e-5, "random")])
def test_compress_matches_reference(gpu, ref, dim, n, order, eps, make):
    base = ref.construct(dim, n, grid_order=order).to_host()
    hm = scaled(base) if make == "scaled" else random_cols(base, drop=0)  # (see module doc)
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    x = np.random.default_rng(3).random(n)
    y0 = R.hmv(x)
    rr = R.compress(eps)
    rg = h2.compress(A, eps)
    inf = A.info()
    assert inf.symmetric == 0
    assert all(abs(a - b) <= 1 for a, b in zip(rg.new_ranks, rr["new_ranks"])), (rg.new_ranks, rr["new_ranks"])
    cr = _col_ranks(R)
    assert all(abs(a - b) <= 1 for a, b in zip(inf.col_ranks, cr)), (inf.col_ranks, cr)
    if rg.new_ranks == rr["new_ranks"] and list(inf.col_ranks) == cr:
        assert rg.bytes_after == int(rr["bytes_after"])
    assert rg.bytes_before == int(rr["bytes_before"])
    assert 0.5 * rr["frobenius_error"] <= rg.frobenius_error <= 2.0 * rr["frobenius_error"] + 1e-15
    assert rg.frobenius_norm == pytest.approx(rr["frobenius_norm"], rel=1e-10)
    yg, yr = h2.hmv(A, x), R.hmv(x)
    assert rel_err(yg, y0) <= 10 * eps
    assert rel_err(yg, yr) <= 10 * eps
    # the compressed matrix round-trips through the reference
    back = ref.from_host(A.to_host())
    assert rel_err(back.hmv(x), yg) <= 1e-12


def test_multi_vector_pass(gpu, ref):
    """16 right-hand sides on the FP64 tensor cores (h2b_hmv_multi): the
    upsweep on the column basis, as in the single-vector path."""
    n = 1 << 12
    hm = random_cols(ref.construct(2, n, grid_order=6).to_host())
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    X = np.random.default_rng(8).random((16, n))
    Y = h2.hmv_multi(A, X)
    for v in (0, 7, 15):
        assert rel_err(Y[v], R.hmv(X[v])) <= 1e-12


@pytest.mark.parametrize("make", ["scaled", "random"])
def test_orthogonalize_each_basis_matches_reference(gpu, ref, make):
    """compression.hpp:69-126 on A.row_basis, then on A.col_basis(): projection
    trees and the orthogonalized pools against the reference's; the other
    basis and the coupling are untouched."""
    base = ref.construct(2, 1 << 12, grid_order=6).to_host()
    hm = scaled(base) if make == "scaled" else random_cols(base)
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    t_row = h2.orthogonalize_basis(A, "row")
    assert rel_err(t_row, R.orthogonalize()) <= 1e-11
    mid = A.to_host()
    assert np.array_equal(mid.col_leaf, hm.col_leaf) and np.array_equal(mid.col_transfer, hm.col_transfer)
    assert np.array_equal(mid.cpl_values, hm.cpl_values)
    t_col = h2.orthogonalize_basis(A, "col")
    assert rel_err(t_col, R.orthogonalize_col()) <= 1e-11
    got, want = A.to_host(), R.to_host()
    for a in ("leaf", "transfer", "col_leaf", "col_transfer"):
        assert rel_err(getattr(got, a), getattr(want, a)) <= 1e-11, a
    assert np.array_equal(got.leaf, mid.leaf)  # the row basis untouched by the column call
    # orthonormal column leaves (acceptance c3 on V)
    m, kq = hm.m, int(hm.col_ranks[-1])
    V = got.col_leaf.reshape(-1, kq, m).transpose(0, 2, 1)
    G = np.einsum("bij,bik->bjk", V, V)
    assert np.max(np.abs(G - np.eye(kq))) <= 1e-12
    with pytest.raises(ValueError):
        h2.orthogonalize_basis(A, "diagonal")


def _with_col_ranks(base, col_ranks, seed):
    """The structure of `base` with a fresh random column basis of the given ranks."""
    from paper_1902_01829_b200.host import HostMatrix
    q, m, n = base.depth, base.m, base.n
    hm = HostMatrix.empty(n, m, q, base.ranks, base.cpl_blocks(), int(base.dense_row_ptr[-1]),
                          np.asarray(col_ranks, np.int32))
    rng = np.random.default_rng(seed)
    for a in ("perm", "leaf", "transfer", "cpl_row_ptr", "cpl_col_idx", "dense_row_ptr", "dense_col_idx",
              "dense_values"):
        getattr(hm, a)[:] = getattr(base, a)
    hm.col_leaf[:] = rng.standard_normal(hm.col_leaf.size) / 8
    hm.col_transfer[:] = rng.standard_normal(hm.col_transfer.size) / 2
    hm.cpl_values[:] = rng.standard_normal(hm.cpl_values.size) * 1e-2
    return hm


@pytest.mark.parametrize("drop", [0, 1, 5])
def test_odd_and_empty_column_ranks(gpu, ref, drop):
    """Odd column ranks, zero on the top levels (no coupling there, as after a
    compress): padded leading dimensions and empty levels on the x^ side.
    hmv / 16 vectors against the reference; compress against the reference
    where its marshaling is defined (drop 0: equal ranks on the levels with
    blocks), otherwise by the operator it preserves."""
    n = 1 << 12
    base = ref.construct(2, n, grid_order=5).to_host()  # rank 25
    cr = [0, 0, 0] + [25 - drop] * (base.depth - 2)
    hm = _with_col_ranks(base, cr, drop)
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    rng = np.random.default_rng(drop)
    x = rng.random(n)
    y0 = R.hmv(x)
    assert rel_err(h2.hmv(A, x), y0) <= 1e-12
    X = rng.random((16, n))
    assert rel_err(h2.hmv_multi(A, X)[3], R.hmv(X[3])) <= 1e-12
    eps = 1e-6
    rg = h2.compress(A, eps)
    assert all(a <= b for a, b in zip(rg.new_ranks, rg.old_ranks))
    assert rel_err(h2.hmv(A, x), y0) <= 10 * eps
    if drop == 0:
        rr = R.compress(eps)
        assert all(abs(a - b) <= 1 for a, b in zip(rg.new_ranks, rr["new_ranks"]))
        assert rel_err(h2.hmv(A, x), R.hmv(x)) <= 10 * eps


def test_invalid_weight_stack_rejected_like_reference(gpu, ref):
    """A column rank above an empty level whose stacks would be shorter than
    wide: the reference's qr_r_only_batched rejects it; so does compress()."""
    import oracle
    n = 1 << 12
    base = ref.construct(2, n, grid_order=5).to_host()
    hm = _with_col_ranks(base, [0, 0] + [24] * (base.depth - 1), 1)
    R = ref.from_host(hm)
    A = h2.H2Matrix.from_host(hm)
    with pytest.raises(oracle.OracleInvalidArgument) as er:
        R.compress(1e-6)
    with pytest.raises(_lib.H2bInvalidArgument) as eg:
        h2.compress(A, 1e-6)
    assert "qr_r_only_batched: requires rows >= cols" in str(er.value)
    assert "qr_r_only_batched: requires rows >= cols" in str(eg.value)


def test_orthogonalize_col_on_symmetric_is_the_row_basis(gpu, ref):
    """A.col_basis() is A.row_basis when symmetric (h2_matrix.hpp:75-78): both
    entry points orthogonalize the one basis, bitwise alike."""
    hm = ref.construct(2, 1 << 12, grid_order=6).to_host()
    A, B = h2.H2Matrix.from_host(hm), h2.H2Matrix.from_host(hm)
    t_row = h2.orthogonalize_basis(A, "row")
    t_col = h2.orthogonalize_basis(B, "col")
    assert np.array_equal(t_row, t_col)
    a, b = A.to_host(), B.to_host()
    assert np.array_equal(a.leaf, b.leaf) and np.array_equal(a.transfer, b.transfer)
    assert rel_err(t_row, ref.from_host(hm).orthogonalize()) <= 1e-11
