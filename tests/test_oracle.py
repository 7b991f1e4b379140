"""CPU: the restated oracle is pinned to the real reference and its KATs."""
import numpy as np
import pytest

from conftest import rel_err

from paper_1902_01829_b200.host import HostMatrix


def test_golden_vectors_reproduced_by_restatement(orc, golden):
    import zlib
    for name, (meta, arr) in golden.items():
        A = orc.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
        hm = A.to_host()
        crc = 0
        for a in hm.arrays():
            crc = zlib.crc32(np.ascontiguousarray(a).tobytes(), crc)
        assert crc == meta["crc32"], name  # construct() bit-identical to the reference
        assert hm.footprint() == meta["footprint"]
        assert hm.hmv_flops() == pytest.approx(meta["hmv_flops"], rel=1e-15)
        assert np.array_equal(A.hmv(arr["x"]), arr["y"]), name  # bit-identical hmv
        assert np.array_equal(A.hmv(arr["x"], arr["y0"], 2.0, 3.0), arr["y2"]), name
        rep = A.compress(meta["eps"])
        assert rep["new_ranks"] == meta["compress"]["new_ranks"], name
        assert rep["frobenius_error"] == meta["compress"]["frobenius_error"], name
        assert int(rep["bytes_after"]) == meta["compress"]["bytes_after"]
        assert np.array_equal(A.hmv(arr["x"]), arr["yc"]), name


def test_restatement_matches_reference_live(orc, ref):
    for dim, n, order in [(2, 2048, 8), (3, 2048, 4)]:
        a, b = ref.construct(dim, n, grid_order=order), orc.construct(dim, n, grid_order=order)
        for x, y in zip(a.to_host().arrays(), b.to_host().arrays()):
            assert np.array_equal(x, y)
        x = ref.random_vector(n, 7)
        xc = x[a.to_host().perm]
        assert np.array_equal(a.upsweep(xc), b.upsweep(xc))
        xh = a.upsweep(xc)
        assert np.array_equal(a.tree_multiply(xh), b.tree_multiply(xh))
        assert np.array_equal(a.dense_mv(xc), b.dense_mv(xc))
        assert np.array_equal(a.downsweep(xh, xc), b.downsweep(xh, xc))
        assert np.array_equal(a.orthogonalize(), b.orthogonalize())
        a2, b2 = ref.construct(dim, n, grid_order=order), orc.construct(dim, n, grid_order=order)
        assert np.array_equal(a2.orth_project_weights(), b2.orth_project_weights())
        ra, rb = a.compress(1e-6), b.compress(1e-6)
        assert ra["new_ranks"] == rb["new_ranks"]
        assert ra["frobenius_error"] == rb["frobenius_error"]
        assert ra["total_flops"] == pytest.approx(rb["total_flops"], rel=1e-14)


def test_import_export_roundtrip(orc, ref):
    a = ref.construct(2, 1024)
    hm = a.to_host()
    b = orc.from_host(hm)
    c = ref.from_host(hm)
    for x, y, z in zip(hm.arrays(), b.to_host().arrays(), c.to_host().arrays()):
        assert np.array_equal(x, y) and np.array_equal(x, z)


def test_hmv_matches_dense_expansion(ref):
    # test_hmv.cpp:74-89: hmv vs the O(n^2) expansion <= 1e-12.
    for n in (256, 1024):
        A = ref.construct(2, n)
        D = A.expand_dense()
        rng = np.random.default_rng(17)
        for _ in range(3):
            x = rng.random(n)
            assert rel_err(A.hmv(x), D @ x) <= 1e-12


def test_kat_qr_3_4(orc):
    # test_batch.cpp:152-161: [3;4] -> R = 5, Q = (0.6, 0.8).
    a = np.array([3.0, 4.0])
    r = np.zeros(1)
    assert orc.lib.h2o_qr(2, 1, a.ctypes.data, r.ctypes.data) == 0
    assert r[0] == pytest.approx(5.0, abs=1e-14)
    assert np.allclose(a, [0.6, 0.8], atol=1e-15)


def test_kat_svd_diag(orc):
    # test_batch.cpp:215-226: diag(1, 1e-9), eps 1e-6 -> rank 1, sigma2 = 1e-9.
    W = np.array([1.0, 0.0, 0.0, 1e-9])
    rank = np.zeros(1, np.int32)
    sig = np.zeros(2)
    assert orc.lib.h2o_svd(2, 2, W.ctypes.data, 1e-6, rank.ctypes.data, sig.ctypes.data) == 0
    assert rank[0] == 1
    assert sig[1] ** 2 == pytest.approx(1e-18, rel=1e-12)


def test_svd_rejects_nan(orc):
    W = np.array([np.nan, 0.0, 0.0, 1.0])
    rank = np.zeros(1, np.int32)
    sig = np.zeros(2)
    assert orc.lib.h2o_svd(2, 2, W.ctypes.data, 1e-6, rank.ctypes.data, sig.ctypes.data) == 1


def test_errors_mirror_reference(orc, ref):
    import oracle
    for be in (orc, ref):
        with pytest.raises(oracle.OracleInvalidArgument, match="leaf_size"):
            be.construct(2, 900)  # perfect square, but not 64 * 2^q
        with pytest.raises(oracle.OracleInvalidArgument, match="dim must be 2 or 3"):
            be.construct(4, 1024)
        A = be.construct(2, 1024)
        with pytest.raises(oracle.OracleInvalidArgument, match="eps must be non-negative"):
            A.compress(-1.0)


def test_host_matrix_layout_helpers(golden):
    import oracle
    meta, _ = golden["2d_n1024_k64"]
    hm = oracle.restated().construct(2, 1024).to_host()
    assert hm.cpl_blocks() == meta["cpl_blocks"]
    assert int(hm.dense_row_ptr[-1]) == meta["dense_blocks"]
    assert isinstance(hm.copy(), HostMatrix)


def test_restatement_matches_reference_above_rank_64(orc, ref):
    """The oracle for the k_hmv_big.cu path (ranks / leaf sizes 65..128): the
    restated construct() and hmv are bit-identical to the reference's."""
    for dim, n, leaf, order in [(2, 4096, 64, 9), (2, 4096, 128, 10), (3, 2048, 128, 5)]:
        a = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
        b = orc.construct(dim, n, leaf_size=leaf, grid_order=order)
        for x, y in zip(a.to_host().arrays(), b.to_host().arrays()):
            assert np.array_equal(x, y)
        x = ref.random_vector(n, 3)
        assert np.array_equal(a.hmv(x), b.hmv(x))
