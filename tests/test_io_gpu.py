"""GPU: container I/O (h2b_matrix_save / h2b_matrix_load == h2kit::save / load,
io.hpp:183-282).  Files written from HBM are byte-identical to the reference's
own containers of the same matrix; the reference reads ours and we read its;
corrupt / truncated / foreign files fail with the reference's IOError texts."""
import os

import numpy as np
import pytest

from conftest import rel_err

import paper_1902_01829_b200 as h2

pytestmark = pytest.mark.gpu

CASES = [(2, 4096, 8), (3, 2048, 3), (2, 1 << 12, 4)]


@pytest.mark.parametrize("dim,n,order", CASES)
def test_save_is_byte_identical_to_reference(gpu, ref, tmp_path, dim, n, order):
    """The reference's matrix uploaded to HBM and saved from there == the
    reference's own save, byte for byte."""
    R = ref.construct(dim, n, grid_order=order)
    A = h2.H2Matrix.from_host(R.to_host())
    ours, theirs = tmp_path / "ours.h2", tmp_path / "ref.h2"
    A.save(ours, build_info=dict(dim=dim, seed=1, perturbation=0.25, ell=0.1 if dim == 2 else 0.2,
                                 eta=2.0, grid_order=order))
    R.save(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.parametrize("dim,n,order", CASES)
def test_reference_reads_device_built_container(gpu, ref, tmp_path, dim, n, order):
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    path = tmp_path / "dev.h2"
    A.save(path)
    R = ref.load(str(path))
    x = np.random.default_rng(3).random(n)
    assert rel_err(R.hmv(x), h2.hmv(A, x)) <= 1e-12
    # structure, ranks and BuildInfo are the reference construct's
    R0 = ref.construct(dim, n, grid_order=order)
    assert R.layout()[0].tolist() == R0.layout()[0].tolist()
    assert R.layout()[1].tolist() == R0.layout()[1].tolist()


@pytest.mark.parametrize("dim,n,order", CASES)
def test_load_reference_container(gpu, ref, tmp_path, dim, n, order):
    R = ref.construct(dim, n, grid_order=order)
    path = tmp_path / "ref.h2"
    R.save(str(path))
    A = h2.H2Matrix.load(path)
    assert A.build_info["dim"] == dim and A.build_info["grid_order"] == order
    x = np.random.default_rng(2).random(n)
    assert rel_err(h2.hmv(A, x), R.hmv(x)) <= 1e-12


def test_compressed_roundtrip_through_reference(gpu, ref, tmp_path):
    n = 1 << 13
    A = h2.H2Matrix.construct(2, n, grid_order=8)
    h2.compress(A, 1e-7)
    x = np.random.default_rng(5).random(n)
    y = h2.hmv(A, x)
    path = tmp_path / "c.h2"
    A.save(path)
    R = ref.load(str(path))
    assert rel_err(R.hmv(x), y) <= 1e-12
    B = h2.H2Matrix.load(path)
    assert B.info().ranks[:B.info().depth + 1] == A.info().ranks[:A.info().depth + 1]
    assert rel_err(h2.hmv(B, x), y) <= 1e-14
    assert B.memory_footprint() == A.memory_footprint()
    # and the reference writes the same bytes back
    path2 = tmp_path / "c2.h2"
    R.save(str(path2))
    assert path2.read_bytes() == path.read_bytes()


def test_build_info_override(gpu, tmp_path):
    A = h2.H2Matrix.construct(2, 4096)
    info = dict(dim=2, seed=7, perturbation=0.5, ell=0.3, eta=1.5, grid_order=8)
    A.save(tmp_path / "a.h2", build_info=info)
    B = h2.H2Matrix.load(tmp_path / "a.h2")
    assert B.build_info == pytest.approx(info)


def test_container_errors(gpu, tmp_path):
    A = h2.H2Matrix.construct(2, 4096)
    good = tmp_path / "g.h2"
    A.save(good)
    data = bytearray(good.read_bytes())
    with pytest.raises(h2.H2bIOError, match="cannot open"):
        h2.H2Matrix.load(tmp_path / "missing.h2")
    with pytest.raises(h2.H2bIOError, match="cannot open for writing"):
        A.save(tmp_path / "no_such_dir" / "x.h2")
    bad = tmp_path / "b.h2"
    bad.write_bytes(b"XXXX" + bytes(data[4:]))
    with pytest.raises(h2.H2bIOError, match="not a valid container"):
        h2.H2Matrix.load(bad)
    v2 = bytearray(data)
    v2[4] = 2
    bad.write_bytes(bytes(v2))
    with pytest.raises(h2.H2bIOError, match="unsupported container version"):
        h2.H2Matrix.load(bad)
    p4 = bytearray(data)
    p4[6] = 4
    bad.write_bytes(bytes(p4))
    with pytest.raises(h2.H2bIOError, match="precision mismatch"):
        h2.H2Matrix.load(bad)
    flip = bytearray(data)
    flip[len(flip) // 2] ^= 0x40
    bad.write_bytes(bytes(flip))
    with pytest.raises(h2.H2bIOError, match="checksum mismatch"):
        h2.H2Matrix.load(bad)
    bad.write_bytes(bytes(data[: len(data) - 10]))
    with pytest.raises(h2.H2bIOError, match="container truncated"):
        h2.H2Matrix.load(bad)
    bad.write_bytes(bytes(data[:9]))
    with pytest.raises(h2.H2bIOError, match="missing section header"):
        h2.H2Matrix.load(bad)
    os.remove(bad)


def test_big_blocks_roundtrip_with_reference(gpu, ref, tmp_path):
    """Ranks / leaf sizes above 64 (leaf 128, rank 100) through the container:
    the reference reads our device-built file and we read the reference's, with
    the same mat-vec (k_hmv_big.cu on our side)."""
    dim, n, leaf, order = 2, 1 << 13, 128, 10
    A = h2.H2Matrix.construct(dim, n, leaf_size=leaf, grid_order=order)
    p1 = tmp_path / "dev_big.h2"
    A.save(p1)
    R = ref.load(str(p1))
    x = np.random.default_rng(31).random(n)
    assert rel_err(R.hmv(x), h2.hmv(A, x)) <= 1e-12
    R2 = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
    p2 = tmp_path / "ref_big.h2"
    R2.save(str(p2))
    B = h2.H2Matrix.load(p2)
    assert rel_err(h2.hmv(B, x), R2.hmv(x)) <= 1e-12
    U = h2.H2Matrix.from_host(R2.to_host())  # uploaded to HBM and saved from there
    p3 = tmp_path / "up_big.h2"
    U.save(p3, build_info=dict(dim=dim, seed=1, perturbation=0.25, ell=0.1, eta=2.0, grid_order=order))
    assert p3.read_bytes() == p2.read_bytes()
