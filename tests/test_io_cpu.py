"""CPU: the containers' CRC-32 (h2b_crc32 == h2kit::crc32, crc32.cpp:6-20 ==
zlib's), including the chunk-parallel path with GF(2) CRC combination."""
import zlib

import numpy as np
import pytest

import paper_1902_01829_b200 as h2


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 65537])
def test_crc32_small(ref, n):
    b = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    c = h2.crc32(b)
    assert c == zlib.crc32(b)
    if ref is not None:
        assert c == ref.crc32(b)


def test_crc32_parallel_chunks():
    # > 64 MiB: per-chunk CRCs on several threads, combined (zlib crc32_combine)
    n = (3 << 26) + 12345
    b = np.random.default_rng(3).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert h2.crc32(b) == zlib.crc32(b)
