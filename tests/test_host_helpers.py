"""CPU tests of the C ABI's host-side helpers (no GPU needed): the threaded
non-temporal staging copy and the symmetric-matrix mirror used by the host-buffer
paths (bgk_host_copy, bgk_host_mirror_lower, bgk_host_mirror_block)."""

import numpy as np
import pytest

from paper_2502_00356_b200 import _lib


@pytest.fixture(scope="module")
def L():
    return _lib.load_library()


@pytest.mark.parametrize("nbytes,off", [(0, 0), (1, 0), (17, 3), (4096, 0), (1 << 20, 8),
                                        ((1 << 22) + 13, 5)])
@pytest.mark.parametrize("threads", [1, 3, 16])
def test_host_copy(L, nbytes, off, threads):
    rng = np.random.default_rng(nbytes + off)
    src = rng.integers(0, 256, nbytes + off + 7, dtype=np.uint8)
    dst = np.zeros_like(src)
    rc = L.bgk_host_copy(dst.ctypes.data + off, src.ctypes.data + 7, nbytes, threads)
    assert rc == 0
    assert np.array_equal(dst[off:off + nbytes], src[7:7 + nbytes])
    assert not dst[:off].any() and not dst[off + nbytes:].any()


def test_host_copy_rejects_null(L):
    assert L.bgk_host_copy(None, None, 8, 1) != 0
    assert L.bgk_host_copy(None, None, 0, 1) == 0


@pytest.mark.parametrize("N,blocks,threads", [(1, [1], 1), (130, [64, 128, 130], 4),
                                              (1000, [1, 300, 301, 640, 1000], 7),
                                              (777, [777], 2)])
def test_host_mirror_lower_builds_symmetric_matrix(L, N, blocks, threads):
    rng = np.random.default_rng(N)
    low = np.tril(rng.random((N, N)))
    full = low + np.tril(low, -1).T
    out = low.copy()
    r0 = 0
    for r1 in blocks:
        out[r0:r1, r0:r1] = full[r0:r1, r0:r1]  # diagonal blocks arrive complete
        assert L.bgk_host_mirror_lower(out.ctypes.data, N, r0, r1, threads) == 0
        r0 = r1
    assert np.array_equal(out, full)


def test_host_mirror_block_ranges(L):
    N = 500
    rng = np.random.default_rng(5)
    a = rng.random((N, N))
    out = a.copy()
    assert L.bgk_host_mirror_block(out.ctypes.data, N, 300, 420, 40, 170, 3) == 0
    exp = a.copy()
    exp[40:170, 300:420] = a[300:420, 40:170].T
    assert np.array_equal(out, exp)
    # overlapping source / destination ranges are rejected, empty ranges are no-ops
    assert L.bgk_host_mirror_block(out.ctypes.data, N, 100, 200, 150, 250, 2) != 0
    assert L.bgk_host_mirror_block(out.ctypes.data, N, 100, 100, 0, 50, 2) == 0
    assert L.bgk_host_mirror_lower(out.ctypes.data, N, 0, 10, 2) == 0
