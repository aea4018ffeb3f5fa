"""The hand-written radix sort and scans (csrc/primitives.cu) against numpy:
stable order on heavy ties, every digit range, sizes around tile edges."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sort(q, keys, vals, b0, b1):
    n = len(keys)
    ko = np.zeros(max(n, 1), np.uint64)
    vo = np.zeros(max(n, 1), np.uint64)
    q._check(q._lib().qvb_test_sort_pairs_u64(0, keys.ctypes.data, vals.ctypes.data, n, b0, b1,
                                               ko.ctypes.data, vo.ctypes.data))
    return ko[:n], vo[:n]


@pytest.mark.parametrize("n", [1, 31, 2047, 2048, 2049, 100_003, 3_000_000])
@pytest.mark.parametrize("b0,b1,span", [(0, 64, 1 << 64), (0, 8, 7), (3, 21, 1 << 21), (32, 64, 1 << 64),
                                         (0, 0, 5)])
def test_radix_sort_stable(qvb, n, b0, b1, span):
    rng = np.random.default_rng(n + b0)
    keys = rng.integers(0, min(span, 1 << 63), n, dtype=np.uint64)
    if span == 7:
        keys = rng.integers(0, 7, n, dtype=np.uint64)  # heavy ties
    vals = np.arange(n, dtype=np.uint64)
    ko, vo = _sort(qvb, keys, vals, b0, b1)
    mask = np.uint64(((1 << (b1 - b0)) - 1) << b0) if b1 > b0 else np.uint64(0)
    order = np.argsort(keys & mask, kind="stable")
    assert (vo == vals[order]).all()
    assert (ko == keys[order]).all()


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 1 << 20, 20_000_011])
def test_scans(qvb, n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 1000, n, dtype=np.uint32)
    out = np.zeros(n, np.uint64)
    qvb._check(qvb._lib().qvb_test_scan_u32(0, a.ctypes.data, n, 0, out.ctypes.data))
    cs = np.cumsum(a.astype(np.uint64))
    assert (out == cs - a).all()
    qvb._check(qvb._lib().qvb_test_scan_u32(0, a.ctypes.data, n, 1, out.ctypes.data))
    assert (out == (cs & 0xFFFFFFFF)).all()
