"""The store path's hand-written device primitives (csrc/gd_sort.cu) against
numpy: the stable LSD radix sort (u64 / u32 keys, with and without values,
partial bit ranges), the exclusive scan and the flagged-index select, at
sizes from empty to beyond one CTA's chunk and with heavy key repetition
(stability is what the store's slot semantics rely on)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 31, 32, 33, 255, 2048, 2049, 10_000, 333_337, 2_500_001]


@pytest.fixture(scope="module")
def L():
    from paper_2507_11094_b200 import _native as N

    return N


def _sort(N, keys, vals, end_bit):
    k = np.ascontiguousarray(keys.copy())
    v = None if vals is None else np.ascontiguousarray(vals.copy())
    N.check(N.lib().gd_prim_sort(k.dtype.itemsize, k.ctypes.data_as(C.c_void_p),
                                 None if v is None else v.ctypes.data_as(C.c_void_p), len(k), end_bit, 0))
    return k, v


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("kind", ["u64_pairs", "u64_keys", "u32_pairs"])
def test_radix_sort_is_a_stable_sort(L, n, kind):
    rng = np.random.default_rng(n + len(kind))
    bits = {"u64_pairs": 44, "u64_keys": 64, "u32_pairs": 22}[kind]
    hi = 1 << min(bits, 62)
    # few distinct keys on half the sizes: long runs of equal keys test stability
    span = 50 if n % 2 else hi
    dtype = np.uint32 if kind == "u32_pairs" else np.uint64
    keys = rng.integers(0, span, n, dtype=np.uint64).astype(dtype)
    if kind == "u64_keys" and n:
        keys[: n // 3] = np.uint64(2**63) + keys[: n // 3]  # the top bit too
    vals = None if kind == "u64_keys" else np.arange(n, dtype=np.int32)
    got_k, got_v = _sort(L, keys, vals, bits)
    order = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(got_k, keys[order])
    if vals is not None:
        np.testing.assert_array_equal(got_v, vals[order])  # equal keys keep their input order


def test_radix_sort_end_bit_limits_the_key_bits(L):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 40, 100_000, dtype=np.uint64)
    vals = np.arange(len(keys), dtype=np.int32)
    got_k, got_v = _sort(L, keys, vals, 16)  # only the low 16 bits are sorted on
    order = np.argsort(keys & np.uint64(0xFFFF), kind="stable")
    np.testing.assert_array_equal(got_v, vals[order])
    np.testing.assert_array_equal(got_k, keys[order])


@pytest.mark.parametrize("n", SIZES)
def test_scan_and_select(L, n):
    rng = np.random.default_rng(n)
    x = rng.integers(-5, 1000, n).astype(np.int64)
    flags = (rng.random(n) < 0.3).astype(np.uint8)
    out = np.zeros(max(n, 1), np.int64)
    idx = np.zeros(max(n, 1), np.int32)
    cnt = C.c_int64()
    L.check(L.lib().gd_prim_scan_select(x.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                        flags.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p), n,
                                        C.byref(cnt), 0))
    np.testing.assert_array_equal(out[:n], np.concatenate([[0], np.cumsum(x)[:-1]]) if n else out[:0])
    want = np.flatnonzero(flags)
    assert cnt.value == len(want)
    np.testing.assert_array_equal(idx[:len(want)], want)
