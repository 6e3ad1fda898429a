"""Parity of the device L0 primitives with the oracle -- the cases of
proj/tests/test_parallel.cpp re-expressed against the C ABI (all through
include/reseq_cuda.h via paper_1404_3456_b200.api)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U32 = np.uint32


def rand_keys(rng, n, small):
    k = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(U32)
    if small:
        k &= U32(0x3F)
    return k, np.arange(n, dtype=U32)


# ---- exclusive_scan (test_parallel.cpp:52-84) ---------------------------------------

def test_scan_basics(rq, ex):
    assert rq.exclusive_scan([3, 1, 7, 0], ex).tolist() == [0, 3, 4, 11]
    assert rq.exclusive_scan([], ex).size == 0
    assert rq.exclusive_scan(np.ones(1024, U32), ex).tolist() == list(range(1024))


def test_scan_overflow_is_an_error_not_a_wrap(rq, ex):
    with pytest.raises(rq.ScanOverflowError):
        rq.exclusive_scan([0xFFFFFFFF, 1], ex)
    assert rq.exclusive_scan([0xFFFFFFFE, 1], ex).tolist() == [0, 0xFFFFFFFE]


def test_scan_is_linear_and_matches_oracle(rq, ex, oracle):
    rng = np.random.default_rng(17)
    for _ in range(20):
        n = int(rng.integers(0, 3000))
        a = rng.integers(0, 1000, n).astype(U32)
        b = rng.integers(0, 1000, n).astype(U32)
        sa, sb, sab = rq.exclusive_scan(a, ex), rq.exclusive_scan(b, ex), rq.exclusive_scan(a + b, ex)
        assert np.array_equal(sab, sa + sb)
        st, want = oracle.exclusive_scan(a)
        assert st == 0 and np.array_equal(sa, want)


@pytest.mark.parametrize("n", [1, 15, 16, 17, 4095, 4096, 4097, 8191, 1 << 20, 5_000_003])
def test_scan_sizes_across_tile_boundaries(rq, ex, n):
    rng = np.random.default_rng(n)
    v = rng.integers(0, 400, n).astype(U32)
    want = np.concatenate(([0], np.cumsum(v, dtype=np.uint64)[:-1])).astype(U32)
    assert np.array_equal(rq.exclusive_scan(v, ex), want)


def test_scan_overflow_large(rq, ex):
    v = np.full(1 << 20, 5000, U32)  # total 5.2e9 > 2^32
    with pytest.raises(rq.ScanOverflowError):
        rq.exclusive_scan(v, ex)


# ---- split_by_bit (test_parallel.cpp:86-123) -------------------------------------------

def test_split_examples(rq, ex, oracle):
    k, _ = rq.split_by_bit([5, 2, 7, 4], None, 0, ex)
    assert k.tolist() == [2, 4, 5, 7]
    k, p = rq.split_by_bit([1, 1, 0, 0], [10, 11, 12, 13], 0, ex)
    assert k.tolist() == [0, 0, 1, 1] and p.tolist() == [12, 13, 10, 11]
    k, p = rq.split_by_bit([6, 3, 6, 2], [0, 1, 2, 3], 1, ex)
    wk, wp = oracle.split_by_bit([6, 3, 6, 2], [0, 1, 2, 3], 1)
    assert np.array_equal(k, wk) and np.array_equal(p, wp)
    k, p = rq.split_by_bit([], [], 3, ex)
    assert k.size == 0 and p.size == 0
    k, p = rq.split_by_bit([9], [4], 0, ex)
    assert k.tolist() == [9] and p.tolist() == [4]


def test_split_matches_the_stable_partition_oracle(rq, ex, oracle):
    rng = np.random.default_rng(23)
    for it in range(60):
        k, p = rand_keys(rng, int(rng.integers(0, 2500)), it % 2)
        bit = int(rng.integers(0, 32))
        gk, gp = rq.split_by_bit(k, p, bit, ex)
        wk, wp = oracle.split_by_bit(k, p, bit)
        assert np.array_equal(gk, wk) and np.array_equal(gp, wp)


def test_split_large_and_bit_validation(rq, ex, oracle):
    rng = np.random.default_rng(29)
    k, p = rand_keys(rng, 300_001, False)
    for bit in (0, 17, 31):
        gk, gp = rq.split_by_bit(k, p, bit, ex)
        wk, wp = oracle.split_by_bit(k, p, bit)
        assert np.array_equal(gk, wk) and np.array_equal(gp, wp)
    with pytest.raises(ValueError):
        rq.split_by_bit(k, p, 32, ex)


# ---- radix_sort / chunked_radix_sort (test_parallel.cpp:125-170) ------------------------

def test_radix_examples(rq, ex):
    k, p = rq.radix_sort([170, 45, 75, 90, 2, 24, 802, 66], None, ex)
    assert k.tolist() == [2, 24, 45, 66, 75, 90, 170, 802] and p.size == 0
    k, _ = rq.radix_sort([], None, ex)
    assert k.size == 0
    k, p = rq.radix_sort([7], [0], ex)
    assert k.tolist() == [7] and p.tolist() == [0]


def test_sorts_match_the_comparison_oracle(rq, ex, oracle):
    rng = np.random.default_rng(31)
    for it in range(40):
        k, p = rand_keys(rng, int(rng.integers(0, 4000)), it % 3 == 0)
        wk, wp = oracle.stable_sort(k, p)
        for fn in (lambda: rq.radix_sort(k, p, ex),
                   lambda: rq.chunked_radix_sort(k, p, ex, 1),
                   lambda: rq.chunked_radix_sort(k, p, ex, 4),
                   lambda: rq.chunked_radix_sort(k, p, ex, 8)):
            gk, gp = fn()
            assert np.array_equal(gk, wk) and np.array_equal(gp, wp)


@pytest.mark.parametrize("n", [2, 31, 32, 33, 4095, 4096, 4097, 12289, 20000, 1 << 18])
def test_sort_sizes_with_and_without_payload(rq, ex, oracle, n):
    rng = np.random.default_rng(37 + n)
    k, p = rand_keys(rng, n, False)
    wk, wp = oracle.stable_sort(k, p)
    gk, gp = rq.radix_sort(k, p, ex)
    assert np.array_equal(gk, wk) and np.array_equal(gp, wp)
    gk, gp = rq.radix_sort(k, None, ex)
    assert np.array_equal(gk, wk) and gp.size == 0
    gk, gp = rq.chunked_radix_sort(k, p, ex, 5)
    assert np.array_equal(gk, wk) and np.array_equal(gp, wp)


def test_sort_stability_on_heavy_duplicates(rq, ex, oracle):
    rng = np.random.default_rng(41)
    n = 200_000
    k = rng.integers(0, 7, n).astype(U32) * U32(0x01010101)
    p = np.arange(n, dtype=U32)
    wk, wp = oracle.stable_sort(k, p)
    gk, gp = rq.radix_sort(k, p, ex)
    assert np.array_equal(gk, wk) and np.array_equal(gp, wp)
    # already sorted / reverse sorted / constant
    for arr in (np.arange(n, dtype=U32), np.arange(n, 0, -1, dtype=U32), np.full(n, 77, U32)):
        wk, wp = oracle.stable_sort(arr, p)
        gk, gp = rq.radix_sort(arr, p, ex)
        assert np.array_equal(gk, wk) and np.array_equal(gp, wp)


def test_bench_input_fingerprint(rq, ex, oracle):
    """make_random_keys(1<<20, 1) -> checksum_keys == 91396105105168530 (BASELINE.md section 2,
    measured with the reference's radix_sort and chunked_radix_sort)."""
    k, p = rq.synth_random_keys(1 << 20, 1)
    gk, gp = rq.radix_sort(k, p, ex)
    assert oracle.checksum_keys(gk, gp) == 91396105105168530
    gk, gp = rq.chunked_radix_sort(k, p, ex, 4)
    assert oracle.checksum_keys(gk, gp) == 91396105105168530


def test_chunked_digit_width_is_validated(rq, ex):
    with pytest.raises(ValueError):
        rq.chunked_radix_sort([1, 2], None, ex, 0)
    with pytest.raises(ValueError):
        rq.chunked_radix_sort([1, 2], None, ex, 9)


def test_split_destinations_and_is_sorted(rq, ex, oracle):
    """radix_sort.hpp:35-66 (Alg. 1's dataflow and the early-exit test) through the C ABI."""
    rng = np.random.default_rng(30)
    for n in [1, 2, 31, 32, 33, 2047, 2048, 2049, 100_003, 1_000_000]:
        keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        for bit in (0, 7, 31, int(rng.integers(0, 32))):
            d, tof = rq.split_destinations(keys, bit, ex)
            wd, wtof = oracle.split_destinations(keys, bit)
            assert tof == wtof and np.array_equal(d, wd), (n, bit)
            ko, _ = rq.split_by_bit(keys, None, bit, ex)
            out = np.empty_like(keys)
            out[d] = keys
            assert np.array_equal(out, ko)
        assert rq.is_sorted(keys, ex) == oracle.is_sorted(keys)
        s = np.sort(keys)
        assert rq.is_sorted(s, ex)
        if n > 2:
            s[n // 2], s[n // 2 - 1] = s[n // 2 - 1], s[n // 2] + np.uint32(1) if s[n // 2] < 2**32 - 1 else s[n // 2]
            assert rq.is_sorted(s, ex) == oracle.is_sorted(s)
    d, tof = rq.split_destinations(np.zeros(0, np.uint32), 0, ex)
    assert d.size == 0 and tof == 0 and rq.is_sorted(np.zeros(0, np.uint32), ex)
    with pytest.raises(ValueError):
        rq.split_destinations(np.zeros(4, np.uint32), 32, ex)
