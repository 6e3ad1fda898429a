"""Pins the oracle (oracle/restate.cpp): the reference's own KATs, the golden vectors
generated from the real reference (tests/golden/golden.json), and -- where
oracle/_ref/libreseq_ref.so is loadable -- the real reference itself.  CPU only."""
import json
from pathlib import Path

import numpy as np
import pytest

from tests.oracle_lib import concat_of

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def b(lst):
    return bytes(lst)


# ---- the reference's KATs (proj/tests/*.cpp) --------------------------------------------

def test_sa_kats(oracle):
    assert oracle.build_sa(b"banana")[0].tolist() == [5, 3, 1, 0, 4, 2]         # test_suffix_array.cpp:11
    assert oracle.build_sa(b"aaa")[0].tolist() == [2, 1, 0]                      # :12
    assert oracle.build_sa(b"")[0].size == 0                                     # :13
    assert oracle.build_sa(b"GA\0TT\0")[0].tolist() == [2, 5, 1, 0, 4, 3]        # :41-43
    sa, rank = oracle.build_sa(b"mississippi")
    assert np.array_equal(rank[sa], np.arange(11, dtype=np.uint32))              # :16-21


def test_primitive_kats(oracle):
    st, out = oracle.exclusive_scan([3, 1, 7, 0])
    assert st == 0 and out.tolist() == [0, 3, 4, 11]                             # test_parallel.cpp:53
    assert oracle.exclusive_scan([0xFFFFFFFF, 1])[0] == 3                        # :62 (overflow)
    st, out = oracle.exclusive_scan([0xFFFFFFFE, 1])
    assert st == 0 and out.tolist() == [0, 0xFFFFFFFE]                           # :64-65
    assert oracle.split_by_bit([5, 2, 7, 4], None, 0)[0].tolist() == [2, 4, 5, 7]  # :88
    k, p = oracle.split_by_bit([1, 1, 0, 0], [10, 11, 12, 13], 0)
    assert k.tolist() == [0, 0, 1, 1] and p.tolist() == [12, 13, 10, 11]         # :90-93
    assert oracle.stable_sort([170, 45, 75, 90, 2, 24, 802, 66], None)[0].tolist() == \
        [2, 24, 45, 66, 75, 90, 170, 802]                                        # :126-128


def test_index_kats(oracle):
    frags = [b"GATT", b"ACA", b"GGT", b"GA", b"TTAC", b"AGGT"]
    concat, starts, lens = concat_of(frags)
    sa, rank = oracle.build_sa(concat)
    lo, hi = oracle.locate(concat, sa, b"GA")
    assert hi - lo == 2 and sorted(sa[lo:hi].tolist()) == [0, 13]                # test_fragment_index.cpp:37-41
    lo, hi = oracle.locate(concat, sa, b"QQ")
    assert lo == hi                                                              # :43-44
    a, e, x = oracle.prefix_related(concat, starts, lens, b"TT")
    assert a.size == 0 and e.tolist() == [4] and x.size == 0                     # :87-90
    assert oracle.prefix_related(concat, starts, lens, b"GGT")[2].tolist() == [2]  # :92-93
    concat, starts, lens = concat_of([b"ab", b"cd", b"efgh", b"abcdef", b"gh"])
    a, e, x = oracle.prefix_related(concat, starts, lens, b"cdef")
    assert a.tolist() == [1] and e.size == 0 and x.size == 0                     # :96-103


def test_overlap_and_greedy_spec_examples(oracle):
    assert oracle.overlap_weight(b"abthatb", b"tbabhhatbpaa") == 2
    assert oracle.overlap_weight(b"hatbpaab", b"paabtabh") == 4
    assert oracle.overlap_weight(b"AAA", b"TTT") == 0
    concat, starts, lens = concat_of([b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"])
    sup, order = oracle.greedy(concat, starts, lens)
    assert sup == b"abthatbabhhatbpaabtabhaabtpb" and len(sup) == 28
    assert order.tolist() == [0, 2, 1, 3, 4]


def test_checksum_definition(oracle):
    # FNV-1a-64 offset basis / prime (bench.hpp:31-38): empty input hashes to the basis
    assert oracle.fnv1a64(b"") == 14695981039346656037
    assert oracle.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert oracle.checksum_u32([0x04030201]) == oracle.fnv1a64(bytes([1, 2, 3, 4]))  # little-endian bytes


# ---- golden vectors from the real reference ------------------------------------------------

def test_golden_suffix_arrays(oracle):
    for case in GOLDEN["suffix_arrays"]:
        sa, rank = oracle.build_sa(b(case["text"]))
        assert sa.tolist() == case["sa"]
        assert oracle.verify_sa(b(case["text"]), sa) == 0
        if len(case["sa"]) > 2:
            bad = list(case["sa"])
            bad[0], bad[1] = bad[1], bad[0]
            assert oracle.verify_sa(b(case["text"]), bad) != 0   # the verifier does reject


def test_golden_primitives(oracle):
    for c in GOLDEN["primitives"]:
        k = np.array(c["keys"], np.uint32)
        p = np.arange(k.size, dtype=np.uint32)
        sk, sp = oracle.split_by_bit(k, p, c["bit"])
        assert sk.tolist() == c["split_keys"] and sp.tolist() == c["split_payload"]
        rk, rp = oracle.stable_sort(k, p)
        assert rk.tolist() == c["sorted_keys"] and rp.tolist() == c["sorted_payload"]
        st, out = oracle.exclusive_scan(c["scan_in"])
        assert st == 0 and out.tolist() == c["scan_out"]


def test_golden_index(oracle):
    for c in GOLDEN["index"]:
        frags = [b(f) for f in c["fragments"]]
        concat, starts, lens = concat_of(frags)
        sa, rank = oracle.build_sa(concat)
        assert sa.tolist() == c["sa"]
        assert oracle.start_rank_list(rank, starts).tolist() == c["start_rank_list"]
        for q in c["queries"]:
            pat = b(q["pattern"])
            assert oracle.locate(concat, sa, pat) == (q["lo"], q["hi"])
            a, e, x = oracle.prefix_related(concat, starts, lens, pat)
            if q["lo"] != q["hi"] or not q["prefixes"]:
                # (fragment_index.hpp:91: for an absent pattern the reference returns early with
                # an unsorted prefix list; the by-definition lists are compared otherwise)
                assert sorted(q["prefixes"]) == a.tolist()
            if q["lo"] != q["hi"]:
                assert q["extensions"] == e.tolist() and q["exact"] == x.tolist()


def test_golden_overlaps_and_greedy(oracle):
    for w in GOLDEN["overlap_weight_spec"]:
        assert oracle.overlap_weight(b(w["a"]), b(w["b"])) == w["w"]
    for c in GOLDEN["overlap"]:
        frags = [b(f) for f in c["fragments"]]
        concat, starts, lens = concat_of(frags)
        dense = oracle.overlap_graph(concat, starts, lens)
        assert dense.tolist() == c["weight"]
        oi, oj, ow = oracle.overlap_list(concat, starts, lens, 1)
        sparse = np.zeros_like(dense)
        sparse[oi, oj] = ow
        assert np.array_equal(sparse, dense)
        assert oracle.absorb_contained(concat, starts, lens).tolist() == c["kept"]
        sup, order = oracle.greedy(concat, starts, lens)
        assert list(sup) == c["superstring"] and order.tolist() == c["order"]


def test_fast_overlap_oracle_equals_the_definitional_one(oracle, ref):
    """orc_overlap_list_fast (the checker of the config-size GPU tests) against orc_overlap_list, the
    dense graph restatement and -- where it was compiled -- the reference's build_overlap_graph
    (overlap.hpp:26-45): golden instances, random read sets with repeats, duplicates, containments,
    mixed lengths and periodic reads (several match lengths per pair), every threshold, 1..5 threads."""
    for c in GOLDEN["overlap"]:
        frags = [b(f) for f in c["fragments"]]
        concat, starts, lens = concat_of(frags)
        oi, oj, ow = oracle.overlap_list_fast(concat, starts, lens, 1, threads=3)
        sparse = np.zeros((len(frags), len(frags)), np.uint32)
        sparse[oi, oj] = ow
        assert sparse.tolist() == c["weight"]
    rng = np.random.default_rng(77)
    for it in range(60):
        alpha = [[65, 67, 71, 84], [65, 67], [65]][it % 3]
        G = int(rng.integers(30, 400))
        genome = rng.choice(alpha, G).astype(np.uint8)
        frags = []
        for _ in range(int(rng.integers(2, 60))):
            ln = min(G, int(rng.integers(1, 40)))
            s0 = int(rng.integers(0, G - ln + 1))
            frags.append(bytes(genome[s0:s0 + ln]))
        frags += frags[:2]                                  # duplicates
        concat, starts, lens = concat_of(frags)
        dense = oracle.overlap_graph(concat, starts, lens)
        if ref is not None and it % 4 == 0:
            assert np.array_equal(ref.overlap_graph(frags), dense)
        for tau in (1, 2, 5, 20):
            a = oracle.overlap_list(concat, starts, lens, tau)
            f = oracle.overlap_list_fast(concat, starts, lens, tau, threads=1 + it % 5)
            assert all(np.array_equal(x, y) for x, y in zip(a, f)), (frags, tau)
            want = np.argwhere(dense >= tau)
            assert np.array_equal(np.stack([f[0], f[1]], 1).astype(np.int64), want) and np.array_equal(f[2], dense[dense >= tau])
    # the text generator used by bench.py's reference arm
    if ref is not None:
        assert np.array_equal(oracle.make_read_text(5000, 60, 300), ref.make_read_text(5000, 60, 300))


# ---- the real reference, where it could be compiled -------------------------------------------

def test_against_the_reference_itself(oracle, ref):
    if ref is None:
        pytest.skip("oracle/_ref not built here (needs /root/reference)")
    rng = np.random.default_rng(7)
    for it in range(40):
        parts = [bytes(rng.choice([65, 67, 71, 84] if it % 2 else [97, 98], int(rng.integers(1, 25))).astype(np.uint8))
                 + (b"\0" if rng.random() < .8 else b"") for _ in range(int(rng.integers(1, 9)))]
        t = b"".join(parts)
        rsa, rrank = ref.build_naive(t)
        st, psa, prank = ref.build_parallel(t, 3, 50)
        osa, orank = oracle.build_sa(t)
        assert st == 0 and np.array_equal(rsa, osa) and np.array_equal(psa, osa) and np.array_equal(prank, orank)
        for _ in range(5):
            i, j = (int(x) for x in rng.integers(0, len(t), 2))
            assert bool(ref.lib.ref_suffix_less(t, len(t), i, j)) == oracle.suffix_less(t, i, j)
    for it in range(20):
        frags = []
        G = int(rng.integers(20, 70))
        genome = rng.choice([65, 67, 71, 84] if it % 2 else [65, 67], G).astype(np.uint8)
        for _ in range(int(rng.integers(2, 12))):
            ln = min(G, int(rng.integers(2, 14)))
            s0 = int(rng.integers(0, G - ln + 1))
            frags.append(bytes(genome[s0:s0 + ln]))
        concat, starts, lens = concat_of(frags)
        assert np.array_equal(ref.overlap_graph(frags), oracle.overlap_graph(concat, starts, lens))
        rs, ro = ref.greedy(frags)
        os_, oo = oracle.greedy(concat, starts, lens)
        assert rs == os_ and ro.tolist() == oo.tolist()
        assert ref.absorb_contained(frags).tolist() == oracle.absorb_contained(concat, starts, lens).tolist()
        ix = ref.index(frags, "dna", builder=it % 2)
        _, _, sa, rank, srl = ix.arrays()
        assert np.array_equal(srl, oracle.start_rank_list(rank, starts))
        for f in frags:
            p = f[int(rng.integers(0, len(f))):]
            assert ix.locate(p) == oracle.locate(concat, sa, p)
            a, e, x = ix.prefix_related(p)
            oa, oe, ox = oracle.prefix_related(concat, starts, lens, p)
            assert a.tolist() == oa.tolist() and e.tolist() == oe.tolist() and x.tolist() == ox.tolist()
        ix.close()
    k = rng.integers(0, 1 << 32, 3000, dtype=np.uint64).astype(np.uint32)
    p = np.arange(3000, dtype=np.uint32)
    for fn in (lambda: ref.radix_sort(k, p, 4, 257), lambda: ref.chunked_radix_sort(k, p, 4, 4, 300),
               lambda: ref.chunked_radix_sort(k, p, 8, 2, 64)):
        st, rk, rp = fn()
        ok, op = oracle.stable_sort(k, p)
        assert st == 0 and np.array_equal(rk, ok) and np.array_equal(rp, op)
    assert ref.chunked_radix_sort(k, p, 0)[0] == 1 and ref.chunked_radix_sort(k, p, 9)[0] == 1  # invalid_argument
    v = (k % 5000).astype(np.uint32)
    st, rs = ref.exclusive_scan(v, 3, 100)
    assert st == 0 and np.array_equal(rs, oracle.exclusive_scan(v)[1])
    assert ref.exclusive_scan([0xFFFFFFFF, 1])[0] == 3
    assert ref.checksum_u32(k) == oracle.checksum_u32(k)
    assert ref.fnv1a64(b"reseq") == oracle.fnv1a64(b"reseq")


def test_split_plan_restatement_against_the_reference(oracle, ref):
    """test_parallel.cpp:109-123 (seed 29 property) on the restatement, and equality with the
    reference's own detail::split_destinations / phase_is_sorted where it could be built."""
    rng = np.random.default_rng(29)
    for it in range(60):
        n = int(rng.integers(1, 801))
        keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        if it % 5 == 0:
            keys &= np.uint32(0xFF)
        bit = int(rng.integers(0, 32))
        d, tof = oracle.split_destinations(keys, bit)
        assert tof == int((((keys >> np.uint32(bit)) & 1) ^ 1).sum())
        assert np.array_equal(np.sort(d), np.arange(n, dtype=np.uint32))
        ko, _ = oracle.split_by_bit(keys, None, bit)
        out = np.empty_like(keys)
        out[d] = keys
        assert np.array_equal(out, ko)                      # the plan IS the split (radix_sort.hpp:126-139)
        assert oracle.is_sorted(keys) == bool(np.all(keys[:-1] <= keys[1:]))
        assert oracle.is_sorted(np.sort(keys))
        if ref is not None:
            rd, rtof = ref.split_destinations(keys, bit, workers=1 + it % 4, chunk=64)
            assert rtof == tof and np.array_equal(rd, d)
            assert ref.is_sorted(keys, workers=2, chunk=100) == oracle.is_sorted(keys)
    d, tof = oracle.split_destinations(np.zeros(0, np.uint32), 3)
    assert d.size == 0 and tof == 0
