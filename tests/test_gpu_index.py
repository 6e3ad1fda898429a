"""Parity of the device fragment index (locate / start ranks / overlaps / greedy) with the
oracle -- the cases of proj/tests/test_fragment_index.cpp plus the overlap result contract
(overlap.hpp), through the C ABI."""
import numpy as np
import pytest

from tests.oracle_lib import concat_of

pytestmark = pytest.mark.gpu

WORKED = [b"GATT", b"ACA", b"GGT", b"GA", b"TTAC", b"AGGT"]
PAPER5 = [b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"]


def random_frags(rng, k, lo, hi, alphabet=(65, 67, 71, 84), probs=None):
    return [bytes(rng.choice(alphabet, int(rng.integers(lo, hi + 1)), p=probs).astype(np.uint8)) for _ in range(k)]


def shotgun(rng, G, k, lo, hi, alphabet=(65, 67, 71, 84)):
    genome = rng.choice(alphabet, G).astype(np.uint8)
    out = []
    for _ in range(k):
        ln = min(G, int(rng.integers(lo, hi + 1)))
        s = int(rng.integers(0, G - ln + 1))
        out.append(bytes(genome[s:s + ln]))
    return out


def test_locate_on_the_worked_instance(rq, ex):
    # test_fragment_index.cpp:33-45
    ix = rq.FragmentIndex(rq.make_fragment_set(WORKED, "dna"), ex)
    lo, hi = ix.locate_prefix_range(b"GA")
    assert hi - lo == 2
    assert sorted(ix.sa()[lo:hi].tolist()) == [0, 13]
    lo, hi = ix.locate_prefix_range(b"QQ")
    assert lo == hi


def test_single_fragment_exact(rq, ex):
    # test_fragment_index.cpp:47-53
    ix = rq.FragmentIndex(rq.make_fragment_set([b"GATT"], "dna"), ex)
    lo, hi = ix.locate_prefix_range(b"GATT")
    assert hi - lo == 1 and ix.sa()[lo] == 0


def test_structure_matches_oracle_on_paper_fragments(rq, ex, oracle):
    # test_fragment_index.cpp:129-138
    fs = rq.make_fragment_set(PAPER5, "generic_byte")
    ix = rq.FragmentIndex(fs, ex)
    wsa, wrank = oracle.build_sa(fs.concat)
    assert np.array_equal(ix.sa(), wsa) and np.array_equal(ix.rank(), wrank)
    assert np.array_equal(ix.start_rank_list(), oracle.start_rank_list(wrank, fs.starts))


def test_intervals_equal_the_oracle_binary_search(rq, ex, oracle):
    # test_fragment_index.cpp:55-80 (maximality) strengthened to exact equality, incl. absent
    # patterns (insertion point) and patterns with bytes outside the alphabet
    rng = np.random.default_rng(51)
    for it in range(60):
        dna = it % 2 == 0
        alpha = (65, 67, 71, 84) if dna else (97, 98)
        frags = random_frags(rng, 1 + int(rng.integers(0, 8)), 1, 6 if not dna else 30, alpha)
        fs = rq.make_fragment_set(frags, "dna" if dna else "generic_byte")
        ix = rq.FragmentIndex(fs, ex)
        sa = ix.sa()
        pats = [bytes(rng.choice(alpha, 1 + int(rng.integers(0, 4))).astype(np.uint8)) for _ in range(12)]
        pats += [b"QQ", b"B", b"AQ", b"z", b"!"]
        pats += [f[int(rng.integers(0, len(f))):] for f in frags]
        lo, hi = ix.locate_batch(pats)
        for p, l, h in zip(pats, lo, hi):
            assert (int(l), int(h)) == oracle.locate(fs.concat, sa, p), (frags, p)


def test_locate_with_directory_on_read_sets(rq, ex, oracle):
    rng = np.random.default_rng(52)
    frags = shotgun(rng, 20_000, 4_000, 40, 120)
    fs = rq.make_fragment_set(frags, "dna")
    ix = rq.FragmentIndex(fs, ex)
    sa = ix.sa()
    assert oracle.verify_sa(fs.concat, sa) == 0
    pats, fr, of = [], [], []
    for _ in range(3000):
        f = int(rng.integers(0, len(frags)))
        o = int(rng.integers(0, len(frags[f])))
        fr.append(f); of.append(o)
        pats.append(frags[f][o:])
    absent = [bytes(rng.choice([65, 67, 71, 84], int(rng.integers(1, 40))).astype(np.uint8)) for _ in range(500)]
    lo, hi = ix.locate_batch(pats + absent)
    rlo, rhi = ix.locate_residuals(fr, of)
    for t, p in enumerate(pats + absent):
        want = oracle.locate(fs.concat, sa, p)
        assert (int(lo[t]), int(hi[t])) == want
        if t < len(pats):
            assert (int(rlo[t]), int(rhi[t])) == want
    with pytest.raises(rq.OffsetOutOfRangeError):
        ix.locate_residuals([0], [len(frags[0])])


def _check_overlaps(rq, ex, oracle, frags, alphabet, min_ov):
    fs = rq.make_fragment_set(frags, alphabet)
    ix = rq.FragmentIndex(fs, ex)
    ov = ix.overlaps(min_ov)
    lens = fs.lengths()
    wi, wj, ww = oracle.overlap_list(fs.concat, fs.starts, lens, min_ov)
    assert np.array_equal(ov.i, wi) and np.array_equal(ov.j, wj) and np.array_equal(ov.w, ww), frags
    keep = oracle.absorb_contained(fs.concat, fs.starts, lens)
    assert np.array_equal(np.flatnonzero(ov.contained == 0).astype(np.uint32), keep), frags
    assert ov.queries == int(np.maximum(lens.astype(np.int64) - min_ov + 1, 0).sum())
    return fs, ix, ov


def test_overlap_lists_equal_the_dense_graph(rq, ex, oracle):
    """overlap.hpp:35-45: every non-zero weight, tau = 1, on adversarial small sets (tiny
    alphabets, duplicates, contained reads, mixed lengths)."""
    rng = np.random.default_rng(53)
    for it in range(120):
        if it % 3 == 0:
            frags = shotgun(rng, int(rng.integers(20, 80)), int(rng.integers(4, 16)), 3, 12, (65, 67))
        elif it % 3 == 1:
            frags = shotgun(rng, int(rng.integers(20, 80)), int(rng.integers(4, 16)), 5, 5)
        else:
            frags = random_frags(rng, int(rng.integers(2, 12)), 1, 9, (65, 67, 71, 84), [.6, .2, .1, .1])
        fs, ix, ov = _check_overlaps(rq, ex, oracle, frags, "dna", 1)
        dense = oracle.overlap_graph(fs.concat, fs.starts, fs.lengths())
        assert np.array_equal(ov.dense(len(frags)), dense)
    for it in range(30):  # generic alphabet
        frags = shotgun(rng, 40, int(rng.integers(3, 12)), 2, 10, (97, 98, 104))
        _check_overlaps(rq, ex, oracle, frags, "generic_byte", 1)


def test_overlap_lists_on_read_sets(rq, ex, oracle):
    rng = np.random.default_rng(54)
    _check_overlaps(rq, ex, oracle, shotgun(rng, 30_000, 6_000, 100, 100), "dna", 20)
    _check_overlaps(rq, ex, oracle, shotgun(rng, 8_000, 3_000, 30, 150), "dna", 16)
    _check_overlaps(rq, ex, oracle, shotgun(rng, 3_000, 2_000, 60, 60), "dna", 5)     # duplicates, deep coverage
    _check_overlaps(rq, ex, oracle, [b"ACGT" * 10] * 5 + [b"CGTA" * 10, b"A" * 30, b"A" * 31], "dna", 3)
    # more raw records per fragment than one warp sorts in shared memory (periodic duplicates: every
    # offset matches every copy): the global sort + unique route
    _check_overlaps(rq, ex, oracle, [b"ACGT" * 10] * 120 + [b"CGTA" * 10] * 40, "dna", 4)
    rng2 = np.random.default_rng(56)
    g = bytes(rng2.choice([65, 67, 71, 84], 300).astype(np.uint8))
    _check_overlaps(rq, ex, oracle, [g[s:s + 50] for s in rng2.integers(0, 250, 2000)], "dna", 10)   # 400x coverage


def test_overlap_search_with_tma_staging_and_with_ragged_long_reads(rq, oracle):
    """The TMA-staged form of the count kernel (overlap_stage = 1: a fragment's rank block and packed text
    brought into shared memory by double-buffered bulk copies) on a uniform read set, and on read sets
    whose fragments are too long (> 255) or too ragged for staging: same lists as the default form."""
    e = rq.Executor(0)
    try:
        e.set_option("overlap_stage", 1)
        rng = np.random.default_rng(58)
        _check_overlaps(rq, e, oracle, shotgun(rng, 20_000, 3_000, 100, 100), "dna", 20)
        rng = np.random.default_rng(59)
        _check_overlaps(rq, e, oracle, shotgun(rng, 30_000, 800, 200, 400), "dna", 25)     # mostly longer than 255
        _check_overlaps(rq, e, oracle, shotgun(rng, 10_000, 2_000, 1, 300), "dna", 3)      # every alignment of start and length
    finally:
        e.close()


def test_index_rejects_a_layout_that_is_not_a_fragment_set(rq, ex):
    """The C ABI takes raw (concat, starts) arrays: what make_fragment_set guarantees (sequence.hpp:103-124)
    is checked before anything is indexed with them."""
    text, starts = rq.synth_read_text(5_000, 50, 100)
    for bad in (starts[::-1].copy(),                                   # not ascending
                np.concatenate([starts[:50], starts[49:50], starts[50:]]),   # duplicate start (an empty fragment)
                np.concatenate([starts[:-1], [text.size + 10]]).astype(np.uint32),   # beyond the text
                (starts + 1).astype(np.uint32),                         # starts[0] != 0
                np.concatenate([[0], starts[1:] + 1]).astype(np.uint32)):   # fragments that do not end at a separator (checked on the device)
        with pytest.raises(ValueError):
            rq.FragmentIndex(rq.fragment_set_from_text(text, bad), ex)
    rq.FragmentIndex(rq.fragment_set_from_text(text, starts), ex).close()


def test_greedy_reconstruction_matches_the_oracle(rq, ex, oracle):
    """overlap.hpp:80-113 end to end: device overlaps + host merge == the reference loop."""
    # the paper's example: SPEC.md:300
    fs = rq.make_fragment_set(PAPER5, "generic_byte")
    sup, order = rq.greedy_superstring_with_order(fs, exec=ex)
    assert sup == b"abthatbabhhatbpaabtabhaabtpb" and order.tolist() == [0, 2, 1, 3, 4]
    rng = np.random.default_rng(55)
    for it in range(150):
        if it % 2:
            frags = shotgun(rng, int(rng.integers(20, 80)), int(rng.integers(4, 16)), 4, 14, (65, 67))
        else:
            frags = shotgun(rng, int(rng.integers(30, 120)), int(rng.integers(4, 20)), 8, 25)
        fs = rq.make_fragment_set(frags, "dna")
        ix = rq.FragmentIndex(fs, ex)
        want = oracle.greedy(fs.concat, fs.starts, fs.lengths())
        for tau in (1, 4):
            sup, order = rq.greedy_superstring_with_order(fs, ix, tau)
            assert sup == want[0] and order.tolist() == want[1].tolist(), (frags, tau)


def test_reconstruction_at_config1_scale_properties(rq, ex):
    """Config 1: every read is a substring of the reconstructed sequence, the order is a
    permutation of the kept reads, and a second run is byte-identical."""
    text, starts = rq.synth_read_text(200_000, 100, 20_000)
    fs = rq.fragment_set_from_text(text, starts)
    ix = rq.FragmentIndex(fs, ex)
    ov = ix.overlaps(20)
    sup, order = rq.greedy_superstring_from_overlaps(fs, ov)
    sup2, order2 = rq.greedy_superstring_from_overlaps(fs, ix.overlaps(20))
    assert sup == sup2 and np.array_equal(order, order2)
    kept = np.flatnonzero(ov.contained == 0)
    assert sorted(order.tolist()) == kept.tolist()
    for i in range(0, len(starts), 97):
        assert fs.bytes(i) in sup


def test_overlaps_at_config2_scale_properties(rq, ex):
    """BASELINE config 2 (920 000 reads of 150 bp, 30x): 120.5 M queries.  Size-independent
    properties of the overlap list: sorted unique (i, j), every sampled triple is a true
    suffix/prefix match and maximal (overlap_weight, overlap.hpp:16-23), the diagonal is absent,
    a second run is identical, and the sharded ranges concatenate to the same list."""
    text, starts = rq.synth_read_text(4_600_000, 150, 920_000)
    fs = rq.fragment_set_from_text(text, starts)
    ix = rq.FragmentIndex(fs, ex)
    ov = ix.overlaps(20)
    assert ov.queries == 920_000 * (150 - 20 + 1)
    key = (ov.i.astype(np.uint64) << np.uint64(32)) | ov.j.astype(np.uint64)
    assert np.all(key[1:] > key[:-1]) and not np.any(ov.i == ov.j)
    assert ov.w.min() >= 20 and ov.w.max() <= 150
    rng = np.random.default_rng(61)
    reads = text.reshape(-1, 151)[:, :150]
    for t in rng.integers(0, ov.i.size, 3000):
        a, b, w = reads[ov.i[t]], reads[ov.j[t]], int(ov.w[t])
        assert np.array_equal(a[150 - w:], b[:w])
        for longer in range(w + 1, 151):                      # no longer overlap exists
            assert not np.array_equal(a[150 - longer:], b[:longer])
    again = ix.overlaps(20, reuse_buffers=True)
    assert np.array_equal(again.i, ov.i) and np.array_equal(again.j, ov.j) and np.array_equal(again.w, ov.w)
    assert np.array_equal(again.contained, ov.contained)
    parts = [ix.overlaps(20, lo, hi) for lo, hi in ((0, 300_000), (300_000, 300_001), (300_001, 920_000))]
    assert np.array_equal(np.concatenate([p.i for p in parts]), ov.i)
    assert np.array_equal(np.concatenate([p.w for p in parts]), ov.w)
    ix.close()


def _uniform_contained(text, L):
    """absorb_contained (overlap.hpp:51-67) restated for reads of ONE length, without a suffix array:
    no read lies inside a longer one, so read i is dropped iff an equal read has a lower id."""
    reads = np.ascontiguousarray(text.reshape(-1, L + 1)[:, :L])
    rows = reads.view(np.dtype((np.void, L))).ravel()
    _, first, inv = np.unique(rows, return_index=True, return_inverse=True)
    return (first[inv.ravel()] != np.arange(rows.size)).astype(np.uint8)


def _exact_overlaps(rq, ex, oracle, G, L, k, tau, threads):
    text, starts = rq.synth_read_text(G, L, k)
    fs = rq.fragment_set_from_text(text, starts)
    ix = rq.FragmentIndex(fs, ex)
    ov = ix.overlaps(tau)
    ix.close()
    wi, wj, ww = oracle.overlap_list_fast(text, starts, fs.lengths(), tau, threads=threads, cap=40 * k)
    assert ov.i.size == wi.size, f"{ov.i.size} overlaps found, {wi.size} exist"
    assert np.array_equal(ov.i, wi) and np.array_equal(ov.j, wj) and np.array_equal(ov.w, ww)
    assert np.array_equal(ov.contained, _uniform_contained(text, L))
    return ov


def test_overlap_list_is_exact_at_config1_full_size(rq, ex, oracle):
    """BASELINE config 1 at full size (100 000 reads of 100 bp, tau = 20): the device list equals, triple
    for triple, the SA-free oracle (every (i, j) with overlap_weight >= 20 and its weight: completeness
    AND maximality, overlap.hpp:16-45), and the containment flags equal absorb_contained (:51-67)."""
    ov = _exact_overlaps(rq, ex, oracle, 1_000_000, 100, 100_000, 20, 16)
    assert ov.queries == 100_000 * 81


def test_overlap_list_is_exact_at_config2_full_size(rq, ex, oracle):
    """BASELINE config 2 at full size (920 000 reads of 150 bp, 30x, tau = 20; 120.5 M queries): set
    equality with the SA-free oracle -- no overlap missing, none spurious, every weight maximal -- and
    the containment flags."""
    ov = _exact_overlaps(rq, ex, oracle, 4_600_000, 150, 920_000, 20, 32)
    assert ov.queries == 920_000 * 131 and ov.i.size > 20_000_000


def test_reconstruction_at_config2_scale(rq, ex):
    """BASELINE config 2 end to end: device index + overlaps, host greedy merge
    (overlap.hpp:80-113 at scale).  With 30x error-free coverage of a random genome every merge is
    a true overlap, so the reconstructed sequence is the genome between the first and the last
    read: an exact substring of it, every kept read a substring of the result."""
    G = 4_600_000
    text, starts = rq.synth_read_text(G, 150, 920_000)
    fs = rq.fragment_set_from_text(text, starts)
    ix = rq.FragmentIndex(fs, ex)
    ov = ix.overlaps(20)
    sup, order = rq.greedy_superstring_from_overlaps(fs, ov)
    genome = rq.synth_random_dna(G, 1).tobytes()
    assert G - 200 < len(sup) <= G and sup in genome
    kept = np.flatnonzero(ov.contained == 0)
    assert sorted(order.tolist()) == kept.tolist()
    rng = np.random.default_rng(62)
    for i in rng.integers(0, 920_000, 500):
        assert fs.bytes(int(i)) in sup
    ix.close()


def test_cpp_shim_drop_in(tmp_path):
    """include/reseq_b200/reseq_cuda.hpp: the reference's KATs through the C++ value-semantics
    shim, standalone and -- where the reference headers exist -- against the reference itself."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    lib = root / "paper_1404_3456_b200" / "libreseq_cuda.so"
    variants = [[]]
    if Path("/root/reference/proj/include").is_dir():
        variants.append(["-DRESEQ_B200_WITH_REFERENCE", "-I/root/reference/proj/include", "-pthread"])
    for extra in variants:
        exe = tmp_path / f"shim{len(extra)}"
        subprocess.run(["g++", "-std=c++20", "-O1", *extra, "-I", str(root / "include"),
                        str(root / "tests" / "cpp" / "test_shim.cpp"), str(lib), f"-Wl,-rpath,{lib.parent}",
                        "-o", str(exe)], check=True)
        r = subprocess.run([str(exe)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr


def test_prefix_related_for_arbitrary_patterns(rq, ex, oracle, ref):
    """fragment_index::prefix_related(std::string_view), fragment_index.hpp:82-109: the golden
    vectors generated from the real reference, random patterns against the reference itself (when
    its shim is there) and the by-definition oracle -- including the early return that leaves
    prefixes_of unsorted (:91)."""
    import json
    from pathlib import Path
    golden = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
    checked = 0
    for inst in golden["index"]:
        frags = [bytes(f) for f in inst["fragments"]]
        fs = rq.make_fragment_set(frags, inst["alphabet"])
        ix = rq.FragmentIndex(fs, ex)
        got = ix.prefix_related_patterns([bytes(q["pattern"]) for q in inst["queries"]])
        for q, (a, e, x) in zip(inst["queries"], got):
            assert a.tolist() == q["prefixes"] and e.tolist() == q["extensions"] and x.tolist() == q["exact"], q
            checked += 1
        ix.close()
    assert checked > 50
    rng = np.random.default_rng(57)
    for it in range(12):
        frags = random_frags(rng, int(rng.integers(3, 40)), 1, 9, (65, 67, 71, 84), [.5, .3, .1, .1])
        fs = rq.make_fragment_set(frags, "dna")
        ix = rq.FragmentIndex(fs, ex)
        lens = fs.lengths()
        pats = [bytes(rng.choice([65, 67, 71, 84], int(rng.integers(1, 12)), p=[.5, .3, .1, .1]).astype(np.uint8))
                for _ in range(60)] + [f + b"A" for f in frags[:5]] + [f[:-1] + b"T" + b"G" for f in frags[:5] if len(f) > 1]
        got = ix.prefix_related_patterns(pats)
        rix = ref.index(frags, "dna") if ref is not None else None
        for p, (a, e, x) in zip(pats, got):
            oa, oe, ox = oracle.prefix_related(fs.concat, fs.starts, lens, p)
            if rix is not None:
                ra, re_, rx = rix.prefix_related(p)
                assert a.tolist() == ra.tolist() and e.tolist() == re_.tolist() and x.tolist() == rx.tolist(), (frags, p)
            full = sorted(a.tolist()) == oa.tolist() and e.tolist() == oe.tolist() and x.tolist() == ox.tolist()
            early = e.size == 0 and x.size == 0 and set(a.tolist()) <= set(oa.tolist())
            assert full or early, (frags, p)
        if rix is not None:
            rix.close()
        ix.close()
