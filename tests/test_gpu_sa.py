"""Parity of the device suffix-array builder with the oracle -- the cases of
proj/tests/test_suffix_array.cpp plus read-set shaped and adversarial texts, through
reseq_cuda_build_sa."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


_doubling = {}


def doubling_executor(rq):
    """A second context forced onto pure prefix doubling (sa_text_rounds = 0), so both
    engines of the builder are checked on every small case."""
    if "ex" not in _doubling:
        e = rq.Executor(0)
        e.set_option("sa_text_rounds", 0)
        _doubling["ex"] = e
    return _doubling["ex"]


def global_doubling_executor(rq):
    """Pure prefix doubling with every round through the global digit passes (the local shared-memory
    form switched off)."""
    if "gd" not in _doubling:
        e = rq.Executor(0)
        e.set_option("sa_text_rounds", 0)
        e.set_option("sa_doubling_local", 0)
        _doubling["gd"] = e
    return _doubling["gd"]


def no_shortcut_executor(rq):
    """A third context: shared-memory refinement by 23-symbol text steps only (the distance
    shortcut switched off)."""
    if "ns" not in _doubling:
        e = rq.Executor(0)
        e.set_option("sa_shortcut", 0)
        _doubling["ns"] = e
    return _doubling["ns"]


def no_uniform_executor(rq):
    """A fourth context: the uniform read-set path switched off (general records, 11 shared symbols)."""
    if "nu" not in _doubling:
        e = rq.Executor(0)
        e.set_option("sa_uniform", 0)
        _doubling["nu"] = e
    return _doubling["nu"]


def check(rq, ex, oracle, text):
    got = rq.build_parallel(text, ex)
    wsa, wrank = oracle.build_sa(text)
    assert np.array_equal(got.sa, wsa), f"sa differs for text of length {len(text)}"
    assert np.array_equal(got.rank, wrank)
    if len(text) <= 300_000:
        alt = rq.build_parallel(text, doubling_executor(rq))
        assert np.array_equal(alt.sa, wsa), f"prefix-doubling sa differs for text of length {len(text)}"
        assert np.array_equal(alt.rank, wrank)
        alt = rq.build_parallel(text, global_doubling_executor(rq))
        assert alt.stats.refined_tile == 0
        assert np.array_equal(alt.sa, wsa), f"global prefix-doubling sa differs for text of length {len(text)}"
        assert np.array_equal(alt.rank, wrank)
        alt = rq.build_parallel(text, no_shortcut_executor(rq))
        assert np.array_equal(alt.sa, wsa), f"text-round sa differs for text of length {len(text)}"
        assert np.array_equal(alt.rank, wrank)
        alt = rq.build_parallel(text, no_uniform_executor(rq))
        assert alt.stats.init_symbols not in (15, 16)
        assert np.array_equal(alt.sa, wsa), f"general-record sa differs for text of length {len(text)}"
        assert np.array_equal(alt.rank, wrank)
    return got


def test_classic_inputs(rq, ex, oracle):
    # test_suffix_array.cpp:10-14
    assert rq.build_parallel(b"banana", ex).sa.tolist() == [5, 3, 1, 0, 4, 2]
    assert rq.build_parallel(b"aaa", ex).sa.tolist() == [2, 1, 0]
    r = rq.build_parallel(b"", ex)
    assert r.sa.size == 0 and r.rank.size == 0
    assert rq.build_parallel(b"x", ex).sa.tolist() == [0]


def test_rank_is_the_inverse_of_sa(rq, ex):
    # test_suffix_array.cpp:16-21
    r = rq.build_parallel(b"mississippi", ex)
    assert np.array_equal(r.rank[r.sa], np.arange(r.sa.size, dtype=np.uint32))


def test_exhaustive_ab_strings(rq, ex, oracle):
    # test_suffix_array.cpp:23-36: all 510 strings over {a,b} of length 1..8
    for length in range(1, 9):
        for mask in range(1 << length):
            s = bytes(ord("b") if (mask >> i) & 1 else ord("a") for i in range(length))
            check(rq, ex, oracle, s)


def test_sentinel_ties_break_by_position(rq, ex, oracle):
    # test_suffix_array.cpp:38-44
    got = check(rq, ex, oracle, b"GA\0TT\0")
    assert got.sa.tolist() == [2, 5, 1, 0, 4, 3]
    assert got.stats.alphabet == 0  # the 2-bit DNA path


def test_random_sentinel_joined_texts(rq, ex, oracle):
    # test_suffix_array.cpp:46-61 (own RNG: the property, not the stream, is what matters)
    rng = np.random.default_rng(41)
    for _ in range(150):
        parts = []
        for _f in range(1 + int(rng.integers(0, 5))):
            ln = 1 + int(rng.integers(0, 6))
            parts.append(bytes(rng.choice([97, 98], ln).astype(np.uint8)) + b"\0")
        check(rq, ex, oracle, b"".join(parts))
    for _ in range(100):  # the same with the DNA alphabet (2-bit path)
        parts = []
        for _f in range(1 + int(rng.integers(0, 6))):
            ln = 1 + int(rng.integers(0, 40))
            parts.append(bytes(rng.choice([65, 67, 71, 84], ln, p=[.7, .1, .1, .1]).astype(np.uint8)) + b"\0")
        check(rq, ex, oracle, b"".join(parts))


def test_random_dna_4096(rq, ex, oracle):
    # test_suffix_array.cpp:63-72
    rng = np.random.default_rng(43)
    check(rq, ex, oracle, bytes(rng.choice([65, 67, 71, 84], 4096).astype(np.uint8)))


@pytest.mark.parametrize("n", [2, 3, 12, 13, 14, 25, 26, 27, 63, 64, 65, 2047, 2048, 2049, 4095, 4096, 4097,
                               8193, 100_003])
def test_sizes_around_tile_and_kmer_boundaries(rq, ex, oracle, n):
    rng = np.random.default_rng(n)
    check(rq, ex, oracle, bytes(rng.choice([65, 67, 71, 84], n).astype(np.uint8)))       # no sentinel at all
    t = rng.choice([65, 67, 71, 84, 0], n, p=[.24, .24, .24, .24, .04]).astype(np.uint8)  # ragged reads
    check(rq, ex, oracle, bytes(t))
    t[-1] = 0
    check(rq, ex, oracle, bytes(t))


def test_adversarial_repeats(rq, ex, oracle):
    check(rq, ex, oracle, b"A" * 5000)                       # one run: log2(n) doubling rounds
    check(rq, ex, oracle, b"A" * 3000 + b"\0")
    check(rq, ex, oracle, (b"A" * 150 + b"\0") * 300)        # identical reads: ties only by sentinel position
    check(rq, ex, oracle, (b"ACGT" * 40 + b"\0") * 200)      # periodic reads
    check(rq, ex, oracle, b"\0" * 1000)                      # only sentinels
    check(rq, ex, oracle, b"\0\0A\0\0\0CC\0" * 50)
    check(rq, ex, oracle, b"AC" * 4000)
    rng = np.random.default_rng(5)
    unit = bytes(rng.choice([65, 67, 71, 84], 700).astype(np.uint8))
    check(rq, ex, oracle, unit * 12)                         # long exact repeats, no sentinel


def test_generic_byte_texts(rq, ex, oracle):
    got = check(rq, ex, oracle, b"abthatb\0hatbpaab\0tbabhhatbpaa\0paabtabh\0bhaabtpb\0")
    assert got.stats.alphabet == 1
    rng = np.random.default_rng(6)
    check(rq, ex, oracle, bytes(rng.integers(1, 256, 20_000).astype(np.uint8)))
    check(rq, ex, oracle, bytes(rng.integers(0, 4, 30_000).astype(np.uint8)))    # bytes 0..3, many sentinels
    check(rq, ex, oracle, bytes(rng.choice([65, 67, 71, 84, 78], 50_000).astype(np.uint8)))  # DNA with N
    check(rq, ex, oracle, b"ab" * 3000 + b"\0" + b"ba" * 1000)
    check(rq, ex, oracle, bytes([255]) * 4000)


@pytest.mark.parametrize("G,L,k", [(5_000, 100, 500), (50_000, 100, 5_000), (100_000, 150, 6_000)])
def test_read_sets_against_the_oracle(rq, ex, oracle, G, L, k):
    text, _ = rq.synth_read_text(G, L, k)
    got = check(rq, ex, oracle, text)
    assert got.stats.alphabet == 0 and got.stats.init_symbols == 16    # the uniform read-set path
    assert got.stats.rounds <= 6 and got.stats.refined_global == 0
    alt = rq.build_parallel(text, no_uniform_executor(rq))
    assert alt.stats.init_symbols == 11 and np.array_equal(alt.sa, got.sa)


def _reads(genome, L, starts):
    return b"".join(genome[int(s):int(s) + L] + b"\0" for s in starts)


def test_uniform_read_sets_with_repeats_and_duplicates(rq, ex, oracle):
    """The uniform path's proofs (one comparison per read) under stress: repeated genomes (several
    loci per 15-mer group), duplicate reads, low-complexity genomes, tiny and maximal periods."""
    rng = np.random.default_rng(77)
    for G, L, k, alpha in [(400, 40, 600, 4), (3000, 100, 2000, 4), (300, 16, 900, 2), (5000, 254, 400, 4),
                           (2000, 60, 1500, 2), (64, 30, 500, 4), (20000, 150, 4000, 4)]:
        letters = [65, 67, 71, 84][:alpha]
        unit = bytes(rng.choice(letters, G).astype(np.uint8))
        for genome in (unit, unit[:G // 2] * 2, unit[:G // 4] + unit[:G // 4][:-3] + b"A" * 3 + unit[G // 2:]):
            starts = rng.integers(0, len(genome) - L + 1, k)
            text = _reads(genome, L, starts)
            got = check(rq, ex, oracle, text)
            assert got.stats.alphabet == 0
    # duplicates of whole reads, reads that differ only in their last base
    g = bytes(rng.choice([65, 67, 71, 84], 500).astype(np.uint8))
    reads = [g[i:i + 50] for i in rng.integers(0, 450, 300)]
    reads += reads[:100] + [r[:-1] + b"A" for r in reads[:100]] + [b"C" + r[1:] for r in reads[:50]]
    check(rq, ex, oracle, b"".join(r + b"\0" for r in reads))
    # more whole reads inside one chunk than the link kernel's queue holds (they are compared inline then)
    check(rq, ex, oracle, (b"ACGTACGTACGTACGT" + b"\0") * 6000)
    check(rq, ex, oracle, (b"A" * 20 + b"\0") * 5000)                 # one group: every suffix of >= 16 A's
    mixed = [b"A" * 20, b"A" * 19 + b"C", b"C" + b"A" * 19, b"ACGTA" * 4] * 1500
    check(rq, ex, oracle, b"".join(r + b"\0" for r in mixed))        # oversize groups mixing loci: handed on


def test_uniform_path_with_many_resorted_groups_at_partitioned_inverse_size(rq, ex, oracle):
    """n >= 2^22 (partitioned inverse) on a genome with long repeats: plenty of groups mix loci and
    take refinement steps; sa by proof, rank as its inverse."""
    rng = np.random.default_rng(79)
    unit = bytes(rng.choice([65, 67, 71, 84], 60_000).astype(np.uint8))
    genome = unit + unit[:30_000] + bytes(rng.choice([65, 67, 71, 84], 20_000).astype(np.uint8)) + unit[10_000:40_000]
    starts = rng.integers(0, len(genome) - 100 + 1, 45_000)
    text = np.frombuffer(_reads(genome, 100, starts), dtype=np.uint8)
    assert text.size >= 1 << 22
    got = rq.build_parallel(text, ex)
    assert got.stats.init_symbols == 16 and got.stats.rounds >= 1     # some groups took refinement steps
    assert oracle.verify_sa(text, got.sa) == 0
    assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))
    alt = rq.build_parallel(text, no_uniform_executor(rq))
    assert np.array_equal(alt.sa, got.sa) and np.array_equal(alt.rank, got.rank)


def test_texts_that_only_look_uniform(rq, ex, oracle):
    """n divisible by the number of sentinels, but the sentinels are not one period apart: the check
    kernel must hand the text to the general paths."""
    rng = np.random.default_rng(78)
    g = bytes(rng.choice([65, 67, 71, 84], 4000).astype(np.uint8))
    reads = []
    for i in range(400):
        L = 30 if i % 2 else 50          # mean period 41
        s = int(rng.integers(0, 3900))
        reads.append(g[s:s + L] + b"\0")
    got = check(rq, ex, oracle, b"".join(reads))
    assert got.stats.init_symbols in (11, 15)   # general records, or the ragged read-set route
    text = bytearray(b"".join(g[int(s):int(s) + 40] + b"\0" for s in rng.integers(0, 3900, 300)))
    text[100], text[40] = 0, 65          # one sentinel moved
    got = check(rq, ex, oracle, bytes(text))
    assert got.stats.init_symbols in (11, 15)   # general records, or the ragged read-set route


def test_speculative_route_is_verified_on_the_device(rq, oracle):
    """A context starts the next build of a text of the same length on the previous build's route
    without a host round trip (sa.cu build_sa_device); the route's premises are re-checked on the
    device every time.  Same length, different kind of text -- ragged reads, a byte outside the
    alphabet, other genome, shifted sentinels -- must still give the reference order, and the
    route must come back for the next uniform text."""
    e = rq.Executor(0)
    try:
        rng = np.random.default_rng(71)
        L, k = 60, 3000
        def uniform(seed):
            g = np.random.default_rng(seed).choice([65, 67, 71, 84], 20_000).astype(np.uint8)
            st = np.random.default_rng(seed + 1).integers(0, 20_000 - L, k)
            return b"".join(bytes(g[x:x + L]) + b"\0" for x in st)
        a = uniform(1)
        n = len(a)
        texts = [a, a, uniform(5)]
        ragged = bytearray(uniform(9))
        ragged[L] = 65; ragged[L - 7] = 0                     # one sentinel moved: k separators, not one per period
        texts.append(bytes(ragged))
        other = bytearray(uniform(11)); other[1234] = ord("N")  # not a DNA text
        texts.append(bytes(other))
        fewer = bytearray(uniform(13)); fewer[L] = 71         # k - 1 separators
        texts.append(bytes(fewer))
        texts += [uniform(17), bytes(rng.choice([65, 67], n).astype(np.uint8)), uniform(19)]
        for t in texts:
            assert len(t) == n
            got = rq.build_parallel(t, e)
            wsa, wrank = oracle.build_sa(t)
            assert np.array_equal(got.sa, wsa) and np.array_equal(got.rank, wrank)
        assert got.stats.init_symbols == 16
    finally:
        e.close()


def test_repeated_device_builds_replay_one_cuda_graph(rq, oracle):
    """A device-resident build whose text buffer, outputs, workspace, stream and options are those of the
    previous one is replayed as one CUDA graph (sa.cu build_sa_device, option "sa_graph").  The graph reads the
    text through its pointer: new contents in the same buffer must give the new text's order; a text of another
    kind must fail the device-side check, fall back and drop the graph; the launch count must keep counting
    the kernels a replay runs; switching the option off must give the same arrays."""
    import ctypes as C
    import torch
    lib = rq._lib.load()
    L, k = 60, 3000
    def uniform(seed):
        g = np.random.default_rng(seed).choice([65, 67, 71, 84], 20_000).astype(np.uint8)
        st = np.random.default_rng(seed + 1).integers(0, 20_000 - L, k)
        return np.frombuffer(b"".join(bytes(g[x:x + L]) + b"\0" for x in st), np.uint8)
    n = k * (L + 1)
    e = rq.Executor(0)
    stream = torch.cuda.Stream()
    try:
        e.set_stream(stream.cuda_stream)
        with torch.cuda.stream(stream):
            d_text = torch.empty(n, dtype=torch.uint8, device="cuda")
            d_sa = torch.empty(n, dtype=torch.int32, device="cuda")
            d_rank = torch.empty(n, dtype=torch.int32, device="cuda")
            texts = [uniform(1), uniform(1), uniform(3), uniform(5)]
            ragged = uniform(9).copy(); ragged[L] = 65; ragged[L - 7] = 0      # same length, not uniform any more
            texts += [ragged, uniform(7), uniform(11), uniform(13)]
            per_build = []
            for i, t in enumerate(texts):
                if i == 6: e.set_option("sa_graph", 0)
                d_text.copy_(torch.from_numpy(t.copy()), non_blocking=False)
                st = rq.SaStats()
                l0 = e.launch_count
                rq._lib.check(lib.reseq_cuda_build_sa_device(e.handle, C.c_void_p(d_text.data_ptr()), n, C.c_void_p(d_sa.data_ptr()),
                                                             C.c_void_p(d_rank.data_ptr()), C.byref(st)))
                e.synchronize()
                per_build.append(e.launch_count - l0)
                wsa, wrank = oracle.build_sa(t.tobytes())
                assert np.array_equal(d_sa.cpu().numpy().view(np.uint32), wsa), f"build {i}"
                assert np.array_equal(d_rank.cpu().numpy().view(np.uint32), wrank), f"build {i}"
            # builds 2 and 3 replay the graph captured by build 1, build 7 launches kernel by kernel: same kernels
            assert per_build[2] == per_build[3] == per_build[7] > 10
    finally:
        e.close()


def _ragged_reads(rng, genome, k, lo, hi):
    out = []
    for _ in range(k):
        ln = int(rng.integers(lo, hi + 1))
        st = int(rng.integers(0, len(genome) - ln + 1))
        out.append(bytes(genome[st:st + ln]) + b"\0")
    return b"".join(out)


def test_ragged_read_sets_take_the_read_set_route(rq, ex, oracle):
    """Reads of mixed lengths (trimmed reads): records born transposed with ragged rows, 15-base keys with
    a short-suffix tag, proofs as one bit per position (sa.cu, ragged read sets).  Lengths from 1 to 254,
    repeats (groups that mix loci), duplicates, reads contained in others, reads shorter than the key."""
    rng = np.random.default_rng(81)
    genome = rng.choice([65, 67, 71, 84], 40_000).astype(np.uint8)
    for lo, hi, k in ((60, 150, 6000), (16, 254, 3000), (1, 40, 5000), (100, 101, 4000), (254, 254, 40), (15, 17, 6000)):
        text = _ragged_reads(rng, genome, k, lo, hi)
        got = check(rq, ex, oracle, text)
        if len(text) // k >= 16 and lo != hi:
            assert got.stats.init_symbols == 15, (lo, hi)          # the ragged route took it
    unit = bytes(rng.choice([65, 67, 71, 84], 3000).astype(np.uint8))
    rep = np.frombuffer(unit + unit[:1500] + unit[500:2500] + unit, np.uint8)     # repeats: groups mix loci
    text = _ragged_reads(rng, rep, 5000, 40, 120)
    text += text[: text.index(b"\0", 4000) + 1]                                   # duplicated reads
    got = check(rq, ex, oracle, text)
    assert got.stats.init_symbols == 15
    low = rng.choice([65, 67], 5000).astype(np.uint8)                             # two-letter genome: long ties
    check(rq, ex, oracle, _ragged_reads(rng, low, 3000, 20, 90))
    # not this route: a read of 255 bases, text behind the last separator, mostly tiny reads
    assert check(rq, ex, oracle, _ragged_reads(rng, genome, 300, 255, 255) + _ragged_reads(rng, genome, 300, 50, 60)).stats.init_symbols != 15
    assert check(rq, ex, oracle, _ragged_reads(rng, genome, 2000, 30, 80) + b"ACGT").stats.init_symbols != 15
    assert check(rq, ex, oracle, _ragged_reads(rng, genome, 4000, 1, 12)).stats.init_symbols != 15


def test_ragged_read_set_at_config2_size(rq, oracle):
    """BASELINE config 2's genome and coverage with read lengths drawn from 100..150: n ~ 116 M suffixes on
    the ragged route, proved equal to the reference order."""
    rng = np.random.default_rng(82)
    genome = rq.synth_random_dna(4_600_000, 1)
    k = 920_000
    lens = rng.integers(100, 151, k)
    starts = rng.integers(0, genome.size - 150, k)
    total = int(lens.sum()) + k
    text = np.zeros(total, np.uint8)
    offs = np.concatenate(([0], np.cumsum(lens + 1)[:-1]))
    idx = np.repeat(starts - offs, lens + 1) + np.arange(total)        # genome index of every text byte (sentinels: garbage)
    idx = np.minimum(idx, genome.size - 1)
    text[:] = genome[idx]
    text[offs + lens] = 0
    e = rq.Executor(0)
    try:
        got = rq.build_parallel(text, e)
        assert got.stats.init_symbols == 15 and got.stats.refined_global == 0
        assert oracle.verify_sa(text, got.sa, threads=32) == 0
        assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))
    finally:
        e.close()


def test_reference_bench_input_fingerprint(rq, ex, oracle):
    """make_random_dna(1<<20, 1): checksum_u32(sa) == 7546189330682201289 (BASELINE.md section 2,
    the reference's own build_parallel and build_naive)."""
    text = rq.synth_random_dna(1 << 20, 1)
    got = rq.build_parallel(text, ex)
    assert oracle.checksum_u32(got.sa) == 7546189330682201289
    assert oracle.verify_sa(text, got.sa) == 0
    assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))


def test_config1_full_size_fingerprint_and_proof(rq, ex, oracle):
    """BASELINE config 1 (1 Mbp genome, 100 bp reads, 10x; n = 10 100 000): the reference's
    build_parallel == build_naive gave checksum_u32(sa) = 11642757783061468293; the
    permutation + adjacent-order verifier is a proof of equality at this size."""
    text, _ = rq.synth_read_text(1_000_000, 100, 100_000)
    got = rq.build_parallel(text, ex)
    assert got.stats.rounds <= 4 and got.stats.refined_global == 0 and got.stats.init_symbols == 16
    assert oracle.checksum_u32(got.sa) == 11642757783061468293
    assert oracle.verify_sa(text, got.sa) == 0
    assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))


def test_config2_full_size_proof(rq, ex, oracle):
    """BASELINE config 2 (4.6 Mbp, 150 bp, 30x; n = 138 920 000): size-independent proof."""
    text, _ = rq.synth_read_text(4_600_000, 150, 920_000)
    got = rq.build_parallel(text, ex)
    assert got.stats.rounds <= 6 and got.stats.refined_global == 0
    assert oracle.verify_sa(text, got.sa, threads=32) == 0
    assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))


def test_config3_full_size_proof(rq, ex, oracle):
    """BASELINE config 3 (one text of ~100 Mbp of reads: 10 Mbp genome, 150 bp, 10x; n = 100 666 566):
    proof of equality with the reference order at full size."""
    text, _ = rq.synth_read_text(10_000_000, 150, 666_666)
    assert text.size == 100_666_566
    got = rq.build_parallel(text, ex)
    assert got.stats.init_symbols == 16 and got.stats.refined_global == 0
    assert oracle.verify_sa(text, got.sa, threads=32) == 0
    assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32))


@pytest.mark.parametrize("option,value,name", [("sa_uniform", 0, "general DNA records (route ii)"),
                                               ("sa_text_rounds", 0, "prefix doubling (route iii)")])
def test_general_routes_at_config2_full_size(rq, oracle, option, value, name):
    """The two general engines forced on BASELINE config 2's full text (n = 138 920 000): the route a
    ragged read set takes (sa_uniform = 0) and the north star's prefix doubling (sa_text_rounds = 0),
    each proved equal to the reference order."""
    e = rq.Executor(0)
    try:
        e.set_option(option, value)
        text, _ = rq.synth_read_text(4_600_000, 150, 920_000)
        got = rq.build_parallel(text, e)
        if option == "sa_uniform":
            assert got.stats.init_symbols != 16 and got.stats.refined_global == 0, name
        else:
            assert got.stats.init_symbols == 13 and got.stats.rounds >= 4, name
        assert oracle.verify_sa(text, got.sa, threads=32) == 0, name
        assert np.array_equal(got.rank[got.sa], np.arange(text.size, dtype=np.uint32)), name
    finally:
        e.close()


def _device_build_and_prove(rq, oracle, G, L, k, need_gib):
    import torch
    free, _total = torch.cuda.mem_get_info()
    if free < need_gib * 2**30:
        pytest.skip(f"needs ~{need_gib} GB of device memory")
    text, _ = rq.synth_read_text(G, L, k)
    n = int(text.size)
    e = rq.Executor(0)
    try:
        d_text = torch.from_numpy(text).cuda()
        d_sa = torch.empty(n, dtype=torch.int32, device="cuda")
        d_rank = torch.empty(n, dtype=torch.int32, device="cuda")
        st = rq.SaStats()
        lib = rq._lib.load()
        rq._lib.check(lib.reseq_cuda_build_sa_device(e.handle, C.c_void_p(d_text.data_ptr()), n,
                                                     C.c_void_p(d_sa.data_ptr()), C.c_void_p(d_rank.data_ptr()), C.byref(st)))
        e.synchronize()
        assert st.init_symbols == 16 and st.refined_global == 0
        chunk = 1 << 27
        for b in range(0, n, chunk):
            hi = min(n, b + chunk)
            sa_c = d_sa[b:hi].to(torch.int64) & 0xFFFFFFFF
            assert torch.equal(d_rank[sa_c].to(torch.int64) & 0xFFFFFFFF, torch.arange(b, hi, device="cuda", dtype=torch.int64))
            del sa_c
        sa = d_sa.cpu().numpy().view(np.uint32)
        del d_sa, d_rank, d_text
    finally:
        e.close()
        torch.cuda.empty_cache()
    assert oracle.verify_sa(text, sa, threads=32) == 0
    return n


def test_config4_one_billion_suffixes(rq, oracle):
    """BASELINE config 4 (100 Mbp genome, 150 bp, 10x; n = 1 006 666 566) on one B200 through the
    device-resident entry point: proof of equality on the host, inverse checked on the device."""
    assert _device_build_and_prove(rq, oracle, 100_000_000, 150, 6_666_666, 45) == 1_006_666_566


def test_config5_three_billion_suffixes_beyond_the_reference_cap(rq, oracle):
    """BASELINE config 5 (300 Mbp genome, 150 bp, 10x; n = 3.02 G > 2^31 - 1, the reference's cap,
    suffix_array.hpp:64) on one B200 through the device-resident entry point: every index above 2^31
    exercises the 64-bit address arithmetic of each kernel.  Proof of equality on the host
    (permutation + adjacent suffix_less over all n), inverse checked on the device."""
    import torch
    free, _total = torch.cuda.mem_get_info()
    if free < 120 * 2**30:
        pytest.skip("needs ~105 GB of device memory")
    try:
        import psutil
        if psutil.virtual_memory().available < 48 * 2**30:
            pytest.skip("needs ~25 GB of host memory")
    except ImportError:
        pass
    text, _ = rq.synth_read_text(300_000_000, 150, 20_000_000)
    n = int(text.size)
    assert n == 3_020_000_000
    e = rq.Executor(0)
    try:
        d_text = torch.from_numpy(text).cuda()
        d_sa = torch.empty(n, dtype=torch.int32, device="cuda")
        d_rank = torch.empty(n, dtype=torch.int32, device="cuda")
        st = rq.SaStats()
        lib = rq._lib.load()
        rq._lib.check(lib.reseq_cuda_build_sa_device(e.handle, C.c_void_p(d_text.data_ptr()), n,
                                                     C.c_void_p(d_sa.data_ptr()), C.c_void_p(d_rank.data_ptr()), C.byref(st)))
        e.synchronize()
        assert st.init_symbols == 16 and st.refined_global == 0
        chunk = 1 << 27
        for b in range(0, n, chunk):
            hi = min(n, b + chunk)
            sa_c = d_sa[b:hi].to(torch.int64) & 0xFFFFFFFF
            assert torch.equal(d_rank[sa_c].to(torch.int64) & 0xFFFFFFFF, torch.arange(b, hi, device="cuda", dtype=torch.int64))
            del sa_c
        sa = d_sa.cpu().numpy().view(np.uint32)
        del d_sa, d_rank, d_text
    finally:
        e.close()
        torch.cuda.empty_cache()
    assert oracle.verify_sa(text, sa, threads=32) == 0


def test_text_too_large_is_rejected_before_any_work(rq, ex):
    lib = rq._lib.load()
    dummy = np.zeros(16, np.uint8)
    out = np.zeros(16, np.uint32)
    st = lib.reseq_cuda_build_sa(ex.handle, dummy.ctypes.data_as(C.c_void_p), C.c_size_t(0xFFFFFFFF),
                                 out.ctypes.data_as(C.c_void_p), None, None)
    assert st == rq._lib.TEXT_TOO_LARGE
    with pytest.raises(rq.TextTooLargeError):
        rq._lib.check(st)


def test_device_resident_entry_point(rq, ex, oracle):
    import torch
    text, _ = rq.synth_read_text(30_000, 100, 3_000)
    d_text = torch.from_numpy(text).cuda()
    d_sa = torch.empty(text.size, dtype=torch.int32, device="cuda")
    d_rank = torch.empty(text.size, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    lib = rq._lib.load()
    st = rq.SaStats()
    rq._lib.check(lib.reseq_cuda_build_sa_device(ex.handle, C.c_void_p(d_text.data_ptr()), text.size,
                                                 C.c_void_p(d_sa.data_ptr()), C.c_void_p(d_rank.data_ptr()),
                                                 C.byref(st)))
    ex.synchronize()
    wsa, wrank = oracle.build_sa(text)
    assert np.array_equal(d_sa.cpu().numpy().view(np.uint32), wsa)
    assert np.array_equal(d_rank.cpu().numpy().view(np.uint32), wrank)
    h = C.c_uint64()
    rq._lib.check(lib.reseq_cuda_checksum_u32_device(ex.handle, C.c_void_p(d_sa.data_ptr()), text.size, C.byref(h)))
    assert h.value == oracle.checksum_u32(wsa)


def test_oversize_groups_hand_over_to_prefix_doubling(rq, ex, oracle):
    """Groups larger than the refine kernel's shared-memory window (identical / low-complexity
    reads) must be finished by the global prefix-doubling rounds."""
    text = (b"ACGTACGTAC" * 12 + b"\0") * 3000          # 3000 identical reads: groups of 3000
    got = check(rq, ex, oracle, text)
    # the uniform path proves every duplicate a prefix of the next one: no group needs sorting, whatever its size
    assert got.stats.init_symbols == 16 and got.stats.refined_global == 0
    alt = rq.build_parallel(text, no_uniform_executor(rq))
    assert alt.stats.refined_global > 0 and np.array_equal(alt.sa, got.sa)
    rng = np.random.default_rng(8)
    unit = bytes(rng.choice([65, 67, 71, 84], 100).astype(np.uint8))
    text = b"".join(unit[int(o):] + unit[:int(o)] + b"\0" for o in rng.integers(0, 100, 2500))  # rotations
    got = check(rq, ex, oracle, text)


def test_doubling_only_mode_on_config1(rq, oracle):
    e = doubling_executor(rq)
    text, _ = rq.synth_read_text(1_000_000, 100, 100_000)
    got = rq.build_parallel(text, e)
    assert got.stats.rounds == 3 and got.stats.init_symbols == 13   # h = 13, 26, 52 -> 104 >= 101
    assert oracle.checksum_u32(got.sa) == 11642757783061468293
