"""The scalable host greedy merge (host/greedy.cpp) against the oracle's literal restatement of
overlap.hpp:80-113 -- CPU only: the overlap lists are supplied by the oracle here, so this
isolates the merge logic (tie-breaks, containment, sub-threshold tail, zero-overlap tail)."""
import numpy as np
import pytest

from tests.oracle_lib import concat_of


def shotgun(rng, G, k, lo, hi, alphabet):
    genome = rng.choice(alphabet, G).astype(np.uint8)
    out = []
    for _ in range(k):
        ln = min(G, int(rng.integers(lo, hi + 1)))
        s = int(rng.integers(0, G - ln + 1))
        out.append(bytes(genome[s:s + ln]))
    return out


def run(rq, oracle, frags, tau):
    concat, starts, lens = concat_of(frags)
    fs = rq.FragmentSet(concat, starts, "generic_byte")
    oi, oj, ow = oracle.overlap_list(concat, starts, lens, tau)
    contained = np.ones(len(frags), np.uint8)
    contained[oracle.absorb_contained(concat, starts, lens)] = 0
    ov = rq.OverlapList(oi, oj, ow, contained, 0, 0.0, tau)
    return rq.greedy_superstring_from_overlaps(fs, ov), oracle.greedy(concat, starts, lens)


def test_paper_example(rq, oracle, ref):
    frags = [b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"]
    (sup, order), want = run(rq, oracle, frags, 1)
    assert sup == b"abthatbabhhatbpaabtabhaabtpb"
    assert order.tolist() == [0, 2, 1, 3, 4]
    assert want[0] == sup and want[1].tolist() == order.tolist()
    if ref is not None:
        rs, ro = ref.greedy(frags, "generic_byte")
        assert rs == sup and ro.tolist() == order.tolist()


@pytest.mark.parametrize("seed", range(8))
def test_random_sets_equal_the_literal_loop(rq, oracle, ref, seed):
    rng = np.random.default_rng(1000 + seed)
    for it in range(250):
        mode = it % 4
        if mode == 0:    # two-letter alphabet: many ties, periodic overlaps, containments
            frags = shotgun(rng, int(rng.integers(20, 80)), int(rng.integers(4, 16)), 3, 14, (65, 67))
        elif mode == 1:  # equal lengths (shotgun reads)
            frags = shotgun(rng, int(rng.integers(30, 120)), int(rng.integers(4, 22)), 10, 10, (65, 67, 71, 84))
        elif mode == 2:  # mixed lengths, 4 letters
            frags = shotgun(rng, int(rng.integers(20, 80)), int(rng.integers(4, 16)), 4, 25, (65, 67, 71, 84))
        else:            # unrelated fragments: mostly zero overlaps -> concatenation order
            frags = [bytes(rng.choice((65, 67, 71, 84), int(rng.integers(1, 8))).astype(np.uint8))
                     for _ in range(int(rng.integers(1, 10)))]
        for tau in (1, 3, 6):
            (sup, order), want = run(rq, oracle, frags, tau)
            assert sup == want[0] and order.tolist() == want[1].tolist(), (frags, tau)
        if ref is not None and it % 10 == 0:
            rs, ro = ref.greedy(frags, "dna")
            assert rs == want[0] and ro.tolist() == want[1].tolist()


def test_single_and_all_contained(rq, oracle):
    (sup, order), want = run(rq, oracle, [b"ACGT"], 1)
    assert sup == b"ACGT" and order.tolist() == [0]
    (sup, order), want = run(rq, oracle, [b"ACGT", b"ACGT", b"CG", b"ACGT"], 1)
    assert sup == want[0] == b"ACGT" and order.tolist() == want[1].tolist() == [0]
