"""The synthetic workload generators (host/synth.cpp) reproduce the reference's inputs
bit-for-bit: bench.hpp:54-72, shotgun.hpp:20-27, sequence.hpp:103-124.  CPU only."""
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def test_fingerprints_of_generated_inputs(rq, oracle):
    fp = GOLDEN["fingerprints"]
    for n in (1 << 10, 1 << 14, 1 << 16):
        text = rq.synth_random_dna(n, 1)
        assert str(oracle.fnv1a64(text)) == fp[f"random_dna_{n}_seed1"]["text_fnv"]
        sa, _ = oracle.build_sa(text)
        assert str(oracle.checksum_u32(sa)) == fp[f"random_dna_{n}_seed1"]["sa_checksum"]
    k, p = rq.synth_random_keys(1 << 14, 1)
    assert str(oracle.checksum_u32(k)) == fp["random_keys_16384_seed1"]["keys_checksum"]
    assert np.array_equal(p, np.arange(1 << 14, dtype=np.uint32))
    text, starts = rq.synth_read_text(50_000, 100, 5_000)
    assert str(oracle.fnv1a64(text)) == fp["read_text_G50000_L100_k5000"]["text_fnv"]
    assert np.array_equal(starts, np.arange(5_000, dtype=np.uint32) * 101)
    sa, _ = oracle.build_sa(text)
    assert str(oracle.checksum_u32(sa)) == fp["read_text_G50000_L100_k5000"]["sa_checksum"]


def test_generators_equal_the_reference(rq, ref):
    if ref is None:
        pytest.skip("oracle/_ref not built here")
    assert np.array_equal(rq.synth_random_dna(5000, 9), ref.make_random_dna(5000, 9))
    k, p = rq.synth_random_keys(4000, 3)
    rk, rp = ref.make_random_keys(4000, 3)
    assert np.array_equal(k, rk) and np.array_equal(p, rp)
    for G, L, kk in ((1000, 30, 100), (7777, 150, 50), (64, 64, 5)):
        text, starts = rq.synth_read_text(G, L, kk, 11, 12)
        assert np.array_equal(text, ref.make_read_text(G, L, kk, 11, 12))
