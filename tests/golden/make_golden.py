"""Generates tests/golden/golden.json from the REAL reference (oracle/_ref, compiled from
/root/reference/proj/include by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_golden.py)
on boxes where /root/reference does not exist."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from tests.oracle_lib import Reference, concat_of  # noqa: E402


def main():
    ref = Reference()
    rng = np.random.default_rng(20240614)
    g = {"generator": "tests/golden/make_golden.py over oracle/_ref (unmodified reference headers)"}

    # suffix arrays: build_naive == build_parallel(workers 2, chunk 64) on assorted texts
    texts = [b"banana", b"aaa", b"mississippi", b"GA\0TT\0", b"abthatb\0hatbpaab\0tbabhhatbpaa\0paabtabh\0bhaabtpb\0"]
    for _ in range(12):
        parts = [bytes(rng.choice([65, 67, 71, 84], int(rng.integers(1, 30))).astype(np.uint8)) + b"\0"
                 for _ in range(int(rng.integers(1, 8)))]
        texts.append(b"".join(parts))
    for _ in range(4):
        texts.append(bytes(rng.choice([97, 98], int(rng.integers(5, 60))).astype(np.uint8)))
    texts.append(bytes(ref.make_read_text(2000, 40, 60)))
    sa_cases = []
    for t in texts:
        sa, rank = ref.build_naive(t)
        st, psa, prank = ref.build_parallel(t, 2, 64)
        assert st == 0 and np.array_equal(sa, psa) and np.array_equal(rank, prank)
        sa_cases.append({"text": list(t), "sa": sa.tolist()})
    g["suffix_arrays"] = sa_cases

    # fingerprints of the reference's bench inputs (bench.hpp:54-72,139-142)
    fp = {}
    for n in (1 << 10, 1 << 14, 1 << 16):
        text = ref.make_random_dna(n, 1)
        st, sa, _ = ref.build_parallel(text, 4, 1 << 12)
        fp[f"random_dna_{n}_seed1"] = {"text_fnv": str(ref.fnv1a64(text)), "sa_checksum": str(ref.checksum_u32(sa))}
    k, p = ref.make_random_keys(1 << 14, 1)
    st, ko, po = ref.radix_sort(k, p)
    fp["random_keys_16384_seed1"] = {"keys_checksum": str(ref.checksum_u32(k)),
                                     "sorted_keys_checksum": str(ref.checksum_u32(ko)),
                                     "sorted_payload_checksum": str(ref.checksum_u32(po))}
    rt = ref.make_read_text(50_000, 100, 5_000)
    st, sa, _ = ref.build_parallel(rt, 8, 1 << 15)
    fp["read_text_G50000_L100_k5000"] = {"text_fnv": str(ref.fnv1a64(rt)), "sa_checksum": str(ref.checksum_u32(sa))}
    fp["published_in_BASELINE_md"] = {"random_dna_1048576_seed1_sa": "7546189330682201289",
                                      "config1_sa": "11642757783061468293",
                                      "random_keys_1048576_seed1_sorted": "91396105105168530"}
    g["fingerprints"] = fp

    # scan / split / sorts
    prim = []
    for _ in range(6):
        n = int(rng.integers(1, 200))
        k = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        if _ % 2:
            k &= np.uint32(0x3F)
        p = np.arange(n, dtype=np.uint32)
        bit = int(rng.integers(0, 32))
        _, sk, sp = ref.split_by_bit(k, p, bit, 3, 16)
        _, rk, rp = ref.radix_sort(k, p, 2, 32)
        _, ck, cp = ref.chunked_radix_sort(k, p, 4, 3, 17)
        assert np.array_equal(rk, ck) and np.array_equal(rp, cp)
        v = (k % 1000).astype(np.uint32)
        _, sc = ref.exclusive_scan(v, 2, 8)
        prim.append({"keys": k.tolist(), "bit": bit, "split_keys": sk.tolist(), "split_payload": sp.tolist(),
                     "sorted_keys": rk.tolist(), "sorted_payload": rp.tolist(), "scan_in": v.tolist(),
                     "scan_out": sc.tolist()})
    g["primitives"] = prim

    # index queries (locate, prefix_related, start_rank_list) incl. double_cut instances
    idx_cases = []
    instances = [([b"GATT", b"ACA", b"GGT", b"GA", b"TTAC", b"AGGT"], "dna"),
                 ([b"ab", b"cd", b"efgh", b"abcdef", b"gh"], "generic_byte"),
                 ([b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"], "generic_byte")]
    for _ in range(6):
        L = int(rng.integers(20, 90))
        seq = bytes(rng.choice([65, 67, 71, 84], L).astype(np.uint8))
        cap = max(1, L // 8)
        frags = ref.double_cut(seq, int(rng.integers(0, cap)), 1 + int(rng.integers(0, cap)),
                               int(rng.integers(0, 1 << 30)), int(rng.integers(0, 1 << 30)))
        instances.append((frags, "dna"))
    for frags, alpha in instances:
        ix = ref.index(frags, alpha, builder=1, workers=2, chunk=64)
        concat, starts, sa, rank, srl = ix.arrays()
        queries = []
        pats = [f[int(rng.integers(0, len(f))):] for f in frags] + [b"GA", b"QQ", b"TT", b"A", b"cdef", b"b"]
        for p in pats:
            lo, hi = ix.locate(p)
            a, b, c = ix.prefix_related(p)
            queries.append({"pattern": list(p), "lo": lo, "hi": hi, "prefixes": a.tolist(),
                            "extensions": b.tolist(), "exact": c.tolist()})
        idx_cases.append({"fragments": [list(f) for f in frags], "alphabet": alpha, "sa": sa.tolist(),
                          "start_rank_list": srl.tolist(), "queries": queries})
        ix.close()
    g["index"] = idx_cases

    # overlap graph + greedy (overlap.hpp) -- no test file in the reference pins these
    ov_cases = []
    sets = [([b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"], "generic_byte")]
    for it in range(14):
        G = int(rng.integers(20, 90))
        genome = rng.choice([65, 67] if it % 2 else [65, 67, 71, 84], G).astype(np.uint8)
        frags = []
        for _ in range(int(rng.integers(3, 14))):
            ln = min(G, int(rng.integers(3, 16)))
            s0 = int(rng.integers(0, G - ln + 1))
            frags.append(bytes(genome[s0:s0 + ln]))
        sets.append((frags, "dna"))
    for frags, alpha in sets:
        w = ref.overlap_graph(frags, alpha)
        sup, order = ref.greedy(frags, alpha)
        keep = ref.absorb_contained(frags, alpha)
        ov_cases.append({"fragments": [list(f) for f in frags], "alphabet": alpha, "weight": w.tolist(),
                         "superstring": list(sup), "order": order.tolist(), "kept": keep.tolist()})
    g["overlap"] = ov_cases
    g["overlap_weight_spec"] = [
        {"a": list(b"abthatb"), "b": list(b"tbabhhatbpaa"), "w": ref.overlap_weight(b"abthatb", b"tbabhhatbpaa")},
        {"a": list(b"hatbpaab"), "b": list(b"paabtabh"), "w": ref.overlap_weight(b"hatbpaab", b"paabtabh")},
        {"a": list(b"AAA"), "b": list(b"TTT"), "w": ref.overlap_weight(b"AAA", b"TTT")}]

    out = Path(__file__).with_name("golden.json")
    out.write_text(json.dumps(g, separators=(",", ":")))
    print(out, out.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
