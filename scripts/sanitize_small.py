"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family once, on inputs small enough for the tool's slowdown.  Asserts parity like the tests do."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1404_3456_b200 as rq
from tests.oracle_lib import Oracle

ora = Oracle()
ex = rq.Executor(0)
rng = np.random.default_rng(1)

def check(text, e=ex):
    got = rq.build_parallel(text, e)
    wsa, wrank = ora.build_sa(text)
    assert np.array_equal(got.sa, wsa) and np.array_equal(got.rank, wrank)
    return got

# uniform read sets: clean, with repeats (refine), at partitioned-inverse size
text, starts = rq.synth_read_text(40_000, 100, 4_000)
assert check(text).stats.init_symbols == 16
unit = bytes(rng.choice([65, 67, 71, 84], 3000).astype(np.uint8))
genome = unit + unit[:1500] + unit
reads = b"".join(genome[int(s):int(s) + 60] + b"\0" for s in rng.integers(0, len(genome) - 60, 3000))
check(np.frombuffer(reads, np.uint8))
big, _ = rq.synth_read_text(400_000, 100, 42_000)          # n = 4.24 M >= 2^22: partition passes + window scatter
got = rq.build_parallel(big, ex)
assert np.array_equal(got.rank[got.sa], np.arange(big.size, dtype=np.uint32)) and ora.verify_sa(big, got.sa) == 0
# ragged read sets (mixed read lengths: transposed records with ragged rows, forward / backward links), with repeats
g40 = rng.choice([65, 67, 71, 84], 40_000).astype(np.uint8)
def ragged_reads(genome, k, lo, hi):
    out = []
    for _ in range(k):
        ln = int(rng.integers(lo, hi + 1)); st = int(rng.integers(0, len(genome) - ln + 1))
        out.append(bytes(genome[st:st + ln]) + b"\0")
    return np.frombuffer(b"".join(out), np.uint8)
assert check(ragged_reads(g40, 3000, 40, 150)).stats.init_symbols == 15
assert check(ragged_reads(np.frombuffer(genome, np.uint8), 3000, 16, 254)).stats.init_symbols == 15
# general DNA records, text steps, prefix doubling (local rounds, global rounds, oversize groups), generic bytes
ragged = rng.choice([65, 67, 71, 84, 0], 60_000, p=[.24, .24, .24, .24, .04]).astype(np.uint8)
check(ragged)
e2 = rq.Executor(0); e2.set_option("sa_text_rounds", 0); check(ragged, e2); check(text, e2)
check(np.frombuffer((b"ACGTACGTAC" * 12 + b"\0") * 3000, np.uint8), e2)       # groups of 3000 > the local window
e4 = rq.Executor(0); e4.set_option("sa_text_rounds", 0); e4.set_option("sa_doubling_local", 0); check(text, e4)
e3 = rq.Executor(0); e3.set_option("sa_uniform", 0); check(text, e3)
e5 = rq.Executor(0); e5.set_option("sort_tma", 1); check(text, e5)             # TMA tile loads in the sort
check(text); check(text)                                                       # speculative route (second and third build)
check(np.frombuffer(b"abthatb\0hatbpaab\0tbabhhatbpaa\0paabtabh\0bhaabtpb\0" * 50, np.uint8))
check(np.frombuffer(b"A" * 5000, np.uint8))
# primitives
keys = rng.integers(0, 2**32, 50_000, dtype=np.uint64).astype(np.uint32)
pay = np.arange(keys.size, dtype=np.uint32)
k2, p2 = rq.radix_sort(keys, pay, ex)
order = np.argsort(keys, kind="stable")
assert np.array_equal(k2, keys[order]) and np.array_equal(p2, pay[order])
assert np.array_equal(rq.exclusive_scan(np.ones(70_000, np.uint32), ex), np.arange(70_000, dtype=np.uint32))
d, tof = rq.split_destinations(keys, 3, ex)
wd, wtof = ora.split_destinations(keys, 3)
assert tof == wtof and np.array_equal(d, wd) and not rq.is_sorted(keys, ex) and rq.is_sorted(k2, ex)
# index, queries, overlaps, merge
fs = rq.fragment_set_from_text(text, starts)
ix = rq.FragmentIndex(fs, ex)
ov = ix.overlaps(20)
lens = fs.lengths()
wi, wj, ww = ora.overlap_list(fs.concat, fs.starts, lens, 20)
assert np.array_equal(ov.i, wi) and np.array_equal(ov.j, wj) and np.array_equal(ov.w, ww)
sup, order = rq.greedy_superstring_from_overlaps(fs, ov)
assert len(sup) > 0
ov2 = ix.overlaps(20, reuse_buffers=True)
assert np.array_equal(ov2.i, wi) and np.array_equal(ov2.w, ww)
e6 = rq.Executor(0); e6.set_option("overlap_stage", 1)                         # TMA-staged rank blocks in the overlap search
ix6 = rq.FragmentIndex(fs, e6); ov6 = ix6.overlaps(20)
assert np.array_equal(ov6.i, wi) and np.array_equal(ov6.w, ww)
pr = ix.prefix_related_batch([0, 1, 2], [0, 5, 10])
assert len(pr) == 3
dup = rq.make_fragment_set([b"ACGT" * 10] * 120 + [b"CGTA" * 10] * 40, "dna")     # overflow route of the overlap fill
ixd = rq.FragmentIndex(dup, ex)
ovd = ixd.overlaps(4)
di, dj, dw = ora.overlap_list(dup.concat, dup.starts, dup.lengths(), 4)
assert np.array_equal(ovd.i, di) and np.array_equal(ovd.j, dj) and np.array_equal(ovd.w, dw)
rel = ix.prefix_related_patterns([fs.bytes(0)[:30], fs.bytes(1), b"ACGTACGTAC"])
assert len(rel) == 3
import os
if os.environ.get("SANITIZE_NO_SHARDED"):
    print("sanitize_small: all parity checks passed (sharded part skipped)")
    raise SystemExit(0)
# the sharded build of a uniform read set as three virtual ranks
import threading, torch
from paper_1404_3456_b200.sharded import GpuBackend, LocalComm, build_sa_sharded
want = rq.build_parallel(text, ex)
for uniform in (True, False):          # bucket generators of both record kinds, rank exchange, slice inverse
    d_text = torch.from_numpy(np.array(text, copy=True)).cuda()
    comms, outs = LocalComm.make(3), [None] * 3
    def work(r):
        e = rq.Executor(0)
        if not uniform:
            e.set_option("sa_uniform", 0)
        st = {}
        sa, rk = build_sa_sharded(d_text, comms[r], GpuBackend(e), st)
        torch.cuda.synchronize()
        outs[r] = (sa.cpu().numpy().view(np.uint32), rk.cpu().numpy().view(np.uint32), st)
        e.close()
    th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
    [t.start() for t in th]; [t.join() for t in th]
    for sa, rk, st in outs:
        assert st["path"] == "sharded" and st["records"] == ("uniform" if uniform else "general")
        assert np.array_equal(sa, want.sa) and np.array_equal(rk, want.rank)
print("sanitize_small: all parity checks passed")
