"""The multi-GPU path (paper_1404_3456_b200/sharded.py) run as G virtual ranks -- threads of one
process sharing the one B200, each with its own context, exchanging through LocalComm.  Checks the
sample-sort partitioned build and the read-sharded overlap search bit-for-bit against the
single-GPU results for several G."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def run_ranks(G, fn):
    from paper_1404_3456_b200.sharded import LocalComm
    comms = LocalComm.make(G)
    out, err = [None] * G, [None] * G

    def work(r):
        try:
            out[r] = fn(comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e
            try:
                comms[r].s.barrier.abort()
            except Exception:
                pass

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out


def sharded_build(rq, text, G, uniform=True):
    from paper_1404_3456_b200.sharded import GpuBackend, build_sa_sharded
    d_text = torch.from_numpy(np.array(text, dtype=np.uint8, copy=True)).cuda()

    def fn(comm):
        ex = rq.Executor(0)
        if not uniform:
            ex.set_option("sa_uniform", 0)
        stats = {}
        sa, rank = build_sa_sharded(d_text, comm, GpuBackend(ex), stats)
        torch.cuda.synchronize()
        res = sa.cpu().numpy().view(np.uint32), rank.cpu().numpy().view(np.uint32), stats
        ex.close()
        return res

    return run_ranks(G, fn)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_build_equals_single_gpu(rq, ex, oracle, G):
    text, _ = rq.synth_read_text(60_000, 100, 6_000)
    want = rq.build_parallel(text, ex)
    assert oracle.verify_sa(text, want.sa) == 0
    for uniform in (True, False):    # the read-slice / proof-table route and the position-slice route
        res = sharded_build(rq, text, G, uniform)
        for sa, rank, stats in res:
            assert stats["path"] == "sharded" and stats["records"] == ("uniform" if uniform else "general")
            assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)
        # the buckets partition the suffixes: every rank sent and received something
        sizes = [s["bucket"] for _, _, s in res]
        assert sum(sizes) == text.size and min(sizes) > 0


@pytest.mark.parametrize("G,uniform", [(4, True), (3, False), (8, True)])
def test_sharded_parts_on_side_streams_at_config1_size(rq, ex, oracle, G, uniform):
    """The build LEFT SHARDED (sa by splitter bucket, rank by position slice) at BASELINE config 1's full
    size, every virtual rank on its own torch.cuda.Stream: the library's kernels, torch's allocations
    and copies and the exchange are ordered by that stream alone (no device-wide synchronisation in
    between), so a missing dependency shows up as a wrong array here."""
    from paper_1404_3456_b200.sharded import GpuBackend, build_sa_sharded_parts
    text, _ = rq.synth_read_text(1_000_000, 100, 100_000)
    n = text.size
    want = rq.build_parallel(text, ex)
    assert oracle.checksum_u32(want.sa) == 11642757783061468293
    d_text = torch.from_numpy(text).cuda()
    torch.cuda.synchronize()

    def fn(comm):
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            e = rq.Executor(0)
            if not uniform:
                e.set_option("sa_uniform", 0)
            stats = {}
            parts = build_sa_sharded_parts(d_text, comm, GpuBackend(e), stats)
            res = (parts.sa_bucket.cpu().numpy().view(np.uint32), parts.sa_offset, parts.rank_slice.cpu().numpy().view(np.uint32),
                   parts.rank_base, stats)
            side.synchronize()
            e.close()
        return res

    res = run_ranks(G, fn)
    assert all(st["path"] == "sharded" for *_, st in res)
    assert [off for _, off, _, _, _ in res] == list(np.cumsum([0] + [b.size for b, *_ in res[:-1]]))
    assert [base for _, _, _, base, _ in res] == [(n * g) // G for g in range(G)]
    assert np.array_equal(np.concatenate([b for b, *_ in res]), want.sa)
    assert np.array_equal(np.concatenate([r for _, _, r, _, _ in res]), want.rank)
    sizes = [b.size for b, *_ in res]
    assert max(sizes) < 1.25 * n / G            # the splitters balance the buckets


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_uniform_build_on_repeats_and_duplicates(rq, ex, oracle, G):
    """Groups that mix loci (re-sorted inside a bucket), duplicate reads, whole reads whose
    predecessor lives in another rank's slice of reads: the proof table must be complete after the
    all-reduce, and the result the single-GPU one."""
    rng = np.random.default_rng(91)
    unit = bytes(rng.choice([65, 67, 71, 84], 4000).astype(np.uint8))
    genome = unit + unit[:2000] + bytes(rng.choice([65, 67, 71, 84], 1500).astype(np.uint8)) + unit[1000:3000]
    starts = rng.integers(0, len(genome) - 80 + 1, 5000)
    reads = [genome[int(s):int(s) + 80] for s in starts]
    reads += reads[:300]
    text = np.frombuffer(b"".join(r + b"\0" for r in reads), np.uint8)
    want = rq.build_parallel(text, ex)
    assert oracle.verify_sa(text, want.sa) == 0
    for sa, rank, stats in sharded_build(rq, text, G):
        assert stats["records"] == "uniform"
        assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)


def test_sharded_build_ragged_and_tiny(rq, ex):
    rng = np.random.default_rng(3)
    t = rng.choice([65, 67, 71, 84, 0], 50_001, p=[.24, .24, .24, .24, .04]).astype(np.uint8)
    t[-1] = 0
    want = rq.build_parallel(t, ex)
    for sa, rank, stats in sharded_build(rq, t, 3):
        assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)
    tiny = np.frombuffer(b"GA\0TT\0", np.uint8)
    for sa, rank, stats in sharded_build(rq, tiny, 2):
        assert sa.tolist() == [2, 5, 1, 0, 4, 3] and stats["path"] == "replicated"


def test_sharded_build_fallbacks(rq, ex):
    generic = np.frombuffer(b"abthatb\0hatbpaab\0tbabhhatbpaa\0paabtabh\0bhaabtpb\0" * 20, np.uint8)
    want = rq.build_parallel(generic, ex)
    for sa, rank, stats in sharded_build(rq, generic, 2):
        assert stats["path"] == "replicated" and np.array_equal(sa, want.sa)
    big_groups = np.frombuffer((b"ACGTACGTAC" * 12 + b"\0") * 3000, np.uint8)   # groups of 3000 > refine window
    want = rq.build_parallel(big_groups, ex)
    for sa, rank, stats in sharded_build(rq, big_groups, 2, uniform=False):
        assert stats["path"] == "replicated-fallback"
        assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)
    for sa, rank, stats in sharded_build(rq, big_groups, 2):     # duplicates are proven, whatever the group size
        assert stats["path"] == "sharded" and stats["records"] == "uniform"
        assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)


@pytest.mark.parametrize("G", [2, 5])
def test_sharded_overlaps_equal_single_gpu(rq, ex, G):
    from paper_1404_3456_b200.sharded import gather_overlaps, overlaps_sharded
    text, starts = rq.synth_read_text(30_000, 80, 4_000)
    fset = rq.fragment_set_from_text(text, starts)
    ix = rq.FragmentIndex(fset, ex)
    want = ix.overlaps(16)
    def fn(comm):   # one context per rank: a context serves one host thread at a time
        e = rq.Executor(0)
        part = overlaps_sharded(fset, comm, e, 16)
        e.close()
        return part

    parts = run_ranks(G, fn)
    got = gather_overlaps(parts)
    assert np.array_equal(got.i, want.i) and np.array_equal(got.j, want.j) and np.array_equal(got.w, want.w)
    assert np.array_equal(got.contained, want.contained) and got.queries == want.queries
