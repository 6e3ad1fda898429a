"""Host logic of the multi-GPU path under REAL collectives: two processes, gloo backend, CPU
tensors.  The per-rank kernels are replaced by a numpy stand-in (NumpyBackend below, checker-grade
code that leans on the oracle), so what is exercised is sharded.py itself: read / position slicing,
splitter selection from the all-reduced prefix histogram, bucket-local record generation and the
ordering guarantee the bucket sort relies on, the combined proof table, the all-to-all of the
(position, index) records that shards rank by position, the gather into place and the fallbacks."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def records_of(text: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """numpy restatement of the 64-bit suffix record of csrc/sa.cu: key24 << 40 | p8 << 32 | pos.
    key24: bases 0..7 in the upper 16 bits; low digit = 0x80 | bases 8..10 | upper bit of base 11
    for suffixes of more than 8 symbols, 2*t + kind for those terminating after t <= 8 symbols."""
    n = text.size
    code = np.zeros(256, np.int64)
    code[[65, 67, 71, 84]] = [0, 1, 2, 3]
    out = np.zeros(hi - lo, np.int64)
    for i, pos in enumerate(range(lo, hi)):
        t = 0
        while pos + t < n and text[pos + t] != 0 and t < 256:
            t += 1
        if pos + t < n and t < 256:
            tt, kind = t, 1                      # a sentinel comes first
        elif n - pos <= 256:
            tt, kind = n - pos, 0                # the text ends first
        else:
            tt, kind = 256, 1
        bases = 0
        for b in range(min(tt, 12)):
            bases |= int(code[text[pos + b]]) << (2 * (11 - b))
        if tt <= 8:
            key, p = ((bases >> 8) << 8) | (2 * tt + kind), 2 * tt + kind
        else:
            b23 = bases >> 1
            key = ((b23 >> 7) << 8) | 0x80 | (b23 & 0x7F)
            if tt < 11:
                p = 2 * tt + kind
            elif tt == 256:
                p = 254
            elif kind == 0:
                p = 255
            else:
                p = tt + 11 if tt + 11 <= 253 else 254
        v = (key << 40) | (p << 32) | pos
        out[i] = v - (1 << 64) if v >= (1 << 63) else v
    return out


def uniform_records_of(text: np.ndarray, period: int, read_begin: int, read_count: int) -> np.ndarray:
    """numpy restatement of gen_uniform_kernel (csrc/sa.cu): key32 << 32 | pos, key32 = the first 16
    bases zero padded from the sentinel on; record t * read_count + r = suffix of read read_begin + r
    with t symbols before its sentinel."""
    code = np.zeros(256, np.int64)
    code[[65, 67, 71, 84]] = [0, 1, 2, 3]
    out = np.zeros(read_count * period, np.int64)
    for t in range(period):
        for r in range(read_count):
            pos = (read_begin + r) * period + (period - 1 - t)
            key = 0
            for b in range(min(t, 16)):
                key |= int(code[text[pos + b]]) << (2 * (15 - b))
            v = (key << 32) | pos
            out[t * read_count + r] = v - (1 << 64) if v >= (1 << 63) else v
    return out


class NumpyBackend:
    def __init__(self, oracle_rank, uniform=False):
        self.oracle_rank = oracle_rank   # inverse SA of the whole text from the oracle
        self.uniform = uniform

    def open(self, d_text):
        self.text = d_text.numpy()
        return bool(np.isin(self.text, [0, 65, 67, 71, 84]).all())

    def close(self):
        pass

    def uniform_info(self):
        if not self.uniform:
            return None
        seps = np.flatnonzero(self.text == 0)
        period = int(seps[0]) + 1
        assert np.array_equal(seps, np.arange(seps.size) * period + period - 1)
        return period, int(seps.size)

    def _all_records(self):
        if not hasattr(self, "_recs"):
            if self.uniform:
                period, reads = self.uniform_info()
                self._recs = uniform_records_of(self.text, period, 0, reads)            # (t, read) order
                self._prefix = (self._recs >> 52) & 0xFFF
            else:
                self._recs = records_of(self.text, 0, self.text.size)                   # position order
                self._prefix = (self._recs >> 52) & 0xFFF
        return self._recs, self._prefix

    def prefix_hist(self, unit_begin, unit_count):
        recs, prefix = self._all_records()
        pos = recs & 0xFFFFFFFF
        if self.uniform:
            period = self.uniform_info()[0]
            mine = (pos // period >= unit_begin) & (pos // period < unit_begin + unit_count)
        else:
            mine = (pos >= unit_begin) & (pos < unit_begin + unit_count)
        return torch.from_numpy(np.bincount(prefix[mine], minlength=1 << 12).astype(np.int64))

    def bucket(self, plo, phi):
        recs, prefix = self._all_records()
        return torch.from_numpy(recs[(prefix >= plo) & (prefix < phi)].copy())

    def uniform_sort_link(self, records, reads):
        r = records.numpy()
        period = self.uniform_info()[0]
        p = r & 0xFFFFFFFF
        t = (period - 1) - p % period
        # the contract the stable digit passes rely on: the bucket is born in (t, position) order
        assert np.all((t[1:] > t[:-1]) | ((t[1:] == t[:-1]) & (p[1:] > p[:-1]))), "bucket not in (t, position) order"
        self._bucket = p
        cov = np.zeros(reads, np.uint8)
        cov[(p[t == period - 1] // period)] = 1      # this rank proves things about the whole reads it holds
        return torch.from_numpy(cov)

    def uniform_finish(self, cov):
        # every whole read lies in exactly one bucket: the all-reduce MAX must have merged all tables
        assert bool(torch.all(cov == 1)), "per-read tables were not combined across ranks"
        p = self._bucket
        by_suffix = p[np.argsort(self.oracle_rank[p], kind="stable")]
        return torch.from_numpy(by_suffix.astype(np.int32)), 0

    def finish(self, records):
        r = records.numpy()
        p = r & 0xFFFFFFFF
        assert np.all(p[1:] > p[:-1]), "general records must be born in position order"
        by_suffix = p[np.argsort(self.oracle_rank[p], kind="stable")]
        return torch.from_numpy(by_suffix.astype(np.int32)), 0

    def rank_records(self, bucket, offset, n, world):
        p = bucket.numpy().astype(np.int64) & 0xFFFFFFFF
        base = np.array([(n * g) // world for g in range(world + 1)], np.int64)
        owner = np.searchsorted(base, p, side="right") - 1
        order = np.argsort(owner, kind="stable")[::-1].copy()          # any order inside an owner's group is allowed
        order = order[np.argsort(owner[order], kind="stable")]
        recs = ((p - base[owner]) << 32) | (offset + np.arange(p.size, dtype=np.int64))
        return torch.from_numpy(recs[order].copy()), [int(c) for c in np.bincount(owner, minlength=world)]

    def rank_finish(self, records, slice_len):
        r = records.numpy()
        assert r.size == slice_len, "a position slice must receive exactly its own records"
        p, v = r >> 32, r & 0xFFFFFFFF
        assert np.array_equal(np.sort(p), np.arange(slice_len)), "records are not a permutation of the slice"
        out = np.empty(slice_len, np.int64)
        out[p] = v
        return torch.from_numpy(out.astype(np.int32))

    def full_build(self, d_text):
        sa = np.argsort(self.oracle_rank, kind="stable")
        return torch.from_numpy(sa.astype(np.int32)), torch.from_numpy(self.oracle_rank.astype(np.int32))


def worker(rank, world, port, text_bytes, oracle_rank, out_dir, uniform=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1404_3456_b200.sharded import TorchComm, build_sa_sharded
    comm = TorchComm()
    d_text = torch.from_numpy(np.frombuffer(text_bytes, np.uint8).copy())
    stats = {}
    from paper_1404_3456_b200.sharded import build_sa_sharded_parts
    parts = build_sa_sharded_parts(d_text, comm, NumpyBackend(oracle_rank, uniform), stats)
    np.save(Path(out_dir) / f"bucket{rank}.npy", parts.sa_bucket.numpy())      # what stays sharded ...
    np.save(Path(out_dir) / f"slice{rank}.npy", parts.rank_slice.numpy())
    assert parts.sa_offset == sum(parts.bucket_sizes[:rank]) and parts.rank_base == (d_text.numel() * rank) // world
    sa, rk = parts.replicate(comm)                                             # ... and the gather into place
    np.save(Path(out_dir) / f"sa{rank}.npy", sa.numpy())
    np.save(Path(out_dir) / f"rank{rank}.npy", rk.numpy())
    (Path(out_dir) / f"stats{rank}.txt").write_text(
        f"{stats['path']} {stats.get('bucket', 0)} {stats.get('sent', 0)} {stats.get('records', '-')}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,uniform", [(2, False), (2, True)])
def test_sample_sort_exchange_under_gloo(oracle, tmp_path, world, uniform):
    """uniform: slices of READS, transposed 16-base records, the bucket re-ordered on the terminator
    distance after the exchange, per-read tables combined by an all-reduce MAX."""
    rng = np.random.default_rng(11)
    genome = rng.choice([65, 67, 71, 84], 900).astype(np.uint8)
    reads = [bytes(genome[s:s + 40]) + b"\0" for s in rng.integers(0, 860, 120)]
    text = np.frombuffer(b"".join(reads), np.uint8)
    want_sa, want_rank = oracle.build_sa(text)
    port = 29500 + int(rng.integers(0, 2000)) + (7 if uniform else 0)
    mp.spawn(worker, args=(world, port, text.tobytes(), want_rank.astype(np.int64), str(tmp_path), uniform),
             nprocs=world, join=True)
    buckets = []
    for r in range(world):
        sa = np.load(tmp_path / f"sa{r}.npy").view(np.uint32)
        rk = np.load(tmp_path / f"rank{r}.npy").view(np.uint32)
        assert np.array_equal(sa, want_sa) and np.array_equal(rk, want_rank)
        path, bucket, sent, records = (tmp_path / f"stats{r}.txt").read_text().split()
        assert path == "sharded" and int(sent) > 0 and records == ("uniform" if uniform else "general")
        buckets.append(int(bucket))
    assert sum(buckets) == text.size and min(buckets) > text.size // 4   # balanced by the splitters
    # the sharded form: buckets concatenate to sa, position slices to rank
    assert np.array_equal(np.concatenate([np.load(tmp_path / f"bucket{r}.npy").view(np.uint32) for r in range(world)]), want_sa)
    assert np.array_equal(np.concatenate([np.load(tmp_path / f"slice{r}.npy").view(np.uint32) for r in range(world)]), want_rank)


def test_bounds_are_balanced_and_monotone():
    sys.path.insert(0, str(ROOT))
    from paper_1404_3456_b200.sharded import choose_bounds
    rng = np.random.default_rng(5)
    hist = torch.from_numpy(rng.integers(0, 50, 1 << 12))
    for G in (2, 3, 4, 8):
        b = choose_bounds(hist, G)
        assert len(b) == G - 1 and all(y >= x for x, y in zip(b, b[1:]))
        edges = [0] + [int(x) for x in b] + [1 << 12]
        loads = [int(hist[edges[g]:edges[g + 1]].sum()) for g in range(G)]
        assert max(loads) - min(loads) <= 2 * 50 + int(hist.sum()) // (50 * G)
    skew = torch.zeros(1 << 12, dtype=torch.int64)
    skew[7] = 1000                       # everything in one prefix: one rank takes it all, no crash
    b = choose_bounds(skew, 4)
    assert all(y >= x for x, y in zip(b, b[1:]))
