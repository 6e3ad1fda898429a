"""Multi-GPU form of the hot path: one process per GPU.

  SA build       sample sort on the record key.  The text is replicated (2-bit packed it is n/4
                 bytes), so NO suffix record travels:
                   1. every rank histograms the 12-bit key prefix (6 bases) of the suffixes of ITS 1/G
                      slice (reads of a uniform read set, positions otherwise); one all-reduce SUM of
                      4096 counters; the G-1 splitters are read off the cumulative counts;
                   2. every rank makes the records of its own splitter range straight from the
                      replicated text, already in the order the stable digit passes start from
                      (a count sweep + scan + write sweep over all suffix keys: the only step that
                      does not shrink with G; ~2 % of a single-GPU build);
                   3. it finishes its bucket with the single-GPU kernels.  Uniform read sets: 4 digit
                      passes, one verified overlap per whole read in the bucket into a per-read table,
                      the ranks' tables combined by an all-reduce MAX (k bytes), accept / refine.  Other
                      DNA texts: 3 passes + shared-memory refinement.  The buckets, in splitter order,
                      ARE the suffix array: it stays sharded;
                   4. rank (the inverse) is sharded by POSITION: each rank turns its bucket into
                      (position - owner's base, global index) records grouped by owner -- ONE all-to-all
                      (NCCL over NVLink: the path's real exchange step, 8 bytes per suffix) -- and the
                      owner scatters its slice with the partitioned inverse of the single-GPU build;
                   5. only when a replica is asked for (the query phase) are sa and rank gathered,
                      each part broadcast straight into its place in the final buffer.
  Overlap search reads partitioned contiguously across ranks against the replicated index; no
                 collective on the query path; per-rank lists concatenate in read order.
  Greedy merge   host, rank 0 (not sharded: global tie-breaking, overlap.hpp:91-108).

Results are byte-identical for every G (and equal to the single-GPU build).  The collectives go
through a small `Comm` interface: `TorchComm` (torch.distributed: NCCL on GPUs, gloo in the CPU
tests) or `LocalComm` (G threads in one process: virtual ranks sharing one GPU, used by the
single-GPU tests).  The per-rank compute goes through a backend object: `GpuBackend` (the C ABI);
the CPU tests substitute a numpy stand-in to exercise the orchestration under gloo.  The library
launches on torch's current stream (Executor.set_stream), so its kernels, torch's copies and NCCL's
collectives are ordered by stream semantics alone.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .api import Executor, FragmentIndex, FragmentSet, OverlapList

PREFIX_BITS = 12   # splitters are chosen on the top 12 key bits (6 bases): kShPrefixBits in csrc/sa.cu


# ---- collectives --------------------------------------------------------------------------------

class TorchComm:
    """torch.distributed (backend nccl for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def all_to_all_v(self, send: torch.Tensor, send_counts: Sequence[int]):
        counts = torch.tensor(list(send_counts), dtype=torch.int64, device=send.device)
        recv_counts = torch.empty_like(counts)
        self.dist.all_to_all_single(recv_counts, counts, group=self.group)
        rc = [int(x) for x in recv_counts.tolist()]
        recv = torch.empty(sum(rc), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=list(send_counts),
                                    group=self.group)
        return recv, rc

    def all_gather_sizes(self, m: int, device) -> list:
        """Every rank's `m` (one small collective; the only host read is of its G results)."""
        mine = torch.tensor([int(m)], dtype=torch.int64, device=device)
        out = torch.empty(self.world, dtype=torch.int64, device=device)
        self.dist.all_gather_into_tensor(out, mine, group=self.group)
        return [int(x) for x in out.tolist()]

    def all_gather_v(self, t: torch.Tensor, sizes: Sequence[int]) -> torch.Tensor:
        """Concatenation of the ranks' parts (sizes known): every part is broadcast straight into its
        place in the final buffer -- no padding, no second copy."""
        out = torch.empty(int(sum(sizes)), dtype=t.dtype, device=t.device)
        off = 0
        for src, sz in enumerate(sizes):
            view = out[off:off + sz]
            if src == self.rank:
                view.copy_(t)
            if sz:
                self.dist.broadcast(view, src=self.dist.get_global_rank(self.group, src) if self.group is not None else src,
                                    group=self.group)
            off += sz
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)


class LocalComm:
    """G virtual ranks as threads of one process (they may share one GPU)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "LocalComm._Shared", rank: int):
        self.s = shared
        self.rank = rank
        self.world = shared.world

    @staticmethod
    def make(world: int):
        shared = LocalComm._Shared(world)
        return [LocalComm(shared, r) for r in range(world)]

    def _exchange(self, value):
        self.s.slots[self.rank] = value
        self.s.barrier.wait()
        got = list(self.s.slots)
        self.s.barrier.wait()
        return got

    def all_reduce_sum(self, t):
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        total = sum(x.clone() for x in self._exchange(t.clone()))
        t.copy_(total)
        return t

    def all_reduce_max(self, t):
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        parts = self._exchange(t.clone())
        total = parts[0].clone()
        for x in parts[1:]:
            total = torch.maximum(total, x)
        t.copy_(total)
        return t

    def all_to_all_v(self, send, send_counts):
        if send.is_cuda:
            torch.cuda.current_stream().synchronize()
        offs = np.concatenate(([0], np.cumsum(send_counts)))
        chunks = [send[int(offs[r]):int(offs[r + 1])].clone() for r in range(self.world)]
        everyone = self._exchange(chunks)
        mine = [everyone[src][self.rank] for src in range(self.world)]
        return torch.cat(mine), [int(c.numel()) for c in mine]

    def all_gather_sizes(self, m, device):
        return [int(x) for x in self._exchange(int(m))]

    def all_gather_v(self, t, sizes):
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        return torch.cat([x.clone() for x in self._exchange(t.clone())])

    def barrier(self):
        self.s.barrier.wait()


# ---- per-rank compute ------------------------------------------------------------------------------

def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


class GpuBackend:
    """The C-ABI building blocks of one rank (include/reseq_cuda.h, "multi-GPU building blocks").  Every
    call is queued on the executor's stream -- torch's current stream when the executor was given it
    (set_stream) -- so nothing here synchronises except where a size has to reach the host."""

    def __init__(self, ex: Executor, device: Optional[torch.device] = None, bind_stream: bool = True):
        self.ex = ex
        self.lib = ex._lib
        self.device = device or torch.device("cuda", ex.device)
        self.shard = None
        if bind_stream:
            # the library's kernels must be ordered with torch's allocations / copies and with the
            # collectives torch enqueues: all of them on the stream that is current now (handle 0 =
            # torch's default stream is passed on as the legacy default stream, not as "own stream")
            ex.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def open(self, d_text: torch.Tensor) -> bool:
        """Packs the replicated text; False when it is not a 2-bit DNA text."""
        h = C.c_void_p()
        dna = C.c_int(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_create(self.ex.handle, _p(d_text), d_text.numel(), C.byref(h),
                                                       C.byref(dna)))
        self.shard = h
        self._text = d_text
        return bool(dna.value)

    def close(self):
        if self.shard is not None:
            self.lib.reseq_cuda_sa_shard_destroy(self.shard)
            self.shard = None

    def uniform_info(self):
        """(period, reads) when the text is k reads of one length, else None."""
        period, reads = C.c_uint32(0), C.c_uint64(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_info(self.shard, C.byref(period), C.byref(reads)))
        return (int(period.value), int(reads.value)) if period.value else None

    def prefix_hist(self, unit_begin: int, unit_count: int) -> torch.Tensor:
        h = torch.empty(1 << PREFIX_BITS, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.reseq_cuda_sa_shard_prefix_hist(self.shard, unit_begin, unit_count, _p(h)))
        return h.to(torch.int64)

    def bucket(self, prefix_lo: int, prefix_hi: int) -> torch.Tensor:
        """The records of this rank's splitter range, in sort-ready order."""
        m = C.c_uint64(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_bucket_size(self.shard, prefix_lo, prefix_hi, C.byref(m)))
        r = torch.empty(int(m.value), dtype=torch.int64, device=self.device)
        _lib.check(self.lib.reseq_cuda_sa_shard_bucket_records(self.shard, _p(r)))
        return r

    def uniform_sort_link(self, records: torch.Tensor, reads: int) -> torch.Tensor:
        cov = torch.zeros(reads, dtype=torch.uint8, device=self.device)
        self._bucket = records     # sorted in place / ping-pong: must stay alive until uniform_finish
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_sort_link(self.shard, _p(records), records.numel(), _p(cov)))
        return cov

    def uniform_finish(self, cov: torch.Tensor):
        m = self._bucket.numel()
        sa = torch.empty(m, dtype=torch.int32, device=self.device)
        unfinished = C.c_uint64(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_finish(self.shard, _p(cov), _p(sa), C.byref(unfinished)))
        self._bucket = None
        return sa, int(unfinished.value)

    def finish(self, records):
        m = records.numel()
        sa = torch.empty(m, dtype=torch.int32, device=self.device)
        unfinished = C.c_uint64(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_finish(self.shard, _p(records), m, _p(sa), C.byref(unfinished)))
        return sa, int(unfinished.value)

    def rank_records(self, bucket: torch.Tensor, offset: int, n: int, world: int):
        """(position - owner's base) << 32 | global index, grouped by owner; per-owner counts."""
        out = torch.empty(bucket.numel(), dtype=torch.int64, device=self.device)
        counts = (C.c_uint64 * world)()
        _lib.check(self.lib.reseq_cuda_rank_shard_partition(self.ex.handle, _p(bucket), bucket.numel(), offset, n, world,
                                                            _p(out), counts))
        return out, [int(c) for c in counts]

    def rank_finish(self, records: torch.Tensor, slice_len: int) -> torch.Tensor:
        rank = torch.empty(slice_len, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.reseq_cuda_rank_shard_finish(self.ex.handle, _p(records), slice_len, _p(rank)))
        return rank

    def full_build(self, d_text):
        n = d_text.numel()
        sa = torch.empty(n, dtype=torch.int32, device=self.device)
        rank = torch.empty(n, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.reseq_cuda_build_sa_device(self.ex.handle, _p(d_text), n, _p(sa), _p(rank), None))
        return sa, rank


def choose_bounds(hist: torch.Tensor, world: int) -> list:
    """world-1 ascending prefix values b_g: rank g owns the key prefixes in [b_{g-1}, b_g).  Read off
    the cumulative histogram at total*g/world; identical on every rank because the histogram is."""
    cum = torch.cumsum(hist.to(torch.int64).cpu(), 0)
    total = int(cum[-1])
    targets = torch.tensor([(total * g) // world for g in range(1, world)], dtype=torch.int64)
    # first prefix whose cumulative count reaches the target, +1: that prefix stays on the left
    return [int(x) for x in (torch.searchsorted(cum, targets, right=False) + 1).tolist()]


class ShardedSuffixArray:
    """What one rank holds after the sharded build: its bucket of the suffix array (global indices
    [sa_offset, sa_offset + sa_bucket.numel())) and its position slice of rank (positions
    [rank_base, rank_base + rank_slice.numel()))."""

    def __init__(self, n, sa_bucket, sa_offset, bucket_sizes, rank_slice, rank_base, slice_sizes, replicated=None):
        self.n = n
        self.sa_bucket, self.sa_offset, self.bucket_sizes = sa_bucket, sa_offset, bucket_sizes
        self.rank_slice, self.rank_base, self.slice_sizes = rank_slice, rank_base, slice_sizes
        self._replicated = replicated

    def replicate(self, comm):
        """(sa, rank) complete on every rank: each part broadcast into its place."""
        if self._replicated is None:
            self._replicated = (comm.all_gather_v(self.sa_bucket, self.bucket_sizes),
                                comm.all_gather_v(self.rank_slice, self.slice_sizes))
        return self._replicated


def build_sa_sharded_parts(d_text: torch.Tensor, comm, backend, stats: Optional[dict] = None,
                           force_sharded: bool = False) -> ShardedSuffixArray:
    """Suffix array + inverse of the (replicated) text `d_text` (uint8), built by all ranks of `comm`
    and LEFT SHARDED: sa by splitter bucket, rank by position."""
    n = d_text.numel()
    G, r = comm.world, comm.rank
    stats = stats if stats is not None else {}
    dev = d_text.device
    if n == 0:
        e = torch.empty(0, dtype=torch.int32, device=dev)
        return ShardedSuffixArray(0, e, 0, [0] * G, e.clone(), 0, [0] * G, (e, e.clone()))
    dna = backend.open(d_text)
    try:
        def replicated(path):
            stats["path"] = path
            sa, rank = backend.full_build(d_text)
            lo, hi = (n * r) // G, (n * (r + 1)) // G
            sizes = [(n * (g + 1)) // G - (n * g) // G for g in range(G)]
            return ShardedSuffixArray(n, sa[lo:hi], lo, sizes, rank[lo:hi], lo, sizes, (sa, rank))

        if (G == 1 and not force_sharded) or not dna or n < 4 * G:   # (force_sharded: the whole pipeline with one rank -- a plumbing / cost check)
            return replicated("replicated")
        uniform = backend.uniform_info()
        if uniform is not None and uniform[1] < G:
            uniform = None
        units = uniform[1] if uniform is not None else n
        lo, hi = (units * r) // G, (units * (r + 1)) // G             # this rank's slice of reads / positions
        hist = comm.all_reduce_sum(backend.prefix_hist(lo, hi - lo))
        bounds = [0] + choose_bounds(hist, G) + [1 << PREFIX_BITS]
        records = backend.bucket(bounds[r], bounds[r + 1])
        m = int(records.numel())
        bucket_sizes = comm.all_gather_sizes(m, dev)
        stats["bucket"] = m
        stats["buckets"] = bucket_sizes
        if uniform is not None:
            cov = comm.all_reduce_max(backend.uniform_sort_link(records, uniform[1]))
            bucket, unfinished = backend.uniform_finish(cov)
            stats["records"] = "uniform"
        else:
            bucket, unfinished = backend.finish(records)
            stats["records"] = "general"
        del records
        flag = comm.all_reduce_sum(torch.tensor([unfinished], dtype=torch.int64, device=dev))
        if int(flag.item()) != 0:
            # a group outgrew the refine window somewhere: every rank builds the whole array
            return replicated("replicated-fallback")
        offset = int(sum(bucket_sizes[:r]))
        recs, counts = backend.rank_records(bucket, offset, n, G)
        mine, _ = comm.all_to_all_v(recs, counts)
        stats["sent"] = int(sum(counts) - counts[r])
        slice_sizes = [(n * (g + 1)) // G - (n * g) // G for g in range(G)]
        rank_slice = backend.rank_finish(mine, slice_sizes[r])
        stats["path"] = "sharded"
        return ShardedSuffixArray(n, bucket, offset, bucket_sizes, rank_slice, (n * r) // G, slice_sizes)
    finally:
        backend.close()


def build_sa_sharded(d_text: torch.Tensor, comm, backend, stats: Optional[dict] = None):
    """The sharded build followed by the gather: every rank returns the complete (sa, rank) as int32
    tensors (bit patterns of u32) -- what the replicated query phase needs."""
    return build_sa_sharded_parts(d_text, comm, backend, stats).replicate(comm)


def overlaps_sharded(fset: FragmentSet, comm, ex: Executor, min_overlap: int = 20,
                     index: Optional[FragmentIndex] = None) -> OverlapList:
    """This rank's share of the overlap list: the reads [k*r/G, k*(r+1)/G) queried against the
    replicated index.  `gather_overlaps` concatenates the shares in read order."""
    ix = index or FragmentIndex(fset, ex)
    k = fset.starts.size
    lo, hi = (k * comm.rank) // comm.world, (k * (comm.rank + 1)) // comm.world
    return ix.overlaps(min_overlap, lo, hi)


def gather_overlaps(parts: Sequence[OverlapList]) -> OverlapList:
    """Concatenation of per-rank shares (ranks own ascending, disjoint read ranges, and every share
    is (i, j)-sorted, so the concatenation is the global (i, j)-sorted list)."""
    return OverlapList(np.concatenate([p.i for p in parts]), np.concatenate([p.j for p in parts]),
                       np.concatenate([p.w for p in parts]),
                       np.maximum.reduce([p.contained for p in parts]),
                       sum(p.queries for p in parts), max(p.device_ms for p in parts), parts[0].min_overlap)


# ---- bench entry (torchrun, N > 1; or --force-sharded on one GPU) ---------------------------------

def bench_main(args, workload: str, rank: int, world: int, local_rank: int) -> None:
    """bench.py --gpus N: the SA of ONE text built by N ranks (strong scaling on the named workload),
    left sharded (sa by bucket, rank by position slice).  `value`: text resident in HBM, CUDA events on
    the launching stream between barriers, maximum over the ranks.  `e2e`: every step copies the text
    from pinned host memory and reads this rank's bucket and rank slice back to pinned host memory."""
    import json
    import time

    import torch.distributed as dist

    import bench as B
    from . import api as rq

    G_, L, k = B.WORKLOADS[workload]
    text, _ = rq.synth_read_text(G_, L, k, 1, 2, pinned=True)
    n = int(text.size)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    h_text = torch.from_numpy(text)
    d_text = h_text.to(dev, non_blocking=True)
    ex = Executor(local_rank)
    comm = TorchComm()
    force = world == 1
    stats = {}

    def step():
        return build_sa_sharded_parts(d_text, comm, GpuBackend(ex, dev), stats, force_sharded=force)

    for _ in range(max(3, args.warmup)):
        parts = step()
    ex.profile(True)
    launches0 = ex.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(local_rank) as clocks:   # nvidia-smi clocks / throttle reasons during the timed region
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            parts = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    prof = ex.profile_read()
    ex.profile(False)
    launches = ex.launch_count - launches0
    dt = torch.tensor([ev0.elapsed_time(ev1) * 1e-3], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    ms = float(dt.item()) / args.steps * 1e3

    # parity of what was just built: buckets and slices gathered once, rank must invert sa
    sa, rk = parts.replicate(comm)
    ok = True
    chunk = 1 << 27
    for b0 in range(0, n, chunk):
        b1 = min(n, b0 + chunk)
        idx = sa[b0:b1].to(torch.int64) & 0xFFFFFFFF
        ok = ok and bool(torch.equal(rk[idx].to(torch.int64) & 0xFFFFFFFF, torch.arange(b0, b1, device=dev, dtype=torch.int64)))
    del sa, rk, idx
    parts._replicated = None

    # e2e: H2D of the text + D2H of this rank's share of the result inside the timed region
    h_bucket = torch.empty(max(parts.bucket_sizes), dtype=torch.int32).pin_memory()
    h_slice = torch.empty(max(parts.slice_sizes), dtype=torch.int32).pin_memory()
    e2e_steps = max(3, min(args.steps, 5))
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        d_text.copy_(h_text, non_blocking=True)
        parts = step()
        h_bucket[: parts.sa_bucket.numel()].copy_(parts.sa_bucket, non_blocking=True)
        h_slice[: parts.rank_slice.numel()].copy_(parts.rank_slice, non_blocking=True)
        stream.synchronize()
    dist.barrier()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())

    if rank == 0:
        cpu = None if args.no_cpu else B.cpu_sa_baseline(text, L)
        line = {
            "metric": B.METRIC, "value": n / (ms * 1e-3) / 1e6, "unit": B.UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": B.DESCRIPTION[workload], "genome_bp": G_, "read_len": L, "reads": k, "suffixes": n,
                       "path": stats.get("path"), "records": stats.get("records"),
                       "bucket_sizes": stats.get("buckets"), "rank_records_sent_rank0": stats.get("sent"),
                       "result_layout": "sa sharded by splitter bucket, rank sharded by position slice (not gathered in the timed region)",
                       "l2_policy": f"inputs larger than L2 (record arrays {8 * n // max(1, world) / 1e6:.0f} MB per rank vs 126 MB L2)"},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "roofline": B.roofline_block(prof, n, L, args.steps, ms, workload, n_kernel=max(stats.get("buckets") or [n])),
            "cpu_baseline": cpu,
            "e2e": {"value": n / e2e_s / 1e6, "unit": B.UNIT, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                    "h2d_bytes_per_step": n * world, "d2h_bytes_per_step": 8 * n,
                    "note": "per step every rank copies the whole text host->device (replicated: n bytes x N) and its bucket of sa "
                            "+ its slice of rank device->host (8n bytes over all ranks)"},
            "checks": {"rank_is_inverse_of_sa": ok},
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
