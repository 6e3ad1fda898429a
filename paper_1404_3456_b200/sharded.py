"""Multi-GPU form of the hot path: one process per GPU.

  SA build       (uniform read sets -- k reads of one length -- take the same route with the
                 single-GPU fast path's kernels: transposed 16-base records of a slice of READS,
                 bucket brought back into (t, position) order after the exchange, one verified
                 overlap per whole read, per-read proof table combined by an all-reduce MAX.)
                 sample sort on the 24-bit initial key (12 bases).  The text is replicated (2-bit
                 packed it is n/4 bytes); every rank makes the 64-bit records (key24 << 40 |
                 terminator byte << 32 | position) of its 1/G slice of positions; G-1 splitters are
                 read off an all-reduced histogram of the key's top 16 bits; one ALL-TO-ALL moves
                 every record to the rank owning its splitter range; each rank finishes
                 its bucket with the single-GPU kernels (refinement keys come from the replicated
                 text, so no further exchange is needed); the buckets, concatenated in splitter
                 order, ARE the suffix array (all-gather); rank = local inverse.
  Overlap search reads partitioned contiguously across ranks against the replicated index; no
                 collective on the query path; per-rank lists concatenate in read order.
  Greedy merge   host, rank 0 (not sharded: global tie-breaking, overlap.hpp:91-108).

Results are byte-identical for every G (and equal to the single-GPU build).  The collectives go
through a small `Comm` interface: `TorchComm` (torch.distributed: NCCL on GPUs, gloo in the CPU
tests) or `LocalComm` (G threads in one process: virtual ranks sharing one GPU, used by the
single-GPU tests).  The per-rank compute goes through a backend object: `GpuBackend` (the C ABI);
the CPU tests substitute a numpy stand-in to exercise the exchange logic under gloo.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .api import Executor, FragmentIndex, FragmentSet, OverlapList

PREFIX_BITS = 16   # splitters are chosen on the top 16 bits (8 bases) of the record's 24-bit key
PREFIX_SHIFT = 64 - PREFIX_BITS


def record_prefix(records: torch.Tensor) -> torch.Tensor:
    """Top 16 key bits of int64-typed records (bit pattern of the u64 record)."""
    return (records >> PREFIX_SHIFT) & ((1 << PREFIX_BITS) - 1)


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

    def all_gather_v(self, t: torch.Tensor) -> torch.Tensor:
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes) if sizes else 0
        padded = torch.zeros(m, dtype=t.dtype, device=t.device)
        padded[: t.numel()] = t
        parts = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in range(self.world)]
        self.dist.all_gather(parts, padded, group=self.group)
        return torch.cat([p[:s] for p, s in zip(parts, sizes)])

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

    def all_gather_v(self, t):
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        return torch.cat([x.clone() for x in self._exchange(t.clone())])

    def barrier(self):
        self.s.barrier.wait()


# ---- per-rank compute ------------------------------------------------------------------------------

def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


class GpuBackend:
    """The C-ABI building blocks of one rank (include/reseq_cuda.h, "multi-GPU building blocks")."""

    def __init__(self, ex: Executor, device: Optional[torch.device] = None):
        self.ex = ex
        self.lib = ex._lib
        self.device = device or torch.device("cuda", ex.device)
        self.shard = None

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

    def records(self, pos_begin: int, count: int) -> torch.Tensor:
        r = torch.empty(count, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.reseq_cuda_sa_shard_records(self.shard, pos_begin, count, _p(r)))
        self.ex.synchronize()
        return r

    def prefix_histogram(self, records: torch.Tensor) -> torch.Tensor:
        return torch.bincount(record_prefix(records), minlength=1 << PREFIX_BITS)

    def partition(self, records, bounds: torch.Tensor):
        """Groups the records by destination rank, keeping their order inside each group.  The
        grouping itself is one stable pass of this library's radix sort on the rank id."""
        dest = torch.bucketize(record_prefix(records), bounds.to(records.device), right=True)
        counts = torch.bincount(dest, minlength=bounds.numel() + 1)
        dest32 = dest.to(torch.int32)
        idx = torch.arange(records.numel(), dtype=torch.int32, device=records.device)
        d_out, i_out = torch.empty_like(dest32), torch.empty_like(idx)
        if records.numel():
            _lib.check(self.lib.reseq_cuda_radix_sort_device(self.ex.handle, _p(dest32), _p(idx), records.numel(),
                                                             _p(d_out), _p(i_out)))
            self.ex.synchronize()
        order = i_out.to(torch.int64)
        return records[order].contiguous(), [int(c) for c in counts.tolist()]

    # -- uniform read sets ---------------------------------------------------------------------
    def uniform_info(self):
        """(period, reads) when the text is k reads of one length, else None."""
        period, reads = C.c_uint32(0), C.c_uint64(0)
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_info(self.shard, C.byref(period), C.byref(reads)))
        return (int(period.value), int(reads.value)) if period.value else None

    def uniform_records(self, read_begin: int, read_count: int) -> torch.Tensor:
        period, _ = self.uniform_info()
        r = torch.empty(read_count * period, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_records(self.shard, read_begin, read_count, _p(r)))
        self.ex.synchronize()
        return r

    def order_by_distance(self, records: torch.Tensor, period: int) -> torch.Tensor:
        """The slices of a bucket arrive source by source, each in (t, position) order; one stable
        pass of this library's radix sort on t = period - 1 - position mod period makes the whole
        bucket (t, position)-ordered (sources own ascending, disjoint position ranges)."""
        if records.numel() == 0:
            return records
        pos = records & 0xFFFFFFFF
        t32 = ((period - 1) - pos % period).to(torch.int32)
        idx = torch.arange(records.numel(), dtype=torch.int32, device=records.device)
        t_out, i_out = torch.empty_like(t32), torch.empty_like(idx)
        _lib.check(self.lib.reseq_cuda_radix_sort_device(self.ex.handle, _p(t32), _p(idx), records.numel(),
                                                         _p(t_out), _p(i_out)))
        self.ex.synchronize()
        return records[i_out.to(torch.int64)].contiguous()

    def uniform_sort_link(self, records: torch.Tensor, reads: int) -> torch.Tensor:
        cov = torch.zeros(reads, dtype=torch.uint8, device=self.device)
        self._bucket = records     # sorted in place / ping-pong: must stay alive until uniform_finish
        _lib.check(self.lib.reseq_cuda_sa_shard_uniform_sort_link(self.shard, _p(records), records.numel(), _p(cov)))
        self.ex.synchronize()
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

    def inverse(self, sa):
        rank = torch.empty_like(sa)
        _lib.check(self.lib.reseq_cuda_inverse_device(self.ex.handle, _p(sa), sa.numel(), _p(rank)))
        self.ex.synchronize()
        return rank

    def full_build(self, d_text):
        n = d_text.numel()
        sa = torch.empty(n, dtype=torch.int32, device=self.device)
        rank = torch.empty(n, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.reseq_cuda_build_sa_device(self.ex.handle, _p(d_text), n, _p(sa), _p(rank), None))
        self.ex.synchronize()
        return sa, rank


def choose_bounds(hist: torch.Tensor, world: int) -> torch.Tensor:
    """world-1 ascending prefix values b_g: rank g owns the key prefixes in [b_{g-1}, b_g).  Read off
    the cumulative histogram at total*g/world; identical on every rank because the histogram is."""
    cum = torch.cumsum(hist.to(torch.int64).cpu(), 0)
    total = int(cum[-1])
    targets = torch.tensor([(total * g) // world for g in range(1, world)], dtype=torch.int64)
    # first prefix whose cumulative count reaches the target, +1: that prefix stays on the left
    return torch.searchsorted(cum, targets, right=False) + 1


def build_sa_sharded(d_text: torch.Tensor, comm, backend, stats: Optional[dict] = None):
    """Suffix array + inverse of the (replicated) text `d_text` (uint8), built by all ranks of
    `comm`.  Every rank returns the complete (sa, rank) as int32 tensors (bit patterns of u32)."""
    n = d_text.numel()
    G, r = comm.world, comm.rank
    stats = stats if stats is not None else {}
    if n == 0:
        e = torch.empty(0, dtype=torch.int32, device=d_text.device)
        return e, e.clone()
    dna = backend.open(d_text)
    try:
        if G == 1 or not dna or n < 4 * G:
            stats["path"] = "replicated"
            return backend.full_build(d_text)
        uniform = backend.uniform_info() if hasattr(backend, "uniform_info") else None
        if uniform is not None and uniform[1] >= G:
            period, reads = uniform
            lo, hi = (reads * r) // G, (reads * (r + 1)) // G          # a slice of READS
            records = backend.uniform_records(lo, hi - lo)
        else:
            uniform = None
            lo, hi = (n * r) // G, (n * (r + 1)) // G                  # a slice of positions
            records = backend.records(lo, hi - lo)
        hist = comm.all_reduce_sum(backend.prefix_histogram(records))
        bounds = choose_bounds(hist, G)
        records, counts = backend.partition(records, bounds)
        mine, _ = comm.all_to_all_v(records, counts)
        stats["bucket"] = int(mine.numel())
        stats["sent"] = int(sum(counts) - counts[r])
        if uniform is not None:
            mine = backend.order_by_distance(mine, period)
            cov = comm.all_reduce_max(backend.uniform_sort_link(mine, reads))
            bucket, unfinished = backend.uniform_finish(cov)
            stats["records"] = "uniform"
        else:
            bucket, unfinished = backend.finish(mine)
            stats["records"] = "general"
        flag = comm.all_reduce_sum(torch.tensor([unfinished], dtype=torch.int64, device=d_text.device))
        if int(flag.item()) != 0:
            # a group outgrew the refine window somewhere: every rank builds the whole array
            stats["path"] = "replicated-fallback"
            return backend.full_build(d_text)
        sa = comm.all_gather_v(bucket)
        stats["path"] = "sharded"
        return sa, backend.inverse(sa)
    finally:
        backend.close()


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


# ---- bench entry (torchrun, N > 1) ---------------------------------------------------------------

def bench_main(args, workload: str, rank: int, world: int, local_rank: int) -> None:
    """bench.py --gpus N: the SA of ONE text built by N ranks (strong scaling on the named
    workload), timed as the max over ranks between barriers."""
    import json
    import time

    import torch.distributed as dist

    import bench as B
    from . import api as rq

    G_, L, k = B.WORKLOADS[workload]
    text, _ = rq.synth_read_text(G_, L, k, 1, 2)
    n = int(text.size)
    dev = torch.device("cuda", local_rank)
    d_text = torch.from_numpy(text).to(dev)
    ex = Executor(local_rank)
    ex.set_stream(torch.cuda.current_stream().cuda_stream)
    comm = TorchComm()
    stats = {}
    for _ in range(max(1, args.warmup)):
        sa, rk = build_sa_sharded(d_text, comm, GpuBackend(ex, dev), stats)
    launches0 = ex.launch_count
    # device time between barriers (CUDA events on the launching stream), maximum over the ranks
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(local_rank) as clocks:   # nvidia-smi clocks / throttle reasons during the timed region
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record()
        for _ in range(args.steps):
            sa, rk = build_sa_sharded(d_text, comm, GpuBackend(ex, dev), stats)
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    dt = torch.tensor([ev0.elapsed_time(ev1) * 1e-3], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    ms = float(dt.item()) / args.steps * 1e3
    idx = torch.arange(n, device=dev, dtype=torch.int64)
    ok = bool(torch.equal(rk[(sa.to(torch.int64) & 0xFFFFFFFF)].to(torch.int64) & 0xFFFFFFFF, idx))
    if rank == 0:
        per_suffix, P, R16 = B.bytes_alg_per_suffix(n, L)
        peak, peak_src = B.measured_peak()
        print(json.dumps({
            "metric": B.METRIC, "value": n / (ms * 1e-3) / 1e6, "unit": B.UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": B.DESCRIPTION[workload], "suffixes": n, "path": stats.get("path"),
                       "records": stats.get("records"),
                       "bucket_rank0": stats.get("bucket"), "records_sent_rank0": stats.get("sent"),
                       "l2_policy": "inputs larger than L2"},
            "gpu_launches": int(ex.launch_count - launches0),
            "clocks": clocks.summary(),
            "roofline": {"bound": "hbm", "kernel": "whole build", "achieved": per_suffix * n / (ms * 1e-3) / 1e9 / world,
                         "peak": peak, "unit": "GB/s", "frac": per_suffix * n / (ms * 1e-3) / 1e9 / world / peak,
                         "traffic": None, "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": n / (ms * 1e-3) / 1e6, "unit": B.UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "note": "multi-GPU line: device-resident replicated text; see the N=1 line for the host-buffer path"},
            "checks": {"rank_is_inverse_of_sa": ok},
        }))
    dist.barrier()
    dist.destroy_process_group()
