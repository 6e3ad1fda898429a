"""Per-phase device times of the sharded SA build for G = 1, 2, 4, 8 ranks, measured on ONE GPU.

Every rank's compute phases are run one rank after another (each rank with its own context, so the
pipeline's state is the real one: complete proof table after the MAX-combine, real bucket sizes); a
phase's parallel time is the MAXIMUM over the ranks.  The collectives are not run (one GPU): their time is
modelled from the bytes each rank sends and the NVLink figures of /opt/skills/guides/B200_PROFILING.md
(peer copy 770 GB/s per direction per GPU; 8-rank all-reduce bus bandwidth 725 GB/s).

    python scripts/model_scaling.py --workload c4 --gpus 1,2,4,8 [--out profiles/...json]
"""
import argparse, json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
from paper_1404_3456_b200.sharded import GpuBackend, choose_bounds, PREFIX_BITS
from bench import WORKLOADS, DESCRIPTION

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--gpus", default="1,2,4,8")
ap.add_argument("--out", default=None)
ap.add_argument("--profile", action="store_true", help="per-kernel table of rank 0's phases (CUDA events around every launch)")
args = ap.parse_args()
PEER_GBS, ALLREDUCE_BUS_GBS = 770.0, 725.0

Gn, L, k = WORKLOADS[args.workload]
text, _ = rq.synth_read_text(Gn, L, k, 1, 2, pinned=True)
n = int(text.size)
d_text = torch.from_numpy(text).cuda()
torch.cuda.synchronize()

def timed(fn, prof=None, ex=None):
    """Device time of one phase of one rank.  With an executor: the SUM of the phase's kernel times (CUDA events around
    every launch) -- the events around the whole call also span the host's work in between (torch allocations of
    gigabyte outputs with eight ranks' buffers alive: tens of ms now and then), which a real rank does not pay per build;
    the host round trips a build does need are a separate modelled term.  prof = phase name: print the kernel table."""
    if ex is not None: ex.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fn(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if ex is not None:
        tab = ex.profile_read(); ex.profile(False)
        ksum = sum(v[1] for v in tab.values())
        if prof:
            print(f"   [{prof}] kernels {ksum:.2f} ms (call {ms:.2f} ms): " + ", ".join(f"{k} x{c} {t:.3f}" for k, (c, t) in sorted(tab.items(), key=lambda kv: -kv[1][1])), flush=True)
        ms = ksum
    return out, ms

# single-GPU reference time
ex0 = rq.Executor(0); ex0.set_stream(torch.cuda.current_stream().cuda_stream)
be0 = GpuBackend(ex0)
for _ in range(2): be0.full_build(d_text)
(_sa, _rk), t_single = timed(lambda: be0.full_build(d_text))
del _sa, _rk
ex0.close()
rows = []
for G in [int(x) for x in args.gpus.split(",")]:
    exs = [rq.Executor(0) for _ in range(G)]
    bes = [GpuBackend(e) for e in exs]
    phases = ("pack", "hist", "bucket", "sort_link", "finish", "rank_partition", "rank_finish")
    best = {p: [float("inf")] * G for p in phases}
    for rep in range(3):   # the first repetition warms the arenas; of the other two the faster time of each (phase, rank) is kept
        ph = {p: [0.0] * G for p in phases}   # (a phase's events also span the host's allocations: one slow cudaMalloc is not kernel time)
        P = (lambda r, name: f"G={G} rank {r} {name}" if args.profile and rep == 2 and r == G - 1 else None)
        for r, be in enumerate(bes):
            _, ph["pack"][r] = timed(lambda: be.open(d_text), None, exs[r])
        period, reads = bes[0].uniform_info()
        hist = None
        for r, be in enumerate(bes):
            lo, hi = (reads * r) // G, (reads * (r + 1)) // G
            h, ph["hist"][r] = timed(lambda: be.prefix_hist(lo, hi - lo), None, exs[r])
            hist = h if hist is None else hist + h
        bounds = [0] + choose_bounds(hist, G) + [1 << PREFIX_BITS]
        recs, covs, buckets = [], None, []
        for r, be in enumerate(bes):
            rec, ph["bucket"][r] = timed(lambda: be.bucket(bounds[r], bounds[r + 1]), P(r, "bucket"), exs[r])
            c, ph["sort_link"][r] = timed(lambda: be.uniform_sort_link(rec, reads), P(r, "sort_link"), exs[r])
            covs = c if covs is None else torch.maximum(covs, c)
            recs.append(rec)
        sizes = [int(x.numel()) for x in recs]
        sa_parts, rank_recs = [], []
        for r, be in enumerate(bes):
            (sa_b, unf), ph["finish"][r] = timed(lambda: be.uniform_finish(covs), P(r, "finish"), exs[r])
            assert unf == 0
            (rr, counts), ph["rank_partition"][r] = timed(lambda: be.rank_records(sa_b, sum(sizes[:r]), n, G), P(r, "rank_partition"), exs[r])
            sa_parts.append(sa_b); rank_recs.append((rr, counts))
        recs = None
        # the exchange, done by hand: owner g receives every rank's group g
        for g, be in enumerate(bes):
            parts = []
            for rr, counts in rank_recs:
                off = sum(counts[:g])
                parts.append(rr[off:off + counts[g]])
            mine = torch.cat(parts)
            slice_len = (n * (g + 1)) // G - (n * g) // G
            assert mine.numel() == slice_len
            rk, ph["rank_finish"][g] = timed(lambda: be.rank_finish(mine, slice_len), P(g, "rank_finish"), exs[g])
            if rep == 2 and g == 0:   # spot check: rank[sa[i]] == i for entries of every bucket that fall in the first slice
                off = 0
                for part in sa_parts:
                    head = part[:400_000].to(torch.int64) & 0xFFFFFFFF
                    sel = (head < slice_len).nonzero().squeeze(1)
                    assert torch.equal(rk[head[sel]].to(torch.int64) & 0xFFFFFFFF, sel + off)
                    off += int(part.numel())
                del head, sel
            del mine, rk
        rank_recs = None; sa_parts = None
        for be in bes: be.close()
        torch.cuda.synchronize()
        if rep >= 1:
            for p in phases: best[p] = [min(a, b) for a, b in zip(best[p], ph[p])]
    ph = best
    for e in exs: e.close()
    torch.cuda.empty_cache()
    # modelled collectives
    max_bucket = max(sizes)
    a2a_ms = (8.0 * max_bucket * (G - 1) / G) / (PEER_GBS * 1e9) * 1e3 if G > 1 else 0.0     # 8-byte (pos, idx) records leaving a rank
    cov_ms = (2.0 * (G - 1) / G * reads) / (ALLREDUCE_BUS_GBS * 1e9) * 1e3 if G > 1 else 0.0  # all-reduce MAX of k bytes
    hist_ms = 0.02 if G > 1 else 0.0                                                            # 16 KB all-reduce: latency only
    syncs_ms = 0.15                                                                             # ~6 host round trips of ~25 us
    compute = {p: max(v) for p, v in ph.items()}
    total = sum(compute.values()) + a2a_ms + cov_ms + hist_ms + syncs_ms
    rows.append({"G": G, "phase_ms_max_over_ranks": compute, "bucket_sizes": sizes,
                 "modelled_ms": {"rank_all_to_all": a2a_ms, "cov_all_reduce_max": cov_ms, "hist_all_reduce": hist_ms, "host_round_trips": syncs_ms},
                 "total_ms": total, "speedup_vs_single_gpu_build": t_single / total})
    print(f"G={G}: " + "  ".join(f"{p} {v:.2f}" for p, v in compute.items()) + f"  | a2a {a2a_ms:.2f} cov {cov_ms:.2f} | total {total:.2f} ms  speed-up {t_single / total:.2f}x", flush=True)
out = {"workload": DESCRIPTION[args.workload], "suffixes": n, "single_gpu_build_ms": t_single, "rows": rows,
       "how": "compute phases = sums of kernel times (CUDA events around every launch) measured on one B200, one rank after another, maximum over ranks; collectives modelled (peer 770 GB/s per direction, all-reduce bus 725 GB/s)"}
print(json.dumps(out))
if args.out:
    open(args.out, "w").write(json.dumps(out, indent=1))
