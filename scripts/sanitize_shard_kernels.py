"""The kernels of the sharded build, one virtual rank after another in ONE thread (racecheck loses track of
launches from several host threads): bucket generation, sort + link, MAX-combine, accept / refine, owner partition,
the exchange done by hand, the owners' inverse -- for a uniform read set and for a ragged one (general records),
G = 3; the assembled suffix array and its inverse are compared with the single-GPU build."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
from paper_1404_3456_b200.sharded import GpuBackend, choose_bounds, PREFIX_BITS

def run(text, G):
    n = int(text.size)
    d_text = torch.from_numpy(np.array(text, copy=True)).cuda()
    exs = [rq.Executor(0) for _ in range(G)]
    bes = [GpuBackend(e) for e in exs]
    for be in bes: assert be.open(d_text)
    info = bes[0].uniform_info()
    units = info[1] if info else n
    hist = None
    for r, be in enumerate(bes):
        lo, hi = (units * r) // G, (units * (r + 1)) // G
        h = be.prefix_hist(lo, hi - lo)
        hist = h if hist is None else hist + h
    bounds = [0] + choose_bounds(hist, G) + [1 << PREFIX_BITS]
    recs = [be.bucket(bounds[r], bounds[r + 1]) for r, be in enumerate(bes)]
    sizes = [int(x.numel()) for x in recs]
    assert sum(sizes) == n
    if info:
        covs = None
        for be, rec in zip(bes, recs):
            c = be.uniform_sort_link(rec, info[1])
            covs = c if covs is None else torch.maximum(covs, c)
        parts = []
        for be in bes:
            sa_b, unf = be.uniform_finish(covs)
            assert unf == 0
            parts.append(sa_b)
    else:
        parts = []
        for be, rec in zip(bes, recs):
            sa_b, unf = be.finish(rec)
            assert unf == 0
            parts.append(sa_b)
    rank_recs = [be.rank_records(sa_b, sum(sizes[:r]), n, G) for r, (be, sa_b) in enumerate(zip(bes, parts))]
    slices = []
    for g, be in enumerate(bes):
        mine = torch.cat([rr[sum(c[:g]):sum(c[:g]) + c[g]] for rr, c in rank_recs])
        slice_len = (n * (g + 1)) // G - (n * g) // G
        assert mine.numel() == slice_len
        slices.append(be.rank_finish(mine, slice_len))
    torch.cuda.synchronize()
    sa = torch.cat(parts).cpu().numpy().view(np.uint32)
    rank = torch.cat(slices).cpu().numpy().view(np.uint32)
    for be in bes: be.close()
    for e in exs: e.close()
    want = rq.build_parallel(text, rq.Executor(0))
    assert np.array_equal(sa, want.sa) and np.array_equal(rank, want.rank)
    return "uniform" if info else "general"

text, _ = rq.synth_read_text(20_000, 100, 1_500)
kinds = [run(text, 3), run(text, 8)]
# a ragged read set (general records on the sharded path)
rng = np.random.default_rng(5)
genome = rq.synth_random_dna(30_000, 3)
pieces = []
for _ in range(900):
    L = int(rng.integers(40, 120)); s = int(rng.integers(0, 30_000 - L))
    pieces.append(genome[s:s + L]); pieces.append(np.zeros(1, np.uint8))
kinds.append(run(np.concatenate(pieces), 3))
assert kinds == ["uniform", "uniform", "general"], kinds
print("sanitize_shard_kernels: parity ok", kinds)
