import numpy as np, sys
sys.path.insert(0, '.')
import paper_1404_3456_b200 as rq
rng = np.random.default_rng(79)
mode = sys.argv[1] if len(sys.argv) > 1 else "repeat"
if mode == "repeat":
    unit = bytes(rng.choice([65, 67, 71, 84], 60_000).astype(np.uint8))
    genome = unit + unit[:30_000] + bytes(rng.choice([65, 67, 71, 84], 20_000).astype(np.uint8)) + unit[10_000:40_000]
    starts = rng.integers(0, len(genome) - 100 + 1, 45_000)
    text = np.frombuffer(b"".join(genome[int(s):int(s) + 100] + b"\0" for s in starts), dtype=np.uint8)
else:
    text, _ = rq.synth_read_text(1_000_000, 100, 100_000)
ex = rq.Executor(0)
got = rq.build_parallel(text, ex)
n = text.size
want = np.empty(n, np.uint32); want[got.sa] = np.arange(n, dtype=np.uint32)
bad = np.nonzero(want != got.rank)[0]
print("n", n, "bad ranks", bad.size, "rounds", got.stats.rounds)
if bad.size:
    print("first bad positions", bad[:20], "got", got.rank[bad[:20]], "want", want[bad[:20]])
    idx = want[bad]
    print("bad sa-index range", idx.min(), idx.max(), "tiles(2048) touched", np.unique(idx // 2048).size, "ip tiles(4096)", np.unique(idx // 4096).size)
    d = got.rank[bad].astype(np.int64) - want[bad].astype(np.int64)
    print("delta stats", d.min(), d.max(), np.abs(d).mean())
    # is got.rank a permutation?
    print("rank values unique:", np.unique(got.rank).size == n)
