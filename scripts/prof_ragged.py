"""Per-kernel device times of the SA build on a ragged read set (config 2's genome, read lengths 100..150)."""
import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
G, L, k = 4_600_000, 150, 920_000
rng = np.random.default_rng(7)
genome = rq.synth_random_dna(G, 1)
lens = rng.integers(100, L + 1, k); st0 = rng.integers(0, G - L, k)
total = int(lens.sum()) + k
offs = np.concatenate(([0], np.cumsum(lens + 1)[:-1]))
idx = np.minimum(np.repeat(st0 - offs, lens + 1) + np.arange(total), G - 1)
rag = genome[idx]; rag[offs + lens] = 0
d = torch.from_numpy(rag).cuda(); sa = torch.empty(total, dtype=torch.int32, device="cuda"); rk = torch.empty_like(sa)
ex = rq.Executor(0); lib = rq._lib.load(); st = rq.SaStats()
run = lambda: rq._lib.check(lib.reseq_cuda_build_sa_device(ex.handle, C.c_void_p(d.data_ptr()), total, C.c_void_p(sa.data_ptr()), C.c_void_p(rk.data_ptr()), C.byref(st)))
for _ in range(2): run()
ex.profile(True); run(); prof = ex.profile_read(); ex.profile(False)
print("n", total, "init_symbols", st.init_symbols, "rounds", st.rounds, "sum", sum(v[1] for v in prof.values()))
for kname, (cnt, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]): print(f"   {kname:28s} x{cnt:<3d} {ms:8.3f} ms")
