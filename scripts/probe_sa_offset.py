"""inv_partition_sa reads the caller's sa array: does its placement relative to the arena matter?
Times the config-2 device build with d_sa sliced at different byte offsets of a larger tensor."""
import ctypes as C, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
from bench import WORKLOADS
G, L, k = WORKLOADS["c2"]
text, _ = rq.synth_read_text(G, L, k, 1, 2, pinned=True)
n = int(text.size)
d_text = torch.from_numpy(text).cuda()
ex = rq.Executor(0); lib = rq._lib.load()
stream = torch.cuda.Stream(); ex.set_stream(stream.cuda_stream)
big_sa = torch.empty(n + (64 << 20), dtype=torch.int32, device="cuda")
big_rk = torch.empty(n + (64 << 20), dtype=torch.int32, device="cuda")
with torch.cuda.stream(stream):
    for off_sa, off_rk in ((0, 0), (256, 0), (4096, 0), (1 << 16, 0), (1 << 20, 0), (1 << 21, 0), (3 << 20, 0), (0, 1 << 20), (1 << 20, 1 << 20), (17 << 20, 5 << 20)):
        sa = big_sa[off_sa // 4: off_sa // 4 + n]; rk = big_rk[off_rk // 4: off_rk // 4 + n]
        run = lambda: rq._lib.check(lib.reseq_cuda_build_sa_device(ex.handle, C.c_void_p(d_text.data_ptr()), n, C.c_void_p(sa.data_ptr()), C.c_void_p(rk.data_ptr()), None))
        for _ in range(3): run()
        ex.profile(True)
        for _ in range(5): run()
        torch.cuda.synchronize()
        prof = ex.profile_read(); ex.profile(False)
        tot = sum(v[1] for v in prof.values()) / 5
        print(f"sa+{off_sa:>9d} rank+{off_rk:>8d} (sa at {sa.data_ptr():#x}): build {tot:.3f} ms  " +
              "  ".join(f"{kn} {prof[kn][1] / prof[kn][0]:.3f}" for kn in ("inv_partition_sa", "inv_partition_rec", "accept_uniform_kernel", "window_scatter_kernel", "onesweep_u64_keys")), flush=True)
