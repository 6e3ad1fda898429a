"""Per-kernel device times of the index build and the overlap search at a bench workload."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1404_3456_b200 as rq
from bench import WORKLOADS
w = sys.argv[1] if len(sys.argv) > 1 else "c2"
G, L, k = WORKLOADS[w]
text, starts = rq.synth_read_text(G, L, k, 1, 2, pinned=True)
ex = rq.Executor(0)
fset = rq.fragment_set_from_text(text, starts)
for rep in range(2):
    ex.profile(True)
    t0 = time.perf_counter(); ix = rq.FragmentIndex(fset, ex); ex.synchronize(); t1 = time.perf_counter()
    p_build = ex.profile_read()
    ex.profile(True)
    ix.overlaps(20, reuse_buffers=True); ex.profile(True)
    t1 = time.perf_counter(); ov = ix.overlaps(20, reuse_buffers=True); t2 = time.perf_counter()
    p_ov = ex.profile_read()
    ex.profile(False)
    if rep == 0: ix.close()
print(f"index build {1e3*(t1-t0):.1f} ms wall; overlaps {1e3*(t2-t1):.1f} ms wall, device {ov.device_ms:.2f} ms, queries {ov.queries}, found {ov.i.size}")
for name, prof in (("build", p_build), ("overlaps", p_ov)):
    print(name, f"sum {sum(v[1] for v in prof.values()):.2f} ms")
    for kname, (cnt, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]): print(f"   {kname:28s} x{cnt:<3d} {ms:8.3f} ms")
