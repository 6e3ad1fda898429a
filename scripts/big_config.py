"""BASELINE configs 3/4 on ONE B200: device-resident SA build at n = 1.0067 G (c4) or 3.02 G (c5, beyond
the reference's 2^31-1 cap), timed, then proved equal to the reference order on the host
(permutation + adjacent suffix_less over the whole array) and checked rank == inverse on the device.
usage: python scripts/big_config.py c4|c5 [--no-verify]"""
import ctypes as C, json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
from bench import WORKLOADS
from tests.oracle_lib import Oracle

w = sys.argv[1]
G, L, k = WORKLOADS[w]
t0 = time.perf_counter()
text, starts = rq.synth_read_text(G, L, k, 1, 2)
n = int(text.size)
print(f"{w}: n={n} generated in {time.perf_counter()-t0:.1f}s", flush=True)
ex = rq.Executor(0)
stream = torch.cuda.current_stream(); ex.set_stream(stream.cuda_stream)
lib = rq._lib.load()
d_text = torch.from_numpy(text).cuda()
d_sa = torch.empty(n, dtype=torch.int32, device="cuda")
d_rank = torch.empty(n, dtype=torch.int32, device="cuda")
st = rq.SaStats()
def step():
    rq._lib.check(lib.reseq_cuda_build_sa_device(ex.handle, C.c_void_p(d_text.data_ptr()), n, C.c_void_p(d_sa.data_ptr()),
                                                 C.c_void_p(d_rank.data_ptr()), C.byref(st)))
step(); torch.cuda.synchronize()
ex.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record(stream)
for _ in range(reps): step()
e1.record(stream); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
prof = ex.profile_read(); ex.profile(False)
print(f"build {ms:.2f} ms = {n/ms/1e3:.0f} Msuffix/s; init_symbols={st.init_symbols} rounds={st.rounds} passes={st.sort_passes} "
      f"refined_global={st.refined_global} peak_mem={torch.cuda.max_memory_allocated()/2**30:.1f} GiB(torch only)", flush=True)
for kname, (cnt, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])[:10]: print(f"   {kname:28s} x{cnt//reps:<3d} {t/reps:9.3f} ms")
# rank[sa[i]] == i, in chunks (no n-sized int64 temporaries)
ok = True
chunk = 1 << 26
for b in range(0, n, chunk):
    e = min(n, b + chunk)
    sa_c = d_sa[b:e].to(torch.int64) & 0xFFFFFFFF
    r_c = d_rank[sa_c].to(torch.int64) & 0xFFFFFFFF
    ok &= bool(torch.equal(r_c, torch.arange(b, e, device="cuda", dtype=torch.int64)))
print("rank is the inverse of sa:", ok, flush=True)
res = {"workload": w, "n": n, "ms_per_build": ms, "msuffix_per_s": n / ms / 1e3, "rank_is_inverse": ok,
       "init_symbols": int(st.init_symbols), "rounds": int(st.rounds), "refined_global": int(st.refined_global),
       "kernels_ms": {kname: t / reps for kname, (cnt, t) in prof.items()}}
if "--no-verify" not in sys.argv:
    sa = d_sa.cpu().numpy().view(np.uint32)
    t0 = time.perf_counter()
    bad = Oracle().verify_sa(text, sa, threads=32)
    print(f"host proof (permutation + adjacent suffix_less): {'OK' if bad == 0 else 'FAILED at ' + str(bad - 1)} in {time.perf_counter()-t0:.0f}s", flush=True)
    res["verified_against_suffix_less"] = bad == 0
import os
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(f"gpurun_out/big_{w}.json", "w"))
