"""Rewrites the measured tables of DESIGN.md section 6 (from "Per kernel (CUDA events" to "## 7.") from the files
under profiles/.  usage: python scripts/design_section6.py"""
import json, subprocess, sys
P = "profiles/"
J = lambda f: json.load(open(P + f))
b, c1, c3, c4, c5 = J("r2_bench.json"), J("r2_bench_c1.json"), J("r2_bench_c3_sweep.json"), J("r2_bench_c4_device_only.json"), J("r2_bench_c5_device_only.json")
ref, fs = J("r2_bench_reference.json"), J("r2_bench_c4_forced_sharded_n1.json")
m4, m5 = J("r2_scaling_model_c4.json"), J("r2_scaling_model_c5.json")
tables = subprocess.run([sys.executable, "scripts/design_tables.py", P + "r2_bench.json", P + "r2_bench_c3_sweep.json",
                         P + "r2_scaling_model_c4.json", P + "r2_scaling_model_c5.json"], capture_output=True, text=True).stdout
per_kernel = tables[tables.index("| kernel | launches"):tables.index("CPU baseline:")]
sweep = tables[tables.index("Sweep ("):tables.index("config[3]: 1 Gbp")]
scaling = tables[tables.index("config[3]: 1 Gbp"):]
cb = b["cpu_baseline"]
ms = lambda x: f"{x:.3f}" if x < 1 else (f"{x:.2f}" if x < 10 else (f"{x:.1f}" if x < 100 else f"{x:.0f}"))
row = lambda name, d: f"| {name} | {d['config']['suffixes'] / 1e6:.2f} M | {ms(d['ms_per_step'])} | {d['value'] / 1e3:.1f} | {ms(d['e2e']['ms_per_step'])} ({d['e2e']['value'] / 1e3:.1f}) |"
g8 = lambda m: next(r for r in m["rows"] if r["G"] == 8)
r8 = g8(m5)
ph = r8["phase_ms_max_over_ranks"]
ov1 = c1["overlap"]
ovb = b["overlap"]
traffic = json.load(open(P + "r2_ncu_overlap_traffic.json"))["c2"]
head = f"""Per kernel (CUDA events around every launch of {b['steps']} further builds run right after the timed region — those builds launch
kernel by kernel, {b['ms_per_step_with_launch_events']:.2f} ms each; the timed region itself is graph replays at {b['ms_per_step']:.2f} ms; fraction of 6 451.8 GB/s on the
kernel's own algorithmic bytes; `profiles/r2_ncu_launches.csv` gives the same shares under ncu; DRAM bytes of the overlap
kernels from the ncu captures in `profiles/r2_ncu_overlap_traffic.json`):

"""
other = f"""CPU baseline in the same run: the reference's `build_parallel` with `executor{{workers={cb['cores']}}}` on a prefix of the
same text ({cb['sample'].split(' of the same')[0]}): {cb['value']:.2f} Msuffix/s ({cb['cores']} cores); `build_naive` on one thread
{cb['also']['build_naive_1_thread_msuffixes_per_s']:.1f} Msuffix/s; `build_parallel` with one worker {cb['also']['build_parallel_1_worker_msuffixes_per_s']:.2f} Msuffix/s. The reference arm
(`--impl reference`, 2²² suffixes, {ref['cpu_baseline']['cores']} threads): {ref['value']:.2f} Msuffix/s (`profiles/r2_bench_reference.json`).

Other configurations, device-resident on one B200 (`profiles/r2_bench_c1.json`, `r2_bench_c3_sweep.json`,
`r2_bench_c4_device_only.json`, `r2_bench_c5_device_only.json`; all proved equal to the reference order in the GPU suite):

| config | n | ms / build | Gsuffix/s | e2e ms (Gsuffix/s) |
|---|---|---|---|---|
{row('C1 (1 Mbp × 10, L = 100)', c1)}
{row('C2 (4.6 Mbp × 30, L = 150)', b)}
{row('C3 (100 Mbp read text)', c3)}
{row('C4 (1 Gbp read set)', c4)}
{row('C5 (3 Gbp read set, beyond the reference’s 2³¹−1 cap)', c5)}

C1 also runs the query half: {ov1['queries'] / 1e6:.1f} M queries in {ov1['device_ms']:.2f} ms = {ov1['value'] / 1e3:.1f} Gq/s, index build {ov1['index_build_ms']:.1f} ms wall. End to end every
configuration sits at the PCIe rate (n bytes in, 8n bytes out: ≈ 5 Gsuffix/s; one of seven visits to the pool measured
33 ms instead of 26–27 ms for config 2 with the same device time: the host side of the box), the suffix array leaving
on a second stream while its inverse is computed. At 1–3 G suffixes the refine kernel's share grows (2–8 % of the groups mix loci
once the genome has 10⁸ loci against 4.3 G keys, and the packed text — 755 MB at C5 — no longer sits in L2:
{c5['roofline']['kernels']['refine_uniform_kernel']['ms_per_step']:.0f} of the {c5['ms_per_step']:.0f} ms; ncu: half of its stall samples are block barriers around steps that only a few dozen of a tile's
2 048 suffixes take part in).

{sweep}
The knee: below ≈ 16 M suffixes a build is a chain of ~30 short kernels whose fixed costs (tile ramp-up, the look-back
chain's latency, one verdict read-back) do not shrink with n — {c3['sweep'][0]['ms_per_build']:.2f} ms at 2²⁰ is ≈ 4 µs per kernel; from 2²⁶ on the
build runs at the per-suffix rate of the table above. The CUDA-graph replay (§4.3) is what moved C1 from 16.9 to
{c1['value'] / 1e3:.1f} Gsuffix/s.

**Sharded build, per-phase model** (§5; ms, maximum over ranks, ONE B200; all-to-all modelled at 770 GB/s per direction;
**unmeasured on more than one physical GPU**):

{scaling}
Reading the table: `sort_link`, `finish` and `rank_finish` shrink as 1/G; `pack` (every rank packs the replicated text)
and the count sweep inside `bucket` (every rank looks at every suffix key once) do not — {ph['pack']:.2f} + 1.4 ms of the {r8['total_ms']:.1f} ms at
C5, G = 8; `rank_partition` + the all-to-all + `rank_finish` = {ph['rank_partition'] + ph['rank_finish'] + r8['modelled_ms']['rank_all_to_all']:.1f} ms are the price of a position-sharded `rank`
(one pass more than the single-GPU inverse, plus the wire). Modelled speed-up over the single-GPU build: **{r8['speedup_vs_single_gpu_build']:.2f} × at C5,
{g8(m4)['speedup_vs_single_gpu_build']:.2f} × at C4 for G = 8** (round 1's design: ≤ 2.3 ×; at the start of this session's bucket-generator and owner-kernel
work: 3.83 ×). What would close the rest of the gap to 6 ×: the sender partitioning on the receiver's first-pass bins so
that the owner runs one pass instead of two (−1.3 ms), and the bucket histogram distributed over the ranks with the keep
masks exchanged (−1 ms). The sharded path on ONE rank (`bench.py --force-sharded`,
`profiles/r2_bench_c4_forced_sharded_n1.json`) costs {fs['ms_per_step']:.1f} ms against {c4['ms_per_step']:.1f} ms for the plain build at C4 ({fs['ms_per_step'] / c4['ms_per_step']:.2f} ×): the
splitter histogram, the bucket generator in place of the transposed generator and the extra owner partition pass are pure
overhead when there is nobody to exchange with.

"""
s = open("DESIGN.md").read()
a, z = s.index("Per kernel (CUDA events around every launch"), s.index("### Tuning knobs")
open("DESIGN.md", "w").write(s[:a] + head + per_kernel + other + s[z:])
print("section 6 rewritten:", b["ms_per_step"], c1["ms_per_step"], c4["ms_per_step"], c5["ms_per_step"], r8["speedup_vs_single_gpu_build"])
