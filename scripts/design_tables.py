"""Markdown tables for DESIGN.md section 6 from the committed measurement files.
usage: python scripts/design_tables.py [bench.json] [sweep.json] [scaling_c4.json] [scaling_c5.json]"""
import json, sys
b = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r2_bench.json"))
n = b["config"]["suffixes"]
print(f"Per kernel at {b['ms_per_step']:.2f} ms (CUDA events around every launch inside the timed region; fraction of "
      f"{b['roofline']['peak']:.1f} GB/s on the kernel's own algorithmic bytes):\n")
print("| kernel | launches | ms | B/suffix | frac of peak |\n|---|---|---|---|---|")
for k, v in b["roofline"]["kernels"].items():
    if v["ms_per_step"] < 0.02: continue
    bs = v["alg_bytes_per_suffix"]
    print(f"| {k} | {v['launches_per_step']:.0f} | {v['ms_per_step']:.3f} | {bs if bs is not None else '–'} | {('%.3f' % v['frac']) if v['frac'] else '–'} |")
print(f"\nsum of kernels {b['roofline']['sum_kernel_ms_per_step']:.2f} ms; e2e {b['e2e']['ms_per_step']:.1f} ms = {b['e2e']['value']:.0f} Msuffix/s "
      f"({b['e2e']['h2d_bytes_per_step']/1e6:.0f} MB in, {b['e2e']['d2h_bytes_per_step']/1e9:.2f} GB out)")
o = b.get("overlap")
if o:
    print(f"\nOverlap search, tau = {o['min_overlap']}: {o['queries']/1e6:.1f} M queries in {o['device_ms']:.2f} ms = {o['value']/1e3:.1f} Gq/s device, "
          f"{o['e2e']['ms']:.1f} ms = {o['e2e']['value']/1e3:.1f} Gq/s end to end ({o['overlaps_found']/1e6:.1f} M overlaps, {o['e2e']['d2h_bytes']/1e6:.0f} MB out); "
          f"index build {o['index_build_ms']:.1f} ms wall.\n")
    print("| overlap kernel | ms | ncu DRAM bytes | GB/s | frac of peak |\n|---|---|---|---|---|")
    for k, v in o["roofline"]["kernels"].items():
        if v["dram_bytes_ncu"]:
            print(f"| {k} | {v['ms']:.3f} | {v['dram_bytes_ncu']/1e9:.2f} GB | {v['dram_gbs']:.0f} | {v['dram_frac_of_peak']:.3f} |")
    if "index_build_kernels" in o:
        print(f"\n| index build kernel (sum {o['index_build_kernel_ms']:.2f} ms) | launches | ms |\n|---|---|---|")
        for k, v in o["index_build_kernels"].items():
            if v["ms"] >= 0.05: print(f"| {k} | {v['launches']} | {v['ms']:.3f} |")
    c = o["cpu_baseline"]
    print(f"\nCPU beside it: {c['what']}: {c['1_thread']['value']:.2f} Mq/s on 1 thread, {c['all_threads']['value']:.1f} Mq/s on {c['cores']} threads ({c['sample']}).")
r = b.get("routes")
if r:
    print("\n| route | option | ms / build | Msuffix/s | vs default | frac of the 8(d) model |\n|---|---|---|---|---|---|")
    for k, v in r.items():
        ratio = v.get("vs_default_route", v.get("vs_default_route_per_suffix"))
        print(f"| {k} | {v['option']} | {v['ms_per_build']:.2f} | {v['msuffixes_per_s']:.0f} | {ratio:.2f} | {v['frac_of_8d_model']:.2f} |")
c = b.get("cpu_baseline")
if c: print(f"\nCPU baseline: {c['value']:.3f} Msuffix/s on {c['cores']} cores ({c['sample']}); {c['also']}")
if len(sys.argv) > 2:
    s = json.load(open(sys.argv[2]))
    print(f"\nSweep ({s['config']['workload']}):\n\n| n | ms / build | Msuffix/s |\n|---|---|---|")
    for x in s["sweep"]: print(f"| {x['suffixes']:,} | {x['ms_per_build']:.3f} | {x['msuffixes_per_s']:.0f} |")
for f in sys.argv[3:]:
    m = json.load(open(f))
    print(f"\n{m['workload']}: single-GPU build {m['single_gpu_build_ms']:.1f} ms\n")
    ph = list(m["rows"][0]["phase_ms_max_over_ranks"])
    print("| G | " + " | ".join(ph) + " | all-to-all (model) | total | speed-up |\n|" + "---|" * (len(ph) + 4))
    for x in m["rows"]:
        print(f"| {x['G']} | " + " | ".join(f"{x['phase_ms_max_over_ranks'][p]:.2f}" for p in ph) +
              f" | {x['modelled_ms']['rank_all_to_all']:.2f} | {x['total_ms']:.1f} | {x['speedup_vs_single_gpu_build']:.2f} |")
