"""Copies the outputs of scripts/gpu_final.sh <tag> from gpurun_out/ into profiles/ under their round-2 names and
refreshes the ncu traffic tables.  usage: python scripts/collect_profiles.py <tag>"""
import csv, json, re, shutil, sys
t = sys.argv[1]
g, P = "gpurun_out/", "profiles/"
for src, dst in ((f"bench_{t}.json", "r2_bench.json"), (f"bench_ref_{t}.json", "r2_bench_reference.json"), (f"bench_{t}_c1.json", "r2_bench_c1.json"),
                 (f"bench_{t}_c4.json", "r2_bench_c4_device_only.json"), (f"bench_{t}_c5.json", "r2_bench_c5_device_only.json"),
                 (f"sweep_{t}_c3.json", "r2_bench_c3_sweep.json"), (f"launches_{t}.csv", "r2_ncu_launches.csv"), (f"pytest_{t}.log", "r2_gputest.log"),
                 ("r2_compute_sanitizer.txt", "r2_compute_sanitizer.txt"), (f"scaling_model_{t}_c4.json", "r2_scaling_model_c4.json"),
                 (f"scaling_model_{t}_c5.json", "r2_scaling_model_c5.json"), (f"ncu_lines_{t}_onesweep.txt", "r2_ncu_lines_onesweep.txt"),
                 (f"ncu_lines_{t}_accept.txt", "r2_ncu_lines_accept.txt"), (f"ncu_lines_{t}_ov_count.txt", "r2_ncu_lines_ov_count.txt")):
    shutil.copy(g + src, P + dst)
kernels = ("onesweep", "accept", "gen", "invpart", "ov_count", "ov_fill", "ov_contained")
for k in kernels: shutil.copy(f"{g}ncu_full_{t}_{k}.txt", f"{P}r2_ncu_full_{k}.txt")
x = open(f"{g}shard_{t}_c4_forced.json").read()
open(P + "r2_bench_c4_forced_sharded_n1.json", "w").write(x[x.index('{"metric"'):])
parts = {k: open(f"{g}ncu_stalls_{t}_{k}.txt").read() for k in kernels}
secs = re.split(r"(?m)^=== ", open(P + "r2_ncu_stalls_summary.txt").read())
out, seen = [], set()
for sec in secs:
    if not sec.strip(): continue
    name = sec.split("\n", 1)[0].strip()
    if name in parts: out.append(f"=== {name}\n{parts[name]}"); seen.add(name)
    else: out.append("=== " + sec)
out += [f"=== {k}\n{parts[k]}" for k in parts if k not in seen]
open(P + "r2_ncu_stalls_summary.txt", "w").write("".join(o if o.endswith("\n") else o + "\n" for o in out))
def traffic(name):
    rows = list(csv.reader(open(f"{g}ncu_raw_{t}_{name}.csv"))); h = rows[0]; u = dict(zip(h, rows[1])); d = dict(zip(h, rows[2]))
    val = lambda k: float(d[k].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u[k]]
    return val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
sa, ov = json.load(open(P + "r2_ncu_sa_traffic.json")), json.load(open(P + "r2_ncu_overlap_traffic.json"))
for name, key in (("onesweep", "onesweep_u64_keys"), ("accept", "accept_uniform_kernel"), ("gen", "gen_uniform_kernel"), ("invpart", "inv_partition_rec")): sa["c2"][key] = traffic(name)
for name, key in (("ov_count", "overlap_count_kernel"), ("ov_fill", "overlap_fill_sorted_kernel"), ("ov_contained", "contained_kernel")): ov["c2"][key] = traffic(name)
json.dump(sa, open(P + "r2_ncu_sa_traffic.json", "w"), indent=1); json.dump(ov, open(P + "r2_ncu_overlap_traffic.json", "w"), indent=1)
print("profiles refreshed from tag", t)
