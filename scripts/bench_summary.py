"""Prints the headline and the per-kernel table of a bench.py JSON line.  usage: bench_summary.py file.json"""
import json, sys
d = json.load(open(sys.argv[1]))
print(f"value {d['value']:.0f} {d['unit']}  ms/step {d['ms_per_step']:.3f}  launches {d['gpu_launches']}  e2e {d['e2e']['value']:.0f} ({d['e2e']['ms_per_step']:.2f} ms)")
print("config", {k: d['config'][k] for k in ('rounds', 'init_symbols', 'sort_passes')}, "checks", d['checks'], "clocks", d['clocks'])
for k, v in d['roofline']['kernels'].items():
    print(f"  {k:26s} {v['ms_per_step']:7.3f} ms/step  x{v['launches_per_step']:.0f}  avg {v['avg_launch_ms']:.3f}  "
          f"frac {v['frac'] if v['frac'] is None else round(v['frac'], 3)}  share {v['share_of_step']:.3f}")
r = d['roofline']
print("roofline", {k: r[k] for k in ('kernel', 'achieved', 'peak', 'frac', 'traffic')}, "build", r['build'])
if d.get('overlap'): print("overlap", d['overlap'])
if d.get('cpu_baseline'): print("cpu", d['cpu_baseline'])
