#!/bin/bash
# Sharded path on one GPU: virtual-rank parity tests, then the forced-sharded bench at N=1 next to the plain one.
tag=${1:-x}; shift || true
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -15
for w in "$@"; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/shard_${tag}_${w}_plain.json 2> gpurun_out/shard_${tag}_${w}_plain.err
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --force-sharded > gpurun_out/shard_${tag}_${w}_forced.json 2> gpurun_out/shard_${tag}_${w}_forced.err
  tail -3 gpurun_out/shard_${tag}_${w}_forced.err
  python - <<PY
import json
a = json.load(open("gpurun_out/shard_${tag}_${w}_plain.json")); t = open("gpurun_out/shard_${tag}_${w}_forced.json").read(); b = json.loads(t[t.index('{"metric"'):])
print("$w plain %.3f ms  forced-sharded %.3f ms  ratio %.3f  e2e %.1f ms  path %s ok %s" % (a["ms_per_step"], b["ms_per_step"], b["ms_per_step"] / a["ms_per_step"], b["e2e"]["ms_per_step"], b["config"]["path"], b["checks"]))
for k, v in b["roofline"]["kernels"].items(): print("   %-28s %8.3f ms x%.0f" % (k, v["ms_per_step"], v["launches_per_step"]))
PY
done
