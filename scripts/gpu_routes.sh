#!/bin/bash
# Per-kernel tables of the three SA routes at config 2 (device-resident).  usage: scripts/gpu_routes.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
for spec in "default:" "general:RESEQ_SA_UNIFORM=0" "doubling:RESEQ_SA_TEXT_ROUNDS=0"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --workload c2 --steps 5 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/route_${tag}_$name.json 2> gpurun_out/route_${tag}_$name.err
  echo "== $name [$envs]"; python scripts/bench_summary.py gpurun_out/route_${tag}_$name.json
done
