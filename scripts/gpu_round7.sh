#!/bin/bash
# usage: scripts/gpu_round7.sh <tag>   TMA tile-load A/B (armed ahead of the block barrier), then the sanitizer suite
set -u
tag=${1:-x}
mkdir -p gpurun_out
for envs in "RESEQ_SORT_TMA=0" "RESEQ_SORT_TMA=1"; do
  python bench.py --workload c2 --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${envs#*=}_c2.json 2> gpurun_out/ab_${tag}_${envs#*=}_c2.err
  echo "== [$envs] c2"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${envs#*=}_c2.json | sed -n 1,4p
done
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_${tag}.log 2>&1
cat gpurun_out/r2_compute_sanitizer.txt
