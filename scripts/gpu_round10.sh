#!/bin/bash
# usage: scripts/gpu_round10.sh <tag>   parity, then A/B of the accept pass layouts (pairs / quads)
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sa.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -6
for envs in "RESEQ_ACCEPT_QUADS=0" "RESEQ_ACCEPT_QUADS=1" "RESEQ_ACCEPT_QUADS=0" "RESEQ_ACCEPT_QUADS=1"; do
  for w in c2 c1; do
    env $envs python bench.py --workload $w --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${envs#*=}_$w.json 2> gpurun_out/ab_${tag}_${envs#*=}_$w.err
    echo "== [$envs] $w"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${envs#*=}_$w.json | sed -n 1,5p | grep -v "^config"
  done
done
