#!/bin/bash
# Quick A/B on the GPU box: SA + primitive parity tests, then the device-only bench under a list of
# environment settings.  usage: scripts/gpu_ab.sh <tag> "ENV1=a ENV2=b" "ENV1=c" ...
set -u
tag=${1:-x}; shift || true
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sa.py tests/test_gpu_primitives.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_${tag}.log
cat gpurun_out/pytest_${tag}.log
i=0
for envs in "$@"; do
  i=$((i+1))
  for w in c2 c1; do
    env $envs python bench.py --workload $w --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${i}_$w.json 2> gpurun_out/ab_${tag}_${i}_$w.err
    echo "== [$envs] $w"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${i}_$w.json
  done
done
