#!/bin/bash
# usage: scripts/gpu_round9.sh <tag>   parity (incl. the graph replay test), then A/B of the CUDA-graph replay
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sa.py tests/test_gpu_primitives.py -m gpu -x -q 2>&1 | tail -6
for envs in "RESEQ_SA_GRAPH=0" "RESEQ_SA_GRAPH=1"; do
  for w in c2 c1; do
    env $envs python bench.py --workload $w --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${envs#*=}_$w.json 2> gpurun_out/ab_${tag}_${envs#*=}_$w.err
    echo "== [$envs] $w"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${envs#*=}_$w.json | sed -n 1,4p
    python -c "import json; d=json.load(open('gpurun_out/ab_${tag}_${envs#*=}_$w.json')); print('   with launch events', d['ms_per_step_with_launch_events'], 'sum kernels', d['roofline']['sum_kernel_ms_per_step'])"
    tail -2 gpurun_out/ab_${tag}_${envs#*=}_$w.err
  done
done
