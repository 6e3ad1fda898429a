#!/bin/bash
# usage: scripts/gpu_round8.sh <tag>   parity, then A/B of the split walkers in onesweep, then the sa-placement probe
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sa.py tests/test_gpu_primitives.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -6
for envs in "RESEQ_SORT_SPLIT=0" "RESEQ_SORT_SPLIT=1" "RESEQ_SORT_SPLIT=0" "RESEQ_SORT_SPLIT=1"; do
  for w in c2 c1; do
    env $envs python bench.py --workload $w --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${envs#*=}_$w.json 2> gpurun_out/ab_${tag}_${envs#*=}_$w.err
    echo "== [$envs] $w"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${envs#*=}_$w.json | sed -n 1,4p
  done
done
python scripts/probe_sa_offset.py 2>&1 | tail -12
python scripts/sanitize_shard_kernels.py 2>&1 | tail -3
timeout 1500 compute-sanitizer --tool racecheck python scripts/sanitize_shard_kernels.py 2>&1 | grep -E "sanitize_|RACECHECK SUMMARY|Error|hazard|Traceback|assert" | head -12
SANITIZE_NO_SHARDED=1 timeout 1500 compute-sanitizer --tool racecheck python scripts/sanitize_small.py 2>&1 | grep -E "sanitize_|RACECHECK SUMMARY|Error|hazard|Traceback|assert" | head -12
