#!/bin/bash
# Round-2 follow-up visit: A/B of the accept pass's shared-memory proof bits, config 3's throughput sweep,
# config 5 through the driver-visible bench, and the per-phase scaling model (G = 1, 2, 4, 8 on one GPU).
# usage: scripts/gpu_round3.sh <tag>
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sa.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -4
for envs in "RESEQ_ACCEPT_LOWBITS=0" "RESEQ_ACCEPT_LOWBITS=1"; do
  for w in c2 c1; do
    env $envs python bench.py --workload $w --steps 20 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ab_${tag}_${envs#*=}_$w.json 2> gpurun_out/ab_${tag}_${envs#*=}_$w.err
    echo "== [$envs] $w"; python scripts/bench_summary.py gpurun_out/ab_${tag}_${envs#*=}_$w.json | head -6
  done
done
python bench.py --workload c3 --sweep --steps 10 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/sweep_${tag}_c3.json 2> gpurun_out/sweep_${tag}_c3.err
python -c "
import json; d = json.load(open('gpurun_out/sweep_${tag}_c3.json'))
print('c3', d['ms_per_step'], 'ms', d['value'], d['unit'])
for r in d['sweep']: print('  n=%d  %.3f ms  %.0f Msuffix/s' % (r['suffixes'], r['ms_per_build'], r['msuffixes_per_s']))
"
python bench.py --workload c5 --steps 3 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/bench_${tag}_c5.json 2> gpurun_out/bench_${tag}_c5.err
python scripts/bench_summary.py gpurun_out/bench_${tag}_c5.json | head -14
timeout 600 python scripts/model_scaling.py --workload c4 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c4.json 2>&1 | grep "^G="
timeout 900 python scripts/model_scaling.py --workload c5 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c5.json 2>&1 | grep "^G=\|Error\|error" | head
