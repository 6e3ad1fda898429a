#!/bin/bash
# usage: scripts/gpu_round6.sh <tag>   sharded parity + model (c5, G=8 profile), then racecheck with full hazard records
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -4
timeout 900 python scripts/model_scaling.py --workload c5 --gpus 8 --profile 2>&1 | grep -v "^{" | tail -8
timeout 900 python scripts/model_scaling.py --workload c5 --gpus 1 2>&1 | grep "^G="
SANITIZE_NO_SHARDED=1 timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_small.py > gpurun_out/racecheck_full_${tag}.log 2>&1
grep -c "hazard" gpurun_out/racecheck_full_${tag}.log
grep -B2 -A12 "Race reported\|hazard detected" gpurun_out/racecheck_full_${tag}.log | head -120
tail -5 gpurun_out/racecheck_full_${tag}.log
