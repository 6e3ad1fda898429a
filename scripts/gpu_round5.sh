#!/bin/bash
# Sharded-path visit: parity tests of the sharded kernels, per-phase scaling model (with rank G-1's kernel tables at G = 8),
# owner-bin sweep, forced-sharded bench at N = 1.   usage: scripts/gpu_round5.sh <tag>
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -6
for bins in 1024 256; do
  echo "== RESEQ_OWNER_BINS=$bins"
  RESEQ_OWNER_BINS=$bins timeout 900 python scripts/model_scaling.py --workload c5 --gpus 8 --profile 2>&1 | grep -v "^{" | tail -8
done
timeout 900 python scripts/model_scaling.py --workload c4 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c4.json 2>&1 | grep "^G="
timeout 1200 python scripts/model_scaling.py --workload c5 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c5.json 2>&1 | grep "^G="
bash scripts/gpu_shard.sh ${tag} c4 2>&1 | tail -12
