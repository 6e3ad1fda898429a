#!/bin/bash
# One GPU-box visit: parity suite, bench line, reference arm, ncu launch list, ncu full captures of the top kernels.
# usage: scripts/gpu_round.sh <tag> [kernel-regex ...]
set -u
tag=${1:-x}; shift || true
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_${tag}.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_${tag}.json 2>> gpurun_out/bench_${tag}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-overlap --no-cpu > gpurun_out/ncu_launch_${tag}.log 2>&1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 \
      -f -o gpurun_out/prof_${tag}_$k python bench.py --steps 1 --warmup 3 --no-overlap --no-cpu > gpurun_out/ncu_${tag}_$k.log 2>&1
done
cat gpurun_out/pytest_${tag}.log
head -c 600 gpurun_out/bench_${tag}.json
