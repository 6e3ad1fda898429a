#!/bin/bash
# One GPU-box visit (round 2): parity suite, bench line, reference arm, ncu launch list, ncu --set full
# captures of the SA kernels (through bench.py) and of the overlap kernels (through scripts/prof_overlap.py).
# usage: scripts/gpu_round2.sh <tag> [--no-tests] [sa:<kernel-regex> ...] [ov:<kernel-regex> ...]
set -u
tag=${1:-x}; shift || true
mkdir -p gpurun_out
if [ "${1:-}" != "--no-tests" ]; then
  python -m pytest tests -m gpu -x -q --durations=12 2>&1 | tail -30 > gpurun_out/pytest_${tag}.log
else shift; fi
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_${tag}.json 2>> gpurun_out/bench_${tag}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-routes > gpurun_out/ncu_launch_${tag}.log 2>&1
for spec in "$@"; do
  kind=${spec%%:*}; k=${spec#*:}
  if [ "$kind" = "ov" ]; then
    ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 --launch-count 1 \
        -f -o gpurun_out/prof_${tag}_$k python scripts/prof_overlap.py c2 > gpurun_out/ncu_${tag}_$k.log 2>&1
  else
    ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 \
        -f -o gpurun_out/prof_${tag}_$k python bench.py --steps 1 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ncu_${tag}_$k.log 2>&1
  fi
done
cat gpurun_out/pytest_${tag}.log
head -c 400 gpurun_out/bench_${tag}.json
