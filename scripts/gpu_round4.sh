#!/bin/bash
# Evidence visit: full bench line (with the index-build kernel table), per-kernel tables of the general routes and
# of the ragged route, compute-sanitizer over the small end-to-end workloads.   usage: scripts/gpu_round4.sh <tag>
set -u
tag=${1:-x}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --workload c1 --steps 20 --warmup 3 > gpurun_out/bench_${tag}_c1.json 2>> gpurun_out/bench_${tag}.err
bash scripts/gpu_routes.sh ${tag} > gpurun_out/routes_${tag}.txt 2>&1
python scripts/prof_ragged.py > gpurun_out/ragged_${tag}.txt 2>&1
python scripts/prof_overlap.py c2 > gpurun_out/overlap_${tag}.txt 2>&1
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_${tag}.log 2>&1
tail -30 gpurun_out/r2_compute_sanitizer.txt
cat gpurun_out/ragged_${tag}.txt
