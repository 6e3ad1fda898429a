#!/bin/bash
# Final evidence of round 2 (one visit): GPU suite, driver-format bench lines, sweep, config 5, ncu launch list and
# --set full captures of the SA kernels, scaling models, forced-sharded bench, sanitizer suite.
# usage: scripts/gpu_final.sh <tag>
set -u
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q --durations=8 2>&1 | tail -16 > gpurun_out/pytest_${tag}.log
cat gpurun_out/pytest_${tag}.log | tail -3
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_${tag}.json 2>> gpurun_out/bench_${tag}.err
python bench.py --workload c1 --steps 20 --warmup 3 > gpurun_out/bench_${tag}_c1.json 2>> gpurun_out/bench_${tag}.err
python bench.py --workload c3 --sweep --steps 10 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/sweep_${tag}_c3.json 2>> gpurun_out/bench_${tag}.err
python bench.py --workload c4 --steps 5 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/bench_${tag}_c4.json 2>> gpurun_out/bench_${tag}.err
python bench.py --workload c5 --steps 3 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/bench_${tag}_c5.json 2>> gpurun_out/bench_${tag}.err
head -c 300 gpurun_out/bench_${tag}.json; echo
bash scripts/gpu_ncu.sh ${tag} onesweep:sa:onesweep_kernel accept:sa:accept_uniform gen:sa:gen_uniform invpart:sa:inv_partition ov_count:ov:overlap_count_kernel ov_fill:ov:overlap_fill_sorted ov_contained:ov:contained_kernel
timeout 900 python scripts/model_scaling.py --workload c4 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c4.json 2>&1 | grep "^G="
timeout 1200 python scripts/model_scaling.py --workload c5 --gpus 1,2,4,8 --out gpurun_out/scaling_model_${tag}_c5.json 2>&1 | grep "^G="
bash scripts/gpu_shard.sh ${tag} c4 2>&1 | grep "plain\|forced" | head -4
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize_${tag}.log 2>&1
cat gpurun_out/r2_compute_sanitizer.txt
