#!/bin/bash
# usage: scripts/sweep_env.sh VAR v1 v2 ... -- runs bench.py (device part only) once per value of the env var
var=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  env $var=$v python bench.py --steps 10 --warmup 3 --no-overlap --no-cpu > gpurun_out/sweep_${var}_$v.json 2>/dev/null
  python scripts/bench_summary.py gpurun_out/sweep_${var}_$v.json | grep -E "^value|onesweep|window|scatter_rec" | sed "s/^/$var=$v  /"
done
