#!/bin/bash
# ncu --set full captures, one kernel per spec.  usage: scripts/gpu_ncu.sh <tag> spec ...
#   spec = name:kind:kernel-regex[:ENV=VAL[,ENV=VAL]]   kind = sa (through bench.py) | ov (through scripts/prof_overlap.py)
set -u
tag=${1:-x}; shift || true
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r name kind k envs <<< "$spec"
  envs=${envs:-}; envs=${envs//,/ }
  if [ "$kind" = "ov" ]; then
    env $envs ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 --launch-count 1 \
        -f -o gpurun_out/prof_${tag}_$name python scripts/prof_overlap.py c2 > gpurun_out/ncu_${tag}_$name.log 2>&1
  else
    env $envs ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 \
        -f -o gpurun_out/prof_${tag}_$name python bench.py --steps 1 --warmup 3 --no-overlap --no-cpu --no-routes > gpurun_out/ncu_${tag}_$name.log 2>&1
  fi
  echo "$name: $(ls -la gpurun_out/prof_${tag}_$name.ncu-rep 2>/dev/null | awk '{print $5}') bytes"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-routes > gpurun_out/ncu_launch_${tag}.log 2>&1
