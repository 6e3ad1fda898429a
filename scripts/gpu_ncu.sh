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
  rep=gpurun_out/prof_${tag}_$name.ncu-rep
  if [ -f $rep ]; then   # text exports here (the reports exceed what gpurun_out/ brings back); the report itself is dropped
    ncu -i $rep --page details > gpurun_out/ncu_full_${tag}_$name.txt 2>&1
    ncu -i $rep --page raw --csv > gpurun_out/ncu_raw_${tag}_$name.csv 2>&1
    python scripts/ncu_lines.py $rep 45 > gpurun_out/ncu_lines_${tag}_$name.txt 2>&1
    python scripts/ncu_stalls.py $rep > gpurun_out/ncu_stalls_${tag}_$name.txt 2>&1
    rm -f $rep
    echo "$name: ok"
  else echo "$name: NO REPORT"; tail -3 gpurun_out/ncu_${tag}_$name.log; fi
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-routes > gpurun_out/ncu_launch_${tag}.log 2>&1
