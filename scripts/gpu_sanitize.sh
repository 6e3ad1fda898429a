#!/bin/bash
# compute-sanitizer over the small end-to-end workloads (every kernel family once, parity asserted).
out=gpurun_out/r2_compute_sanitizer.txt
mkdir -p gpurun_out
echo "compute-sanitizer on the B200, final code of round 2 (scripts/sanitize_small.py: every kernel family once, parity asserted;" > $out
echo "scripts/sanitize_sharded.py: the sharded uniform build as three virtual ranks -- threads; scripts/sanitize_shard_kernels.py: the same kernels from one thread)" >> $out
i=0
run() { i=$((i+1)); echo "" >> $out; echo "--- $1" >> $out; shift; timeout 1500 "$@" > gpurun_out/sanitize_full_$i.log 2>&1; echo "exit code $?" >> gpurun_out/sanitize_full_$i.log
        grep -E "sanitize_|ERROR SUMMARY|RACECHECK SUMMARY|Error|error:|hazard|Traceback|assert|exit code" gpurun_out/sanitize_full_$i.log | head -20 >> $out
        tail -c 20000 gpurun_out/sanitize_full_$i.log > gpurun_out/sanitize_tail_$i.log; rm -f gpurun_out/sanitize_full_$i.log; }
run "memcheck, sanitize_small.py (incl. the sharded part)" compute-sanitizer --tool memcheck python scripts/sanitize_small.py
run "racecheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool racecheck python scripts/sanitize_small.py
run "racecheck, sanitize_shard_kernels.py (the sharded kernels, one virtual rank after another)" compute-sanitizer --tool racecheck python scripts/sanitize_shard_kernels.py
run "initcheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool initcheck python scripts/sanitize_small.py
run "synccheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool synccheck python scripts/sanitize_small.py
cat $out
