#!/bin/bash
# compute-sanitizer over the small end-to-end workloads (every kernel family once, parity asserted).
out=gpurun_out/r2_compute_sanitizer.txt
mkdir -p gpurun_out
echo "compute-sanitizer on the B200, final code of round 2 (scripts/sanitize_small.py: every kernel family once, parity asserted;" > $out
echo "scripts/sanitize_sharded.py: the sharded uniform build as three virtual ranks)" >> $out
run() { echo "" >> $out; echo "--- $1" >> $out; shift; timeout 1500 "$@" 2>&1 | grep -E "sanitize_|ERROR SUMMARY|RACECHECK SUMMARY|Error|error:|hazard|Traceback|assert" | head -20 >> $out; }
run "memcheck, sanitize_small.py (incl. the sharded part)" compute-sanitizer --tool memcheck python scripts/sanitize_small.py
run "racecheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool racecheck python scripts/sanitize_small.py
run "racecheck, sanitize_sharded.py" compute-sanitizer --tool racecheck python scripts/sanitize_sharded.py
run "initcheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool initcheck python scripts/sanitize_small.py
run "synccheck, sanitize_small.py (SANITIZE_NO_SHARDED=1)" env SANITIZE_NO_SHARDED=1 compute-sanitizer --tool synccheck python scripts/sanitize_small.py
cat $out
