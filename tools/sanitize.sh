#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over every library kernel
# (tools/sanitize_run.py: config 1 + a hub graph); logs -> gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > /dev/null 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --launch-timeout 0 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$t.log | tail -1)"
done
