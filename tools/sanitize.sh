#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every in-place kernel at
# small sizes (tools/sanitize_cases.py), logs into gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitize_summary.txt
  tail -3 gpurun_out/r2_sanitize_$tool.log >> gpurun_out/r2_sanitize_summary.txt
done
