#!/usr/bin/env bash
# compute-sanitizer over the small all-kernels workload (tools/sanitize_workload.py); one log per
# tool under gpurun_out/ (summaries are copied to profiles/r02_sanitizer.md).
#   gpurun --timeout 1800 -- bash tools/sanitize.sh
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 $CS --tool $tool $extra --print-limit 20 python tools/sanitize_workload.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
