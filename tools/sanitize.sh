#!/bin/bash
# compute-sanitizer over every libdstack entry point on configs 1-5 at small sizes.
# Logs: gpurun_out/san_<tool>.log; summary lines: gpurun_out/san_summary.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/san_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 --target-processes all \
      python tools/sanitize_run.py all > gpurun_out/san_$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -1)" >> gpurun_out/san_summary.txt
done
cat gpurun_out/san_summary.txt
