#!/bin/bash
# compute-sanitizer over the small cases of every kernel family (tools/sanitize_cases.py); logs -> gpurun_out
cd "$(dirname "$0")/.."
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|done|max \|int16" gpurun_out/r2_sanitize_$tool.txt | tail -8
done
