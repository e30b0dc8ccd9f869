#!/bin/bash
# compute-sanitizer over every kernel (tools/sanitize_cases.py); logs -> gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.txt 2>&1 || { cat gpurun_out/sanitize_plain.txt; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_cases:' gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done
