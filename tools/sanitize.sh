#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py); logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$? $(grep -c 'CASE .* ok' gpurun_out/sanitize_${tool}.log) ok, $(grep -c FAIL gpurun_out/sanitize_${tool}.log) fail, $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}.log | tail -1)"
done
