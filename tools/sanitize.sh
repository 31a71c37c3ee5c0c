#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_driver.py); summaries -> gpurun_out/san_*.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for stage in gram16 gram32 gram64 chol eigh svd apply; do
    timeout 400 $CS --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_driver.py $stage > gpurun_out/san_${tool}_${stage}.log 2>&1
    echo "$tool $stage rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|HAZARD|Error' gpurun_out/san_${tool}_${stage}.log | tail -2 | tr '\n' ' ')" >> gpurun_out/san_summary.txt
  done
done
