#!/bin/bash
# compute-sanitizer over the small all-kernel workload (one GPU): memcheck,
# racecheck (shared-memory hazards), synccheck; summaries in gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  BP_TMA_STREAM=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
      python scripts/debug/sanitize_driver.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
  tail -4 gpurun_out/sanitize_$tool.txt
done
