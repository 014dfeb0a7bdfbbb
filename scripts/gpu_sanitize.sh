#!/bin/bash
# compute-sanitizer over the sort path (all tools), logs under gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for hl in 0 1; do
    TSQ_HOST_LEVELS=$hl timeout 420 $CS --tool $tool --print-limit 20 python scripts/sanitize_run.py 60000 \
      > gpurun_out/sanitizer_${tool}_hl${hl}.log 2>&1
    echo "$tool host_levels=$hl exit $?" >> gpurun_out/sanitizer_summary.txt
    tail -3 gpurun_out/sanitizer_${tool}_hl${hl}.log >> gpurun_out/sanitizer_summary.txt
  done
done
