#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small shapes).
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_r02.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
echo done
