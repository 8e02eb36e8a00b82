#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on scripts/sanitize_run.py (config 0, both
# criterion kernel paths, the wave path, a hex block); summaries to gpurun_out/sanitize_*.log
set -u
OUT=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
      python scripts/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
done
