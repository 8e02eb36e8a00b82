#!/bin/bash
# ncu full capture (with source) of one kernel family of a short bench run; plain run first.
set -u
OUT=gpurun_out
K=${1:-k_C}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -c 2 -o $OUT/prof_$K $CMD > $OUT/ncu_$K.log 2>&1
echo done
