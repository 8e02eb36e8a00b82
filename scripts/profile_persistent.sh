#!/bin/bash
set -u
OUT=gpurun_out
export CEM_SCHED_SLACK=8
CMD="python scripts/variant_bench.py 12 20"
$CMD > $OUT/plain_p.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 1 -c 1 -o $OUT/prof_persist $CMD > $OUT/ncu_p.log 2>&1
echo done
