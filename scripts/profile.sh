#!/bin/bash
# Run on the GPU box: plain bench (must exit 0), then the ncu launch list and one full
# capture of every kernel of a short bench.  Outputs under gpurun_out/.
set -u
OUT=gpurun_out
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_' -c 24 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo done
