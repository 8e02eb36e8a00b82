#!/bin/bash
# Round evidence on one B200: full bench line, the ncu launch list of a short bench and one
# `ncu --set full` capture of each stage kernel (each only after its plain command exited 0).
set -u
OUT=gpurun_out
python bench.py > $OUT/bench_full.log 2>&1; echo "bench rc=$?" >> $OUT/bench_full.log
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_(AB|C|D)$' -s 3 -c 3 -o $OUT/prof_stages $CMD \
    > $OUT/ncu_full.log 2>&1
echo done
