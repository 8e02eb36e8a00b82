#!/bin/bash
# Round evidence on one B200 (each ncu pass only after its plain command exited 0):
#  1. the full bench line;
#  2. the ncu launch list of a short bench run (per-launch time + DRAM bytes, cold cache);
#  3. live per-stage DRAM traffic in the steady state (no cache flush between kernels);
#  4. one `ncu --set full` capture of each stage kernel in the steady state (step ~350).
set -u
OUT=gpurun_out
python bench.py > $OUT/bench_full.log 2>&1; echo "bench rc=$?" >> $OUT/bench_full.log
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
VB="python scripts/variant_bench.py 0 400"
$VB > $OUT/plain_vb.log 2>&1 || { echo "variant_bench failed"; exit 1; }
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k_(AB|C|crit|D)$' -s 1400 -c 12 --csv --log-file $OUT/live_traffic.csv $VB > $OUT/ncu_live.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_(AB|C|D)$' -s 1050 -c 3 -o $OUT/prof_stages \
    $VB > $OUT/ncu_full.log 2>&1
echo done
