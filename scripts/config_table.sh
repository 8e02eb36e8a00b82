#!/bin/bash
# per-config step times (config_table.py) + live DRAM bytes per step from ncu (no cache flush,
# 3 steps after 12 warm-up steps of scripts/short_run.py) -> gpurun_out/config_table.*
set -u
OUT=gpurun_out
python scripts/config_table.py > $OUT/config_table.jsonl 2> $OUT/config_table.err || exit 1
for k in 0 1 2 3 6; do
  CEM_CFG=$k ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:'k_(AB|C|crit|filter|eval|D)$' --csv --log-file $OUT/config_traffic_$k.csv python scripts/short_run.py 12 3 > /dev/null 2>&1
done
echo done
