#!/bin/bash
# per-kernel DRAM bytes with the caches left as the previous kernel left them (no flush),
# i.e. the traffic of the live pipeline rather than of cold isolated launches
cd /root/repo
python scripts/variant_bench.py 0 400 > /dev/null || exit 1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:'k_(AB|C|D)$' -s 1050 -c 9 --csv --log-file gpurun_out/live_traffic.csv python scripts/variant_bench.py 0 400 > gpurun_out/live_traffic.log 2>&1
echo "ncu rc=$?"
