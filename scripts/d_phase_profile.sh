#!/bin/bash
# k_D in config 1 before (step ~500) and during (step ~3000) the cracking phase: time, DRAM bytes, L2 hit rate
cd /root/repo
CEM_CFG=1 python scripts/variant_bench.py 0 3300 > gpurun_out/dplain.log 2>&1 || exit 1
for sk in 500 3000; do
CEM_CFG=1 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --clock-control none -k regex:'k_D$' -s $sk -c 1 --csv --page raw --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct python scripts/variant_bench.py 0 3300 > gpurun_out/dprof_$sk.csv 2>&1
done
echo done
