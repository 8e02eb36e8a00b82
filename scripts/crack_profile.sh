#!/bin/bash
# ncu --set full of the long-list criterion kernels (k_filter, k_eval) in config 1's cracking
# phase (step ~3000), after the same command ran clean without ncu
cd /root/repo
CMD="python scripts/variant_bench.py 0 3300"
CEM_CFG=1 $CMD > gpurun_out/crack_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
CEM_CFG=1 ncu --set full --clock-control none --import-source on -k regex:'k_(filter|eval)$' -s 2000 -c 2 \
    -o gpurun_out/prof_crack $CMD > gpurun_out/ncu_crack.log 2>&1
echo "ncu rc=$?"
