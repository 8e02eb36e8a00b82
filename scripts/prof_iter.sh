#!/bin/bash
# stage timings + one ncu --set full capture of each stage kernel (steady state) for the current build
cd /root/repo
CEM_STAGES=1 python scripts/variant_bench.py 0 300 || exit 1
ncu --set full --clock-control none --import-source on -k regex:'k_(AB|C|D)$' -s 1050 -c 3 -o gpurun_out/prof_iter \
    python scripts/variant_bench.py 0 400 > gpurun_out/ncu_iter.log 2>&1
echo "ncu rc=$?"
