#!/bin/bash
# one ncu --set full capture of each stage kernel in the steady state (step ~350) for the current build
cd /root/repo
python scripts/variant_bench.py 0 400 || exit 1
ncu --set full --clock-control none --import-source on -k regex:'k_(AB|C|D)$' -s 1050 -c 3 -o gpurun_out/prof_iter \
    python scripts/variant_bench.py 0 400 > gpurun_out/ncu_iter.log 2>&1
echo "ncu rc=$?"
