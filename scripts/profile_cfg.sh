#!/bin/bash
# steady-state ncu --set full capture of every stage kernel (incl. k_crit) of one config: profile_cfg.sh <cfg> <steps> <skip>
cd /root/repo
CFG=${1:-6}; STEPS=${2:-310}; SKIP=${3:-1200}
CEM_CFG=$CFG python scripts/variant_bench.py 0 $STEPS || exit 1
CEM_CFG=$CFG ncu --set full --clock-control none --import-source on -k regex:'k_(AB|C|critb?|D)$' -s $SKIP -c 4 \
    -o gpurun_out/prof_cfg$CFG python scripts/variant_bench.py 0 $STEPS > gpurun_out/ncu_cfg$CFG.log 2>&1
echo "ncu rc=$?"
