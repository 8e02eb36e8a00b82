#!/bin/bash
# partial-mode (R27) check: its parity tests, per-stage times in both assembly modes, one ncu
# capture of stage C and D in partial mode (steady state, config 3)
set -u
OUT=gpurun_out
python -m pytest tests/test_gpu_partials.py -m gpu -x -q > $OUT/pytest_partials.log 2>&1; echo rc=$? >> $OUT/pytest_partials.log
tail -3 $OUT/pytest_partials.log
for m in 1 0; do CEM_PARTIALS=$m CEM_STAGES=1 python scripts/variant_bench.py 0 500 2>&1 | tail -2; done
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'k_CILb1|k_DILb1' -s 500 -c 2 -o $OUT/prof_part \
    python scripts/variant_bench.py 0 400 > $OUT/ncu_part.log 2>&1; tail -2 $OUT/ncu_part.log
