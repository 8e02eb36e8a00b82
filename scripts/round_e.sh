#!/bin/bash
# final-build evidence of round 2 (after the hex-path changes): the default GPU suite, smoke, the driver's
# bench command, the full bench line, the reference arm, the hex profile.  The tet stage kernels' SASS
# equals the r02d build's (whose ncu captures profiles/r02d_* hold).
set -u
OUT=gpurun_out
( time python -m pytest tests -x -q -m gpu --durations=6 ) > $OUT/pytest_gpu_e.log 2>&1; tail -14 $OUT/pytest_gpu_e.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_e.log 2>&1; tail -1 $OUT/smoke_e.log
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench20_e.log 2>&1; tail -1 $OUT/bench20_e.log | cut -c1-200
python bench.py > $OUT/bench_full_e.log 2>&1; tail -1 $OUT/bench_full_e.log | cut -c1-200
python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $OUT/bench_ref_e.log 2>&1; tail -1 $OUT/bench_ref_e.log | cut -c1-200
bash scripts/hex_profile.sh
