#!/bin/bash
# end-of-round evidence on one B200: every GPU test (full horizons, CEM_LONG_TESTS=1), smoke(), the driver's bench command (and the
# reference arm), then the profile pass (scripts/round_profile.sh)
set -u
OUT=gpurun_out
CEM_LONG_TESTS=1 python -m pytest tests -x -q -m gpu --durations=8 > $OUT/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_final.log
tail -12 $OUT/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_final.log 2>&1; tail -1 $OUT/smoke_final.log
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench20_final.log 2>&1; tail -1 $OUT/bench20_final.log | cut -c1-300
python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $OUT/bench_ref_final.log 2>&1; tail -1 $OUT/bench_ref_final.log | cut -c1-300
bash scripts/round_profile.sh
