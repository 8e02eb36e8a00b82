#!/bin/bash
# the driver's bench window (20 steps after 5) and the steady state, plus the per-step cracking window
OUT=gpurun_out
python bench.py --steps 20 --warmup 5 > $OUT/bench20.log 2>&1; tail -1 $OUT/bench20.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench20', d['ms_per_step'], d['kernels'])"
python bench.py --no-cpu-baseline --no-e2e > $OUT/bench1000.log 2>&1; tail -1 $OUT/bench1000.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench1000', d['ms_per_step'], d['kernels'])"
python scripts/crack_window.py 60 > $OUT/crack_window.log 2>&1; tail -30 $OUT/crack_window.log
