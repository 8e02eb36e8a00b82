#!/bin/bash
for sl in 0.5 1 2 4 8 16; do
  echo -n "slack=$sl "; CEM_SCHED_SLACK=$sl timeout 120 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys; l=json.loads(sys.stdin.readline()); print(round(l['ms_per_step']*1e3,1),'us/step')"
done
