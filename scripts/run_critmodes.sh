#!/bin/bash
# the driver's bench window (20 steps after 5 warm-up, config 3's cracking phase) per criterion mode
for env in "X=1" "CEM_CRITB_MIN=0" "CEM_CRITB_MIN=300" "CEM_CRIT_STREAM=0"; do
  env $env python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$env', round(d['ms_per_step']*1e3,1), {a.split('_')[1]: round(b['ms_per_launch']*1e3,1) for a,b in k.items()})"
done
