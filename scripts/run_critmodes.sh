#!/bin/bash
# the driver's bench window (20 steps after 5 warm-up, config 3's cracking phase) and the steady state
# per criterion mode (CEM_CRIT_MODE: 0 list, 1 heavy, 2 stream, 3 idle; unset = the host heuristic)
for env in "X=1" "CEM_CRIT_MODE=0" "CEM_CRIT_MODE=1" "CEM_CRIT_MODE=2" "CEM_CRIT_MODE=3"; do
  for w in "--steps 20 --warmup 5" "--steps 300 --warmup 100"; do
  env $env python bench.py $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$env', '$w', round(d['ms_per_step']*1e3,1), {a.split('_')[1]: round(b['ms_per_launch']*1e3,1) for a,b in k.items()})"
  done
done
