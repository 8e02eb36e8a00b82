#!/bin/bash
# L2 persistence window variants (CEM_L2_WIN: 1 sigma planes, 2 partials, 3 both with hit ratio < 1)
for w in 1 2 3; do echo "== CEM_L2_WIN=$w"; CEM_L2_WIN=$w CEM_STAGES=1 python scripts/variant_bench.py 0 500 2>&1 | tail -2; done
echo "== off"; CEM_L2_PERSIST=0 CEM_STAGES=1 python scripts/variant_bench.py 0 500 2>&1 | tail -2
