#!/bin/bash
# timing of experiment libraries (CEM_LIB) on config 3, per-stage event times
for lib in "$@"; do
  echo "== $lib"; CEM_LIB=paper_2508_04076_b200/$lib CEM_STAGES=1 python scripts/variant_bench.py 0 500 2>&1 | tail -2
done
