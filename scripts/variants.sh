#!/bin/bash
for lib in paper_2508_04076_b200/libcem.so build/libcem_occ5.so build/libcem_occ6.so build/libcem_occ8.so; do
  CEM_LIB=$lib timeout 120 python scripts/variant_bench.py 2 200
done
