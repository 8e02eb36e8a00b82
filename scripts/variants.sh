#!/bin/bash
for lib in paper_2508_04076_b200/libcem.so build/libcem_ab4.so build/libcem_ab3c3.so; do
  CEM_LIB=$lib timeout 120 python scripts/variant_bench.py 2 200
done
