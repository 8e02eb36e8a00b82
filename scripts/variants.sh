#!/bin/bash
export CEM_SCHED_SLACK=${CEM_SCHED_SLACK:-8}
for lib in paper_2508_04076_b200/libcem.so build/libcem_minb2.so build/libcem_minb4.so; do
  for fl in 0 4; do CEM_LIB=$lib timeout 120 python scripts/variant_bench.py $fl 200; done
done
CEM_LIB=paper_2508_04076_b200/libcem.so timeout 120 python scripts/variant_bench.py 2 200
