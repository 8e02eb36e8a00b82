#!/bin/bash
# parity tests, then stage timings on several configs (tuning aid)
cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_energy.py tests/test_gpu_dist.py -x -q -m gpu 2>&1 | tail -3
for c in 3 6 2 1; do CEM_CFG=$c CEM_STAGES=1 python scripts/variant_bench.py 0 300; done
