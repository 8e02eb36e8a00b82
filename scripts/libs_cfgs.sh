#!/bin/bash
# stage timings of several library builds on several configs (tuning aid): libs_cfgs.sh "cfgs" lib...
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
CFGS=$1; shift
for lib in "$@"; do for c in $CFGS; do CEM_LIB=$lib CEM_CFG=$c CEM_STAGES=1 python scripts/variant_bench.py 0 300; done; done
