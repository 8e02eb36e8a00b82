#!/bin/bash
export CEM_SCHED_SLACK=8
for blk in 256 128; do
  for fl in 0 12; do CEM_BLK=$blk timeout 120 python scripts/variant_bench.py $fl 200 | sed "s/^/blk=$blk /"; done
done
CEM_BLK=128 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cfg0_full or weak_block or persistent" 2>&1 | tail -1
