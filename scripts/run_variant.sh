#!/bin/bash
# parity tests, stage timings and live DRAM traffic for each library build given (CEM_LIB)
cd /root/repo
for lib in "$@"; do
  echo "=== $lib"
  CEM_LIB=$lib python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
  CEM_LIB=$lib CEM_STAGES=1 python scripts/variant_bench.py 0 500
  CEM_LIB=$lib ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k_(AB|C|D)$' -s 1050 -c 3 --csv --log-file gpurun_out/live_v.csv python scripts/variant_bench.py 0 400 > /dev/null 2>&1
  python scripts/live_summary.py gpurun_out/live_v.csv
done
