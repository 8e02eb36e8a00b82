#!/bin/bash
# one tuning iteration on the GPU box: parity tests, stage timings, live (no-flush) DRAM
# traffic per stage kernel, then timings of any extra library builds given as arguments
cd /root/repo
python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -3 gpurun_out/pytest_iter.log
CEM_STAGES=1 python scripts/variant_bench.py 0 500
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k_(AB|C|D)$' -s 1050 -c 3 --csv --log-file gpurun_out/live_traffic.csv python scripts/variant_bench.py 0 400 > gpurun_out/live_traffic.log 2>&1
python scripts/live_summary.py gpurun_out/live_traffic.csv
for lib in "$@"; do
  CEM_LIB=$lib python scripts/variant_bench.py 0 500
done
