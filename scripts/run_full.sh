#!/bin/bash
# all GPU tests, then the default bench line (with e2e and cpu_baseline)
cd /root/repo
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
CEM_TIMING=1 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
grep "cem timing" gpurun_out/bench.err | head -20
