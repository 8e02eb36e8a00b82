#!/bin/bash
# bitwise parity of every documented build/run option (tests/test_gpu_parity.py, -m gpu)
cd /root/repo
for lib in build/libcem_fes4.so build/libcem_geox.so build/libcem_b12.so build/libcem_coop32.so; do
  echo "== $lib: $(CEM_LIB=$lib python -m pytest tests/test_gpu_parity.py tests/test_gpu_energy.py -x -q -m gpu 2>&1 | tail -1)"
done
echo "== CEM_BLK=128: $(CEM_BLK=128 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_energy.py -x -q -m gpu 2>&1 | tail -1)"
