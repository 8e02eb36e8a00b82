#!/bin/bash
# bitwise parity of every documented build/run option (tests/test_gpu_parity.py, -m gpu)
cd /root/repo
# (build them first: CEM_FES=4, CEM_C_GEOX=1, CEM_D_BATCH=12, CEM_CRIT_COOP_MAX=32, CEM_BANK_SWAP=1)
for lib in build/libcem_fes4.so build/libcem_geox.so build/libcem_b12.so build/libcem_coop32.so build/libcem_swap.so; do
  echo "== $lib: $(CEM_LIB=$lib python -m pytest tests/test_gpu_parity.py tests/test_gpu_energy.py -x -q -m gpu 2>&1 | tail -1)"
done
echo "== CEM_CRITB_MIN=0: $(CEM_CRITB_MIN=0 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -m gpu 2>&1 | tail -1)"
echo "== CEM_BLK=128: $(CEM_BLK=128 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_energy.py -x -q -m gpu 2>&1 | tail -1)"
