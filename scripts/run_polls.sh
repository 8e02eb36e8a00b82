set -x
cd /root/repo
for sl in 3 8 16; do
  CEM_SCHED_SLACK=$sl python scripts/variant_bench.py 8 200
  CEM_SCHED_SLACK=$sl CEM_STATS=1 CEM_LIB=build/libcem_polls.so python scripts/variant_bench.py 8 200
done
python scripts/variant_bench.py 0 500
CEM_SCHED_SLACK=8 python scripts/variant_bench.py 8 500
