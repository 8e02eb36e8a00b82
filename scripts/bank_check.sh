#!/bin/bash
# shared-memory wavefronts and bank conflicts of the stage kernels (one steady-state launch each)
cd /root/repo
python scripts/variant_bench.py 0 400 > /dev/null 2>&1 || exit 1
ncu --clock-control none -k regex:'k_(AB|C)$' -s 600 -c 2 --csv --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum python scripts/variant_bench.py 0 400 > gpurun_out/bank_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/bank_raw.csv")) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    print(r[h.index("Kernel Name")].split("(")[0], r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
