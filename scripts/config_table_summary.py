#!/usr/bin/env python3
"""gpurun_out/config_table.jsonl + config_traffic_<k>.csv -> profiles/<round>_config_table.md
(R_ach = live ncu DRAM bytes per step / step time / HBM peak; R_alg = algorithmic bytes / step time / peak)."""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
g = os.path.join(ROOT, "gpurun_out")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6554.9


def per_step_bytes(path, steps=3):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    L = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        k = (int(r[h.index("ID")]), r[h.index("Kernel Name")].split("(")[0].split("::")[-1])
        L.setdefault(k, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    launches = list(L.items())
    starts = [i for i, ((_, n), _) in enumerate(launches) if n == "k_AB"]
    sel = launches[starts[-steps]:] if len(starts) >= steps else launches
    b = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in sel)
    t = sum(m.get("gpu__time_duration.sum", 0) for _, m in sel)
    return b / steps, t / steps


rows = [json.loads(x) for x in open(os.path.join(g, "config_table.jsonl")) if x.startswith("{")]
out = ["# " + rnd + " — per-config table (one B200)", "",
       "Step time over steps 10–210 (config 4: 10–60) with the criterion and split pass every step "
       "(`scripts/config_table.py`); R_alg = B_alg / step time / " + f"{peak} GB/s (B_alg = 177 B/node + 17 B/tet + 96 B/edge); "
       "R_ach = live DRAM bytes per step (ncu `--cache-control none`, 3 steps after 12 warm-up, kernels serialised by ncu) / "
       "the same step time / peak (`scripts/config_table.sh`).", "",
       "| config | tets | nodes | edges | µs/step | G tet·steps/s | B_alg MB/step | R_alg | DRAM MB/step (live) | R_ach | DRAM/B_alg |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    path = os.path.join(g, f"config_traffic_{r['cfg']}.csv")
    dram = per_step_bytes(path)[0] if os.path.exists(path) else None
    rach = dram / (r["us_per_step"] * 1e-6) / 1e9 / peak if dram else None
    out.append(f"| {r['cfg']} ({r['name']}) | {r['tets']} | {r['nodes']} | {r['edges']} | {r['us_per_step']:.1f} | "
               f"{r['G_tet_steps_per_s']:.2f} | {r['B_alg_MB']:.1f} | {r['R_alg']:.3f} | "
               + (f"{dram / 1e6:.1f} | {rach:.3f} | {dram / 1e6 / r['B_alg_MB']:.2f} |" if dram else "– | – | – |"))
open(os.path.join(ROOT, "profiles", f"{rnd}_config_table.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
