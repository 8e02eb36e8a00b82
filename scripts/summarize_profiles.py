#!/usr/bin/env python3
"""Summarise gpurun_out/{launches.csv, prof_stages.ncu-rep} into profiles/ (per round)."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.path.join(ROOT, "profiles")
g = os.path.join(ROOT, "gpurun_out")

# ---- launch list: per-launch device time and DRAM bytes
rows = list(csv.reader(open(os.path.join(g, "launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
h = rows[hi]
L = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    k = (int(r[h.index("ID")]), r[h.index("Kernel Name")].split("(")[0].split("::")[-1])
    L[k][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
launches = [(i, n, m) for (i, n), m in sorted(L.items())]
stage = [x for x in launches if x[1] in ("k_AB", "k_C", "k_D")]
# steps = consecutive (k_AB, k_C, k_D) triples; use the last complete step (steady state)
steps = []
for j in range(len(stage) - 2):
    if [stage[j][1], stage[j + 1][1], stage[j + 2][1]] == ["k_AB", "k_C", "k_D"]:
        steps.append(stage[j:j + 3])
last = steps[-1]
traffic = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for _, _, m in last)
t_step = sum(m["gpu__time_duration.sum"] for _, _, m in last)
json.dump({"round": rnd, "dram_bytes_per_step": traffic, "ncu_step_time_ns": t_step,
           "per_kernel": {n: {"time_ns": m["gpu__time_duration.sum"], "dram_read": m["dram__bytes_read.sum"],
                              "dram_write": m["dram__bytes_write.sum"]} for _, n, m in last},
           "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     "--clock-control none (cold-cache, serialised launches)"},
          open(os.path.join(out_dir, "traffic_per_step.json"), "w"), indent=1)
shutil.copy(os.path.join(g, "launches.csv"), os.path.join(out_dir, f"{rnd}_launches.csv"))

# ---- full captures
raw = subprocess.run(["ncu", "-i", os.path.join(g, "prof_stages.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H, U = rr[0], rr[1]


def gv(r, k):
    try:
        return float(r[H.index(k)].replace(",", ""))
    except Exception:
        return float("nan")


lines = [f"# {rnd} — stage kernels, config 3 (1.02M tets), one B200", "",
         "Source: `scripts/round_profile.sh` (ncu --set full --clock-control none, one launch of each stage "
         "kernel in the steady state) and the launch list `" + f"{rnd}_launches.csv`.", "",
         f"Per-step DRAM traffic (sum over k_AB, k_C, k_D of one step, launch list): **{traffic/1e6:.1f} MB** "
         f"vs B_alg = 168.0 MB; serialised ncu step time {t_step/1e3:.1f} µs.", "",
         "| kernel | time (µs) | DRAM R/W (MB) | DRAM % | L1 % | L2 % | warps active % | IPC | fp64 pipe % | regs | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rr[2:]:
    name = r[H.index("Kernel Name")].split("(")[0].split("::")[-1]
    st = sorted(((gv(r, c), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in H
                 if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")), reverse=True)
    tot = sum(v for v, _ in st) or 1
    unit = U[H.index("dram__bytes_read.sum")]
    scale = 1e3 if unit.startswith("G") else (1.0 if unit.startswith("M") else 1e-3)
    lines.append(f"| {name} | {gv(r, 'gpu__time_duration.sum'):.1f} | {gv(r, 'dram__bytes_read.sum')*scale:.0f}/"
                 f"{gv(r, 'dram__bytes_write.sum')*scale:.0f} | {gv(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                 f"{gv(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                 f"{gv(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'sm__inst_executed.avg.per_cycle_active'):.2f} | "
                 f"{gv(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'launch__registers_per_thread'):.0f} | "
                 + ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in st[:3]) + " |")
open(os.path.join(out_dir, f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
