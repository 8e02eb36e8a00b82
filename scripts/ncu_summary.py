#!/usr/bin/env python3
"""Summarise an ncu report: per kernel time, DRAM bytes, throughputs, occupancy, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
col = {c: i for i, c in enumerate(h)}


def g(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except Exception:
        return float("nan")


stall_cols = [c for c in h if c.startswith("smsp__average_warp_latency_issue_stalled_") and c.endswith("ratio")]
if not stall_cols:
    stall_cols = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
seen = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
    t = g(r, "gpu__time_duration.sum")
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    l1 = g(r, "l1tex__throughput.avg.pct_of_peak_sustained_active")
    l2 = g(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
    dr = g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    occ = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    regs = g(r, "launch__registers_per_thread")
    fp64 = g(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
    l1hit = g(r, "l1tex__t_sector_hit_rate.pct")
    l2hit = g(r, "lts__t_sector_hit_rate.pct")
    st = sorted(((g(r, c), c.split("stalled_")[1]) for c in stall_cols), reverse=True)[:4]
    key = name
    seen[key] = seen.get(key, 0) + 1
    print(f"{name:>14s}#{seen[key]} t={t/1e3:8.1f}us dram R/W={rd/1e6:7.1f}/{wr/1e6:6.1f}MB "
          f"({(rd+wr)/max(t,1):6.0f} GB/s) dram%={dr:5.1f} L1%={l1:5.1f} L2%={l2:5.1f} L1hit={l1hit:4.1f} "
          f"L2hit={l2hit:4.1f} occ={occ:5.1f} regs={regs:.0f} fp64%={fp64:5.1f} stalls: " +
          ", ".join(f"{n}={v:.1f}" for v, n in st))
