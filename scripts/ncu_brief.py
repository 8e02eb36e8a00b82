#!/usr/bin/env python3
"""Key metrics of each kernel in an ncu report (time, DRAM, occupancy, pipes, top stalls)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[0], rows[2:]
col = {k: i for i, k in enumerate(h)}
def g(r, k):
    return r[col[k]] if k in col else "-"
keys = [("time us", "gpu__time_duration.sum"), ("dram R MB", "dram__bytes_read.sum"), ("dram W MB", "dram__bytes_write.sum"),
        ("dram %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("warps act %", "sm__warps_active.avg.pct_of_peak_sustained_active"), ("regs", "launch__registers_per_thread"),
        ("blk/SM", "launch__occupancy_limit_registers"), ("waves", "launch__waves_per_multiprocessor"),
        ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_active"), ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 hit %", "lts__t_sector_hit_rate.pct"), ("fp64 %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("issue %", "sm__inst_issued.avg.pct_of_peak_sustained_active")]
stall = [k for k in h if k.startswith("smsp__average_warp_latency_issue_stalled_") or k.startswith("smsp__pcsamp_warps_issue_stalled_")]
for r in data:
    print(g(r, "Kernel Name")[:60])
    print("   " + "  ".join(f"{a}={g(r, b)}" for a, b in keys))
    st = []
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((float(r[col[k]]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    st.sort(reverse=True)
    print("   stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:6]))
