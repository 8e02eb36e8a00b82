#!/usr/bin/env python3
"""Summarise gpurun_out/{launches.csv, live_traffic.csv, prof_stages.ncu-rep} (scripts/round_profile.sh)
into profiles/: <round>_ncu_summary.md, <round>_launches.csv, <round>_live_traffic.csv, traffic_per_step.json."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.path.join(ROOT, "profiles")
g = os.path.join(ROOT, "gpurun_out")
STAGES = ("k_AB", "k_C", "k_D")


def metric_csv(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    L = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        k = (int(r[h.index("ID")]), r[h.index("Kernel Name")].split("(")[0].split("::")[-1])
        L.setdefault(k, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    return [(i, n, m) for (i, n), m in L.items()]


def steps_of(launches):
    """Complete steps k_AB, k_C, [k_crit], k_D in launch order (k_crit: the criterion list kernel)."""
    st = [x for x in launches if x[1] in STAGES + ("k_crit",)]
    out, cur = [], []
    for x in st:
        if x[1] == "k_AB":
            cur = [x]
        elif cur:
            cur.append(x)
            if x[1] == "k_D":
                if [y[1] for y in cur if y[1] != "k_crit"] == list(STAGES):
                    out.append(cur)
                cur = []
    return out


# ---- launch list of the bench command (cold cache, serialised): shares per step
launch_steps = steps_of(metric_csv(os.path.join(g, "launches.csv")))
lastL = launch_steps[-1]
t_launch = sum(m["gpu__time_duration.sum"] for _, _, m in lastL)
shutil.copy(os.path.join(g, "launches.csv"), os.path.join(out_dir, f"{rnd}_launches.csv"))
# ---- live traffic (no flush), steady state: average over the captured steps
live_steps = steps_of(metric_csv(os.path.join(g, "live_traffic.csv")))
live = defaultdict(lambda: defaultdict(float))
for stp in live_steps:
    for _, n, m in stp:
        for k, v in m.items():
            live[n][k] += v / len(live_steps)
ALL = STAGES + (("k_crit",) if "k_crit" in live else ())
live_bytes = sum(live[n]["dram__bytes_read.sum"] + live[n]["dram__bytes_write.sum"] for n in ALL)
live_t = sum(live[n]["gpu__time_duration.sum"] for n in ALL)
shutil.copy(os.path.join(g, "live_traffic.csv"), os.path.join(out_dir, f"{rnd}_live_traffic.csv"))

# ---- full captures (steady state)
raw = subprocess.run(["ncu", "-i", os.path.join(g, "prof_stages.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H, U = rr[0], rr[1]


def gv(r, k):
    try:
        return float(r[H.index(k)].replace(",", ""))
    except Exception:
        return float("nan")


def mb(r, k):
    unit = U[H.index(k)]
    scale = {"G": 1e3, "M": 1.0, "K": 1e-3}.get(unit[:1], 1e-6)
    return gv(r, k) * scale


full = OrderedDict()
for r in rr[2:]:
    full[r[H.index("Kernel Name")].split("(")[0].split("::")[-1]] = r


# ---- on-chip floors of each stage kernel (the same capture): L1 data-pipe wavefronts (shared +
# global, one per SM and clock), warp instructions (4 issue slots per SM and clock) and fp64
# thread operations (DADD + DMUL + DFMA, against the measured DFMA rate of tools/dfma_peak)
def pipe(n):
    r = full[n]
    cyc = gv(r, "sm__cycles_elapsed.avg")
    wf = gv(r, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg")
    wf_sh = gv(r, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg")
    fp64 = sum(gv(r, f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed") for o in ("dadd", "dmul", "dfma")) * cyc
    return {"sm_cycles": cyc, "l1_wavefronts_per_sm": wf, "l1_wavefronts_shared_per_sm": wf_sh,
            "l1_pipe_frac": wf / cyc, "warp_inst": gv(r, "smsp__inst_executed.sum"),
            "issue_frac": gv(r, "sm__inst_issued.avg.pct_of_peak_sustained_active") / 100.0,
            "fp64_thread_ops": fp64,
            "shared_bank_conflict_wavefronts": gv(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")}


cold_bytes = sum((mb(full[n], "dram__bytes_read.sum") + mb(full[n], "dram__bytes_write.sum")) * 1e6 for n in STAGES)
json.dump({"round": rnd,
           "dram_bytes_per_step": cold_bytes,
           "dram_bytes_per_step_live": live_bytes,
           "ncu_step_time_ns_live": live_t,
           "per_kernel_live": {n: {"time_ns": live[n]["gpu__time_duration.sum"], "dram_read": live[n]["dram__bytes_read.sum"],
                                   "dram_write": live[n]["dram__bytes_write.sum"]} for n in ALL},
           "per_kernel_cold": {n: {"time_ns": gv(full[n], "gpu__time_duration.sum") * 1e3,
                                   "dram_read": mb(full[n], "dram__bytes_read.sum") * 1e6,
                                   "dram_write": mb(full[n], "dram__bytes_write.sum") * 1e6} for n in STAGES},
           "per_kernel_pipes": {n: pipe(n) for n in STAGES},
           "source": {"dram_bytes_per_step": "ncu --set full (default cache flush) of k_AB, k_C, k_D at step ~350",
                      "dram_bytes_per_step_live": "ncu --cache-control none --metrics dram__bytes_*.sum, steady state"}},
          open(os.path.join(out_dir, "traffic_per_step.json"), "w"), indent=1)

lines = [f"# {rnd} — stage kernels, config 3 (1.02M tets), one B200", "",
         "Source: `scripts/round_profile.sh`: `ncu --set full --clock-control none` of one launch of each stage kernel "
         "at step ~350 (steady state, `scripts/variant_bench.py`, same kernels and config as `bench.py`), "
         f"the live-traffic pass `{rnd}_live_traffic.csv` (`--cache-control none`) and the launch list "
         f"`{rnd}_launches.csv` of `bench.py --steps 4 --warmup 3`.", "",
         f"Per-step DRAM traffic, live (no flush): **{live_bytes/1e6:.1f} MB** in {live_t/1e3:.1f} µs of serialised kernel "
         f"time = {live_bytes/live_t:.0f} GB/s; cold (ncu flushes L2 before each kernel): {cold_bytes/1e6:.1f} MB. "
         f"B_alg = 168.0 MB.", "",
         "| kernel | time (µs) | DRAM R/W live (MB) | DRAM R/W cold (MB) | DRAM % | L1 % | L2 % | warps active % | IPC | fp64 pipe % | regs | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for n in STAGES:
    r = full[n]
    st = sorted(((gv(r, c), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in H
                 if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")), reverse=True)
    tot = sum(v for v, _ in st) or 1
    lines.append(f"| {n} | {gv(r, 'gpu__time_duration.sum'):.1f} | {live[n]['dram__bytes_read.sum']/1e6:.0f}/"
                 f"{live[n]['dram__bytes_write.sum']/1e6:.0f} | {mb(r, 'dram__bytes_read.sum'):.0f}/"
                 f"{mb(r, 'dram__bytes_write.sum'):.0f} | {gv(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                 f"{gv(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                 f"{gv(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'sm__inst_executed.avg.per_cycle_active'):.2f} | "
                 f"{gv(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'launch__registers_per_thread'):.0f} | "
                 + ", ".join(f"{nm} {100*v/tot:.0f}%" for v, nm in st[:3]) + " |")
P = {n: pipe(n) for n in STAGES}
SM, CLK, DFMA = 148, 1.965e9, 18.1e12  # SMs, SM clock under load, measured fp64 instructions/s (36.2 TFLOP/s / 2)
lines += ["", "On-chip floors of the same launches (what the time would be if that unit alone ran at its peak): the L1 data "
          "pipe (shared-memory and global-load wavefronts, one per SM and clock), warp-instruction issue (4 per SM and "
          "clock) and the fp64 pipe (DADD + DMUL + DFMA thread operations at the measured 18.1 T instructions/s).", "",
          "| kernel | time (µs) | L1 data-pipe wavefronts per SM (shared) | L1 pipe floor (µs) / busy | warp instructions | issue floor (µs) | fp64 thread ops | fp64 floor (µs) | shared bank-conflict wavefronts |",
          "|---|---|---|---|---|---|---|---|---|"]
for n in STAGES:
    q = P[n]
    lines.append(f"| {n} | {gv(full[n], 'gpu__time_duration.sum'):.1f} | {q['l1_wavefronts_per_sm']:.0f} ({q['l1_wavefronts_shared_per_sm']:.0f}) | "
                 f"{q['l1_wavefronts_per_sm'] / CLK * 1e6:.1f} / {100 * q['l1_pipe_frac']:.0f} % | {q['warp_inst'] / 1e6:.1f} M | "
                 f"{q['warp_inst'] / (SM * 4 * CLK) * 1e6:.1f} | {q['fp64_thread_ops'] / 1e6:.0f} M | {q['fp64_thread_ops'] / DFMA * 1e6:.1f} | "
                 f"{q['shared_bank_conflict_wavefronts'] / 1e6:.2f} M |")
lines.append(f"| step | | | {sum(P[n]['l1_wavefronts_per_sm'] for n in STAGES) / CLK * 1e6:.1f} | "
             f"{sum(P[n]['warp_inst'] for n in STAGES) / 1e6:.1f} M | {sum(P[n]['warp_inst'] for n in STAGES) / (SM * 4 * CLK) * 1e6:.1f} | "
             f"{sum(P[n]['fp64_thread_ops'] for n in STAGES) / 1e6:.0f} M | {sum(P[n]['fp64_thread_ops'] for n in STAGES) / DFMA * 1e6:.1f} | |")
lines += ["", f"Launch list (cold, serialised) of one bench step: " +
          ", ".join(f"{n} {m['gpu__time_duration.sum']/1e3:.1f} µs" for _, n, m in lastL) + f" (sum {t_launch/1e3:.1f} µs)."]
open(os.path.join(out_dir, f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
