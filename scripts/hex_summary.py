#!/usr/bin/env python3
"""Summarise gpurun_out/{hex_bench.jsonl, hex_launches.csv, prof_hex.ncu-rep} (scripts/hex_profile.sh) into
profiles/<round>_hex.md and copy the launch list and the bench lines beside it."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02e"
g, out = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
bench = [json.loads(x) for x in open(os.path.join(g, "hex_bench.jsonl")) if x.startswith("{")]
shutil.copy(os.path.join(g, "hex_bench.jsonl"), os.path.join(out, f"{rnd}_hex_bench.jsonl"))
shutil.copy(os.path.join(g, "hex_launches.csv"), os.path.join(out, f"{rnd}_hex_launches.csv"))

rows = list(csv.reader(open(os.path.join(g, "hex_launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
h = rows[hi]
L = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    k = (int(r[h.index("ID")]), r[h.index("Kernel Name")].split("(")[0].split("::")[-1])
    L.setdefault(k, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
launches = [(n, m) for (_, n), m in L.items()]
# the launch list covers the elastodynamics case first (4 kernels per step), then the cracking case
first_crit = next((i for i, (n, _) in enumerate(launches) if n == "k_hexcrit"), len(launches))
parts = {"elastodynamics": launches[:max(first_crit - 3, 0)], "criterion every step": launches[max(first_crit - 3, 0):]}

raw = subprocess.run(["ncu", "-i", os.path.join(g, "prof_hex.ncu-rep"), "--page", "raw", "--csv"],
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
    return gv(r, k) * {"G": 1e3, "M": 1.0, "K": 1e-3}.get(unit[:1], 1e-6)


lines = [f"# {rnd} — hexahedral path (N3), 100^3 hexes (1.03M nodes, 3.06M hex edges), one B200", "",
         "Source: `scripts/hex_profile.sh` — `scripts/hex_bench.py 100 100 100 50` (CUDA events on the context's stream), "
         f"the ncu launch list of a short run (`{rnd}_hex_launches.csv`, cold cache, serialised) and one `ncu --set full` "
         "capture of each hex stage kernel in the elastodynamics case.", "",
         "| case | µs/step | hex·steps/s | B_alg per step | achieved | frac of measured HBM peak | split records |", "|---|---|---|---|---|---|---|"]
for b in bench:
    lines.append(f"| {b['case']} | {b['ms_per_step'] * 1e3:.1f} | {b['hex_steps_per_s'] / 1e9:.2f} G | {b['b_alg_bytes_per_step'] / 1e6:.0f} MB | "
                 f"{b['achieved_gbs']:.0f} GB/s | {b['roofline_frac']:.3f} (peak {b['peak_gbs']:.0f} GB/s) | {b['records']} |")
lines += ["", "Launch list (cold, serialised), mean per launch:", "", "| case | kernel | launches | µs | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
for case, ls in parts.items():
    agg = defaultdict(list)
    for n, m in ls:
        agg[n].append(m)
    for n, ms in agg.items():
        f = lambda k: sum(m[k] for m in ms) / len(ms)
        lines.append(f"| {case} | {n} | {len(ms)} | {f('gpu__time_duration.sum') / 1e3:.1f} | {f('dram__bytes_read.sum') / 1e6:.0f} | "
                     f"{f('dram__bytes_write.sum') / 1e6:.0f} |")
lines += ["", "`ncu --set full` (elastodynamics, one launch each):", "",
          "| kernel | time (µs) | DRAM R/W (MB) | DRAM % | L1 % | L2 % | warps active % | fp64 pipe % | regs | top stalls |", "|---|---|---|---|---|---|---|---|---|---|"]
for r in rr[2:]:
    n = r[H.index("Kernel Name")].split("(")[0].split("::")[-1]
    st = sorted(((gv(r, c), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in H
                 if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")), reverse=True)
    tot = sum(v for v, _ in st) or 1
    lines.append(f"| {n} | {gv(r, 'gpu__time_duration.sum'):.1f} | {mb(r, 'dram__bytes_read.sum'):.0f}/{mb(r, 'dram__bytes_write.sum'):.0f} | "
                 f"{gv(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | {gv(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | {gv(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
                 f"{gv(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f} | {gv(r, 'launch__registers_per_thread'):.0f} | "
                 + ", ".join(f"{nm} {100 * v / tot:.0f}%" for v, nm in st[:3]) + " |")
open(os.path.join(out, f"{rnd}_hex.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
