#!/usr/bin/env python3
"""Per-step kernel durations from an ncu --csv launch list of stage kernels (k_AB, k_C, k_crit /
k_filter / k_eval, k_D): one line per step, a step starting at each k_AB launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
kn, mv, mn, idc = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
seq = []
for r in rows[hdr_i + 1:]:
    if len(r) > mv and r[mn] == "gpu__time_duration.sum":
        name = r[kn].split("(")[0].split("::")[-1]
        seq.append((int(r[idc]), name, float(r[mv].replace(",", "")) / 1e3))
seq.sort()
steps, cur = [], None
for _, name, t in seq:
    if name.startswith("k_AB"):
        cur = []
        steps.append(cur)
    if cur is not None:
        cur.append((name, t))
for i, st in enumerate(steps):
    print(f"step {i:3d}: total {sum(t for _, t in st):6.1f}  " + "  ".join(f"{n} {t:5.1f}" for n, t in st))
