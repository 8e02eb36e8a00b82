#!/usr/bin/env python3
"""Average gpu__time_duration per kernel name of an ncu --csv launch list (last N launches of each)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(list)
for r in rows[hdr_i + 1:]:
    if len(r) > mv and r[mn] == "gpu__time_duration.sum":
        tot[r[kn].split("(")[0]].append(float(r[mv].replace(",", "")))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
    v2 = v[skip:] if len(v) > skip else v
    print(f"{k:40s} n={len(v):5d} mean={sum(v2)/len(v2)/1e3:9.2f} us  total={sum(v2)/1e3:10.1f} us")
