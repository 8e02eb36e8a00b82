#!/usr/bin/env python3
"""Per-kernel time and DRAM bytes from an ncu --csv metrics log (one line per kernel launch)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
i = h.index
acc = collections.OrderedDict()
for r in rows[1:]:
    k = (r[i("ID")], r[i("Kernel Name")].split("::")[-1].split("(")[0])
    acc.setdefault(k, {})[r[i("Metric Name")]] = float(r[i("Metric Value")].replace(",", ""))
tot = collections.defaultdict(float)
for (kid, name), m in acc.items():
    rd, wr, t = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6, m.get("gpu__time_duration.sum", 0) / 1e3
    print(f"{kid:>3} {name:6} {t:7.1f} us  R {rd:6.1f} MB  W {wr:6.1f} MB  {(rd + wr) / t if t else 0:5.2f} TB/s")
    tot["R"] += rd; tot["W"] += wr; tot["t"] += t
n = max(1, len(acc) // 3)
print(f"per step (avg of {n}): {tot['t'] / n:.1f} us, R {tot['R'] / n:.1f} MB, W {tot['W'] / n:.1f} MB, total {(tot['R'] + tot['W']) / n:.1f} MB")
