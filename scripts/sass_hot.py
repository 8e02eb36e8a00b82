#!/usr/bin/env python3
"""Group SASS of one kernel in an ncu report into runs of equal execution count (≈ basic blocks)
and print the instruction-count / stall-sample share of each, plus the opcode mix."""
import collections
import csv
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
isrc, iex, iss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")


def n(x):
    try:
        return int(x)
    except Exception:
        return 0


tot_i = sum(n(r[iex]) for r in data)
tot_s = sum(n(r[iss]) for r in data) or 1
print(f"{kern}: {tot_i} warp-instructions, {tot_s} stall samples, {len(data)} SASS lines")
mix = collections.Counter()
for r in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0].split(".")[0]
    mix[op] += n(r[iex])
print("  mix:", ", ".join(f"{o} {100 * v / tot_i:.0f}%" for o, v in mix.most_common(12)))
groups = []
for i, r in enumerate(data):
    c = n(r[iex])
    if groups and groups[-1][1] == c:
        groups[-1][2] += 1
        groups[-1][3] += n(r[iss])
        groups[-1][4].append(r[isrc].strip())
    else:
        groups.append([i, c, 1, n(r[iss]), [r[isrc].strip()]])
for g in groups:
    if g[1] * g[2] > 0.02 * tot_i or g[3] > 0.03 * tot_s:
        ops = [re.sub(r"^@!?U?P\w+\s+", "", x).split(" ")[0] for x in g[4]]
        print(f"  #{g[0]:5d} len={g[2]:4d} exec={g[1]:8d} instr={100 * g[1] * g[2] / tot_i:5.1f}% "
              f"stall={100 * g[3] / tot_s:5.1f}%  {' '.join(ops[:12])}")
