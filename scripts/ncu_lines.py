#!/usr/bin/env python3
"""Warp-stall samples per CUDA source line of one kernel in an ncu report (needs -lineinfo)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
iss, iex = 4, h.index("Instructions Executed")
lines = []
for r in rows[hi + 1:]:
    if r and r[0].strip():
        try:
            lines.append((int(r[iss]), int(r[iex] or 0), int(r[0]), r[1].strip()))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in lines) or 1
print(f"{kern}: {tot} stall samples")
for s, ex, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  L{ln:<5} ex={ex:<9} {src[:100]}")
