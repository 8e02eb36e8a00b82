#!/usr/bin/env python3
"""Per-step time and split count over config 3's cracking window (steps 0..N): events between single
steps enqueued back to back (the host runs ahead), then a profiled pass for the stage split.

  python scripts/crack_window.py [N=60] [cfg=3]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = ci.config(cfg)
sim = cem.Simulation.from_problem(p)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
torch.cuda.synchronize()
ev[0].record(sim.torch_stream)
for s in range(N):
    sim.step(1, 1)
    ev[s + 1].record(sim.torch_stream)
torch.cuda.synchronize()
t = [ev[s].elapsed_time(ev[s + 1]) * 1e3 for s in range(N)]
sim.close()

sim = cem.Simulation.from_problem(p)
prev = 0
rows = []
for s in range(N):
    sim.set_profiling(True)
    sim.step(1, 1)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    n = sim.state(records=True).rec_elem.size
    rows.append((n - prev, kt))
    prev = n
for s in range(N):
    d, kt = rows[s]
    print(f"step {s:3d}: {t[s]:6.1f} us  splits {d:5d}  " + "  ".join(f"{k.split('_')[1]} {v * 1e3:5.1f}" for k, v in kt.items()),
          flush=True)
print(f"[{os.environ.get('CEM_CRITB_MIN', 'default')}] mean 5-25: {sum(t[5:25]) / 20:.1f} us; mean {N - 20}-{N}: {sum(t[N - 20:]) / 20:.1f} us")
