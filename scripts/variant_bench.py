#!/usr/bin/env python3
"""Time cem_step on config 3 for a given library build (CEM_LIB) and flag set (tuning aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = int(os.environ.get("CEM_CFG", "3"))
p = ci.config(cfg)
sim = cem.Simulation.from_problem(p, flags=flags)
sim.step(10, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(sim.torch_stream)
sim.step(steps, 1)
e1.record(sim.torch_stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"lib={os.path.basename(cem.LIB_PATH)} flags={flags} cfg={cfg}: {ms*1e3:.1f} us/step  {p.n_tets/ms/1e6:.2f} G tet-steps/s")
if os.environ.get("CEM_STATS"):
    sim.state()  # libcem built with -DCEM_POLL_STATS prints the dependency-poll counters here
if os.environ.get("CEM_STAGES"):
    sim.set_profiling(True)
    sim.step(100, 1)
    torch.cuda.synchronize()
    kt = sim.kernel_times()
    print("  stages (events between kernels, no PDL overlap): " +
          ", ".join(f"{k.split('_')[1]} {v * 10:.1f} us" for k, v in kt.items()))
