#!/usr/bin/env python3
"""Short config run for launch lists under ncu: W warm-up steps + K steps (env knobs as wave_sweep)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

cfg = int(os.environ.get("CEM_CFG", "3"))
W, K = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else ("60", "10")))
p = ci.config(cfg)
sim = cem.Simulation.from_problem(p)
sim.step(W, 1)
torch.cuda.synchronize()
sim.step(K, 1)
torch.cuda.synchronize()
print("done", sim.state(records=False).n_active)
