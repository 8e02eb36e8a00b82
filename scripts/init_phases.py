#!/usr/bin/env python3
"""cem_init_mesh phase times (CEM_TIMING=1) for config 3, cold then warm, plus the e2e pieces."""
import os
import sys
import time

os.environ["CEM_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

p = ci.config(3)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = cem.Simulation.from_problem(p)
    torch.cuda.synchronize()
    print(f"[run {it}] cem_init_mesh {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
    s.close()
