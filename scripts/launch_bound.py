#!/usr/bin/env python3
"""Is cem_step launch-bound on a config?  Host time to enqueue K steps vs device time."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["0", "1", "6", "3"])]:
    p = ci.config(cfg)
    sim = cem.Simulation.from_problem(p)
    sim.step(20, 1)
    torch.cuda.synchronize()
    K = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream)
    t0 = time.perf_counter()
    sim.step(K, 1)
    t1 = time.perf_counter()
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    print(f"cfg{cfg} ({p.n_tets} tets): device {e0.elapsed_time(e1) / K * 1e3:.2f} us/step, "
          f"host enqueue {(t1 - t0) / K * 1e6:.2f} us/step", flush=True)
    sim.close()
