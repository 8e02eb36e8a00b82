#!/usr/bin/env python3
"""Host cost of enqueueing steps (a few steps, far below the launch-queue depth) vs device time."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["0", "1"])]:
    p = ci.config(cfg)
    sim = cem.Simulation.from_problem(p)
    sim.step(20, 1)
    torch.cuda.synchronize()
    host = []
    for _ in range(20):
        t0 = time.perf_counter()
        sim.step(10, 1)
        host.append((time.perf_counter() - t0) / 10)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream); sim.step(500, 1); e1.record(sim.torch_stream); torch.cuda.synchronize()
    print(f"cfg{cfg}: host enqueue {sorted(host)[len(host)//2]*1e6:.1f} us/step (10-step bursts), "
          f"device {e0.elapsed_time(e1)/500*1e3:.1f} us/step", flush=True)
    sim.close()
