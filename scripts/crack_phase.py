#!/usr/bin/env python3
"""Step time over the course of a cracking run (chunks of K steps): where k_crit matters."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 6
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 10
K = int(sys.argv[3]) if len(sys.argv) > 3 else 200
p = ci.config(cfg)
sim = cem.Simulation.from_problem(p)
for c in range(chunks):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream)
    sim.step(K, 1)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    st = sim.state(records=True)
    sim.set_profiling(True)
    sim.step(20, 1)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    print(f"steps {c * (K + 20):6d}+{K}: {e0.elapsed_time(e1) / K * 1e3:7.1f} us/step, splits {st.rec_elem.size:6d}; "
          + ", ".join(f"{k.split('_')[1]} {v / 20 * 1e3:.1f}" for k, v in kt.items()), flush=True)
