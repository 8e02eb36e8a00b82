#!/usr/bin/env python3
"""Whole BASELINE.json workload runs (config k for its stated step count): device time per step."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

for k in [int(c) for c in (sys.argv[1:] or ["1", "2"])]:
    p = ci.config(k)
    sim = cem.Simulation.from_problem(p)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(sim.torch_stream)
    sim.step(p.steps, 1)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = sim.state(records=True)
    print(f"cfg{k}: {p.steps} steps, {p.n_tets} tets: {ms:.1f} ms = {ms / p.steps * 1e3:.1f} us/step "
          f"({p.n_tets * p.steps / ms / 1e6:.2f} G tet-steps/s), splits {st.rec_elem.size}, "
          f"lib {os.path.basename(cem.LIB_PATH)}", flush=True)
    sim.close()
