import os, sys, torch
sys.path.insert(0, '/root/repo')
import cem_inputs as ci, paper_2508_04076_b200 as cem
p = ci.config(3)
for ce in (1, 0, 1, 0):
    sim = cem.Simulation.from_problem(p)
    sim.step(20, ce); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream); sim.step(400, ce); e1.record(sim.torch_stream); torch.cuda.synchronize()
    print(f"crack_every={ce}: {e0.elapsed_time(e1)/400*1e3:.1f} us/step", flush=True)
    sim.close()
