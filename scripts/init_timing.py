import time, os, sys
sys.path.insert(0, '/root/repo')
import cem_inputs as ci
t0=time.perf_counter(); p = ci.config(3); t1=time.perf_counter()
print("inputs", t1-t0, flush=True)
import torch
import paper_2508_04076_b200 as cem
torch.cuda.init()
for i in range(2):
    torch.cuda.synchronize()
    t0=time.perf_counter(); s = cem.Simulation.from_problem(p); torch.cuda.synchronize(); t1=time.perf_counter()
    s.step(1000,1); st = s.state(records=True); t2=time.perf_counter()
    print(f"init {t1-t0:.3f}s steps+state {t2-t1:.3f}s", flush=True)
    s.close()
