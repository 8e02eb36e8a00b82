#!/usr/bin/env python3
"""Config-3 step time under launch-mode variants (env knobs read at cem_init_mesh):
cracking window (steps 5-25, the driver's bench window) and steady state (steps 60-560).

  python scripts/wave_sweep.py "CEM_WAVE=0" "CEM_WAVE_K=8" "CEM_WAVE_K=16,CEM_GRAPH_M=0" ...
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

cfg = int(os.environ.get("CEM_CFG", "3"))
p = ci.config(cfg)
KNOBS = ("CEM_WAVE", "CEM_WAVE_K", "CEM_WAVE_LA", "CEM_GRAPH_M", "CEM_WAVE_DISCARD", "CEM_L2_PERSIST", "CEM_CRITB_MIN",
         "CEM_C_PIPE", "CEM_STAGE_CHUNKS", "CEM_AB_EDGES", "CEM_CRITB_MIN")


def timed(sim, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(sim.torch_stream)
    sim.step(n, 1)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for spec in sys.argv[1:] or [""]:
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    sim = cem.Simulation.from_problem(p)
    sim.step(5, 1)
    crack = timed(sim, 20)
    sim.step(15, 1)
    steady = timed(sim, 500)
    st = sim.state(records=False)
    print(f"cfg{cfg} [{spec or 'default'}]: cracking {crack:.1f} us/step, steady {steady:.1f} us/step "
          f"({p.n_tets / steady / 1e3:.2f} G tet-steps/s), splits {st.n_records if hasattr(st, 'n_records') else ''}"
          f" active {st.n_active}", flush=True)
    sim.close()
