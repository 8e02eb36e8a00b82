#!/usr/bin/env python3
"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck): config 0 with cracking
(staged path incl. the criterion kernels), the long-list kernels forced, the wave path, a hex
block, each compared with the oracle at the end."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import oracle  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

p = ci.config(0)
for name, env in (("staged", {}), ("long-list", {"CEM_CRITB_MIN": "0"}), ("wave", {"CEM_WAVE": "1", "CEM_GRAPH_M": "0"})):
    for k in ("CEM_CRITB_MIN", "CEM_WAVE", "CEM_GRAPH_M"):
        os.environ.pop(k, None)
    os.environ.update(env)
    sim = cem.Simulation.from_problem(p)
    sim.step(40, 1)
    o = oracle.Oracle(p).run(40, 1)
    assert np.array_equal(sim.state().u, o.state()["u"]), name
    sim.close()
    print(f"{name}: 40 steps bitwise", flush=True)
# multi-rank (loopback, copies and P2P stores), the crack-update entry point, device readback
import paper_2508_04076_b200.dist as cdist  # noqa: E402
for flags in (0, cem.CEM_F_P2P):
    g = cdist.LoopbackGroup(p, 3, flags=flags)
    g.step(40, 1)
    assert np.array_equal(g.state()["u"], oracle.Oracle(p).run(40, 1).state()["u"])
    print(f"loopback P=3 flags={flags}: 40 steps bitwise", flush=True)
sim = cem.Simulation.from_problem(p)
sim.step(30, 0)
sim.crack_update()
sim.device_state()
sim.state()
print("crack update + device readback", flush=True)
ph = ci.hex_block((6, 4, 2), dims=(0.03, 0.02, 0.01))
sh = cem.Simulation.from_problem(ph)
sh.step(20, 0)
assert np.array_equal(sh.state(records=False).u, oracle.HexOracle(ph).run(20).state()["u"])
print("hex: 20 steps bitwise", flush=True)
