#!/usr/bin/env python3
"""The FMA ("fast") build against the oracle at the north star's tolerance (SURVEY.md §8(c)
"Parity protocol"): relative L2 of u <= 1e-11 per 1000 steps and an identical split set.  Run with
CEM_LIB pointing at libcem_fast.so; prints one JSON line per case."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import oracle  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

cases = [(0, 200), (1, 1000), (3, 1000)] if len(sys.argv) < 2 else [tuple(map(int, a.split(":"))) for a in sys.argv[1:]]
for cfg, steps in cases:
    p = ci.config(cfg)
    sim = cem.Simulation.from_problem(p)
    sim.step(steps, 1)
    g = sim.state()
    o = oracle.Oracle(p).run(steps, 1)
    s = o.state()
    r = o.records()
    du = float(np.linalg.norm(g.u - s["u"]) / np.linalg.norm(s["u"]))
    same_split = bool(np.array_equal(np.sort(g.rec_elem), np.sort(r.elem)))
    same_steps = bool(same_split and np.array_equal(g.rec_step, r.step))
    bitwise = bool(np.array_equal(g.u, s["u"]))
    print(json.dumps({"cfg": cfg, "steps": steps, "lib": os.path.basename(cem.LIB_PATH), "rel_l2_u": du,
                      "same_split_set": same_split, "same_split_steps": same_steps, "splits": int(r.elem.size),
                      "bitwise_u": bitwise}), flush=True)
    sim.close()
