#!/usr/bin/env python3
"""Per-config table: step time, tet·steps/s and the algorithmic roofline fraction
R_alg = B_alg / step time / measured HBM peak, B_alg = 177 B/node + 17 B/tet + 96 B/edge (SURVEY.md
§8(d)).  Window: steps 10-210 (criterion + split every step).  R_ach (real DRAM bytes) comes from
the ncu pass of scripts/config_table.sh.  Prints one JSON line per config."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6554.9
cfgs = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4, 6]
for k in cfgs:
    p = ci.config(k)
    sim = cem.Simulation.from_problem(p)
    N, E, S = sim.n_nodes, sim.n_tets, sim.n_edges
    sim.step(10, 1)
    n = 200 if E < 5_000_000 else 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(sim.torch_stream)
    sim.step(n, 1)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    balg = 177 * N + 17 * E + 96 * S
    print(json.dumps({"cfg": k, "name": p.name, "tets": E, "nodes": N, "edges": S, "window": f"steps 10-{10 + n}",
                      "us_per_step": round(us, 2), "G_tet_steps_per_s": round(E / us / 1e3, 3),
                      "B_alg_MB": round(balg / 1e6, 2), "R_alg": round(balg / (us * 1e-6) / 1e9 / peak, 4)}), flush=True)
    sim.close()
