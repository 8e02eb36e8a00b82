#!/usr/bin/env python3
"""Hexahedral path on one B200: hex-element steps per second of the ES-H-FEM step,
with and without the crack criterion (patterns III-VI), CUDA events on the caller's stream around the
C-ABI call (the library's private stream is fenced against it on both sides).

B_alg per step (the tet path's model): 177 B/node + 33 B/hex (8 int32 connectivity, state)
+ 96 B per hex edge (sigma written once, read once).  Prints one JSON line per case.
    python scripts/hex_bench.py [nx ny nz] [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

cells = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
steps = int(sys.argv[4]) if len(sys.argv) >= 5 else 50
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6554.9)
h = 0.0005
for name, kw, every in (("elastodynamics", dict(), 0),
                        ("cracking (III-VI, criterion every step)", dict(gc=2.0, notch=0.3, traction=4e6), 1)):
    p = ci.hex_block(cells, dims=(h * cells[0], h * cells[1], h * cells[2]), seed=1, **kw)
    t0 = time.perf_counter()
    sim = cem.Simulation.from_problem(p)
    init_s = time.perf_counter() - t0
    sim.step(5, every)  # warm-up
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(sim.torch_stream)   # the context's stream (opts.stream): the library fences its private stream against it
    sim.step(steps, every)
    b.record(sim.torch_stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    st = sim.state()
    E, N = p.n_tets, p.n_nodes
    nx, ny, nz = cells
    S_h = nx * (ny + 1) * (nz + 1) + ny * (nx + 1) * (nz + 1) + nz * (nx + 1) * (ny + 1)  # hex edges
    B = 177 * N + 33 * E + 96 * S_h
    print(json.dumps({"case": name, "hexes": E, "nodes": N, "steps": steps, "warmup": 5, "ms_per_step": ms,
                      "hex_steps_per_s": E / (ms * 1e-3), "b_alg_bytes_per_step": B,
                      "achieved_gbs": B / (ms * 1e-3) / 1e9, "roofline_frac": B / (ms * 1e-3) / 1e9 / peak,
                      "peak_gbs": peak, "init_s": init_s, "records": int(st.rec_elem.size),
                      "finite": int(np.isfinite(st.u).all())}), flush=True)
    sim.close()
