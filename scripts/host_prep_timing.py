#!/usr/bin/env python3
"""Host preprocessing time (cem_workspace_size builds the mesh tables and the storage plan
without device work): CEM_TIMING=1 prints the phases.  Runs without a GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402

p = ci.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    t0 = time.perf_counter()
    b = cem.workspace_size(p.X, p.tets)
    print(f"host preprocessing {time.perf_counter() - t0:.3f} s ({b / 1e6:.0f} MB workspace)", flush=True)
