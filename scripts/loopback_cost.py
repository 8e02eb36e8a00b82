#!/usr/bin/env python3
"""Cost of the multi-rank decomposition on ONE GPU (loopback emulation): config 3 at
P = 2 (global grid 200x100x17, 2.04M tets) as one domain vs two loopback ranks with the P2P halo
(stage D stores into the peer's buffer, an unpack kernel per rank and step).  The ranks run one
after the other on one stream, so the difference is the ghost-layer recompute plus the exchange
kernels -- an upper bound of what is exposed per step when the ranks run concurrently."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cem_inputs as ci  # noqa: E402
import paper_2508_04076_b200 as cem  # noqa: E402
import paper_2508_04076_b200.dist as cdist  # noqa: E402


def timed(obj, stream, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    obj.step(n, 1)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = ci.config(3, P=P)
one = cem.Simulation.from_problem(p)
one.step(60, 1)
t1 = timed(one, one.torch_stream, 200)
one.close()
for flags, name in ((cem.CEM_F_P2P, "P2P stores + unpack"), (0, "pack + copies + unpack")):
    g = cdist.LoopbackGroup(p, P, flags=flags)
    g.step(60, 1)
    tg = timed(g, g.torch_stream, 200)
    print(f"config 3 x P={P} ({p.n_tets} tets): one domain {t1:.1f} us/step; {P} loopback ranks ({name}) "
          f"{tg:.1f} us/step -> decomposition overhead {tg - t1:.1f} us/step ({(tg / t1 - 1) * 100:.1f} %)", flush=True)
