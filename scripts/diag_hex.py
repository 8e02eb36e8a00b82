"""(diagnostic) first divergence of the hex cracking path from the hex oracle"""
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, cem_inputs as ci, oracle
from test_gpu_parity import _gpu
cem = _gpu()
p = ci.hex_block((10, 6, 2), dims=(0.05, 0.03, 0.01), seed=2, traction=4e6, gc=2.0, notch=0.3)
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sim = cem.Simulation.from_problem(p); orc = oracle.HexOracle(p)
for it in range(400 // chunk):
    sim.step(chunk, 1); orc.run(chunk, 1)
    g = sim.state(); r = orc.records(); o = orc.state()
    same = g.rec_elem.size == r.elem.size and np.array_equal(g.rec_elem, r.elem) and np.array_equal(g.rec_step, r.step)
    du = np.abs(g.u - o["u"]).max()
    if not same or du > 0:
        print("step", (it + 1) * chunk, "gpu", g.rec_elem.size, "orc", r.elem.size, "du", du)
        d = np.nonzero((g.rec_elem[:min(g.rec_elem.size, r.elem.size)] != r.elem[:min(g.rec_elem.size, r.elem.size)]))[0]
        i0 = d[0] if d.size else min(g.rec_elem.size, r.elem.size)
        print(" first diff at", i0)
        print(" gpu", list(zip(g.rec_step[i0:i0+8], g.rec_elem[i0:i0+8], g.rec_cand[i0:i0+8], g.rec_G[i0:i0+8])))
        print(" orc", list(zip(r.step[i0:i0+8], r.elem[i0:i0+8], r.cand[i0:i0+8], r.G[i0:i0+8])))
        break
else:
    print("identical", r.elem.size)
