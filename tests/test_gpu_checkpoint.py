"""Checkpoint / resume (include/cem.h cem_set_state): a snapshot taken with
cem_get_state and restored with cem_set_state -- into a fresh context or back into the same
one -- continues bitwise as if the run had never stopped, and equals the oracle's uninterrupted
run (u, v, a, masses, active flags, every split record, U_d)."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from test_gpu_parity import _gpu, assert_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["cfg0", "edge_impact", "predamage"])
def test_resume_in_fresh_context_equals_oracle(case):
    cem = _gpu()
    if case == "cfg0":
        p, n1, n2 = ci.config(0), 120, 80
    elif case == "edge_impact":
        p, n1, n2 = ci.edge_impact_plate(cells=(40, 20, 3), dims=(0.04, 0.02, 0.003), steps=300), 150, 150
    else:
        p, n1, n2 = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=300), 4, 60
    a = cem.Simulation.from_problem(p)
    a.step(n1, 1)
    snap = a.state(records=True)
    assert snap.rec_elem.size > 0 or case == "edge_impact"
    a.close()
    b = cem.Simulation.from_problem(p)
    b.step(7, 1)                       # some other state first: everything must be overwritten
    b.set_state(snap)
    b.step(n2, 1)
    orc = oracle.Oracle(p)
    orc.run(n1 + n2, 1)
    g = assert_parity(b, orc, p)
    assert g.rec_elem.size > snap.rec_elem.size or case == "edge_impact"


def test_rewind_same_context_is_bitwise():
    cem = _gpu()
    p = ci.config(0)
    ref = cem.Simulation.from_problem(p)
    ref.step(100, 1)
    r = ref.state()
    s = cem.Simulation.from_problem(p)
    s.step(50, 1)
    snap = s.state()
    s.step(37, 1)                      # run ahead, then rewind to step 50
    s.set_state(snap)
    s.step(50, 1)
    g = s.state()
    assert g.step == 100
    for k in ("u", "v", "a", "mass", "tet_state", "rec_elem", "rec_step", "rec_G", "rec_area"):
        assert np.array_equal(getattr(g, k), getattr(r, k)), k
    assert g.dissipated == r.dissipated


def test_set_state_persistent_path():
    """the persistent wavefront kernel's per-block step counters are refilled after a restore"""
    cem = _gpu()
    p = ci.config(0)
    a = cem.Simulation.from_problem(p, flags=cem.CEM_F_PERSISTENT)
    a.step(60, 1)
    snap = a.state()
    b = cem.Simulation.from_problem(p, flags=cem.CEM_F_PERSISTENT)
    b.set_state(snap)
    b.step(40, 1)
    orc = oracle.Oracle(p)
    orc.run(100, 1)
    assert_parity(b, orc, p)


def test_set_state_reaction_work_not_restored_and_hex_refused():
    cem = _gpu()
    p = ci.edge_impact_plate(cells=(20, 10, 2), dims=(0.02, 0.01, 0.002), steps=50)
    a = cem.Simulation.from_problem(p)
    a.step(30, 0)
    snap = a.state()
    a.set_state(snap)
    assert np.isnan(a.energy()["reaction"])   # (not part of the checkpoint, include/cem.h)
    h = cem.Simulation.from_problem(ci.hex_block((6, 4, 3)))
    hs = h.state()
    with pytest.raises(cem.CemError) as ei:
        h.set_state(hs)
    assert ei.value.status == cem.CEM_ESTATE
