"""GPU parity of the dataflow ("wave") launch path (DESIGN.md §6 "Wavefront") in all its
configurations: chunk count K, lookahead, CUDA-graph replay length M, switching to and from the
staged path (profiling, the long-list criterion kernels, cem_crack_update) -- bitwise against the
oracle.  The wave path is opt-in (CEM_WAVE=1): it measured slower than the staged path on B200
(DESIGN.md §6), but it stays correct and tested."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from test_gpu_parity import _gpu, assert_parity

pytestmark = pytest.mark.gpu


def _plate():
    return ci.notched_plate(cells=(40, 16, 4), dims=(0.1, 0.04, 0.005), seed=11, steps=300)


@pytest.mark.parametrize("K,LA,M", [(1, 0, 0), (1, 1, 16), (3, 0, 5), (8, 1, 16), (8, 2, 7), (64, 1, 16),
                                    (1000, 1, 3)])
@pytest.mark.parametrize("case", ["cfg0", "plate", "predamage"])
def test_wave_configurations_bitwise(case, K, LA, M, monkeypatch):
    monkeypatch.setenv("CEM_WAVE", "1")
    monkeypatch.setenv("CEM_WAVE_K", str(K))
    monkeypatch.setenv("CEM_WAVE_LA", str(LA))
    monkeypatch.setenv("CEM_GRAPH_M", str(M))
    cem = _gpu()
    if case == "cfg0":
        p, steps = ci.config(0), 200
    elif case == "plate":
        p, steps = _plate(), 150
    else:
        p, steps = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=120), 120
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    for n in (37, steps - 37):      # graph blocks and eager remainders
        sim.step(n, 1)
        orc.run(n, 1)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


def test_wave_mixed_with_staged_and_crack_update(monkeypatch):
    """Wave steps, profiled (staged) steps, criterion-free steps and cem_crack_update interleaved:
    bitwise equal to the oracle up to the crack update, whose splits equal the oracle's criterion
    on that state; the continuation equals the staged path's (CEM_WAVE=0) bit for bit."""
    monkeypatch.setenv("CEM_WAVE", "1")
    monkeypatch.setenv("CEM_GRAPH_M", "8")
    cem = _gpu()
    p = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=200)

    def run(sim):
        sim.step(30, 1)
        sim.set_profiling(True)
        sim.step(11, 1)
        sim.set_profiling(False)
        sim.step(20, 0)
        return sim

    sim = run(cem.Simulation.from_problem(p))
    orc = oracle.Oracle(p)
    orc.run(30, 1); orc.run(11, 1); orc.run(20, 0)
    assert_parity(sim, orc, p)
    G, k, A, fl = orc.criterion(orc.state()["u"])
    n = sim.crack_update()
    assert n == int(fl.sum())
    sim.step(40, 1)
    monkeypatch.setenv("CEM_WAVE", "0")
    ref = run(cem.Simulation.from_problem(p))
    assert ref.crack_update() == n
    ref.step(40, 1)
    a, b = sim.state(), ref.state()
    for key in ("u", "v", "a", "mass", "tet_state", "rec_elem", "rec_step", "rec_cand", "rec_G"):
        assert np.array_equal(getattr(a, key), getattr(b, key)), key


def test_wave_opt_in_counts_launches(monkeypatch):
    """CEM_WAVE=1 launches the wave kernels (more launches per step than the staged kernels)
    and stays bitwise equal to the oracle."""
    monkeypatch.setenv("CEM_WAVE", "1")
    monkeypatch.setenv("CEM_GRAPH_M", "0")
    cem = _gpu()
    p = ci.config(0)
    sim = cem.Simulation.from_problem(p)
    l0 = sim.launch_count
    sim.step(32, 1)
    per_step = (sim.launch_count - l0) / 32
    assert per_step > 10
    orc = oracle.Oracle(p).run(32, 1)
    assert_parity(sim, orc, p)


@pytest.mark.parametrize("case", ["cfg0", "plate", "predamage"])
def test_pipelined_stage_c_bitwise(case, monkeypatch):
    """The software-pipelined stage C (k_Cp, cp.async ring of D blocks per persistent CTA; opt-in
    CEM_C_PIPE=1, measured slower -- DESIGN.md §6) gives the oracle's bits."""
    monkeypatch.setenv("CEM_C_PIPE", "1")
    cem = _gpu()
    if case == "cfg0":
        p, steps = ci.config(0), 200
    elif case == "plate":
        p, steps = _plate(), 150
    else:
        p, steps = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=120), 120
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    sim.step(steps, 1)
    orc.run(steps, 1)
    assert assert_parity(sim, orc, p).rec_elem.size > 0
