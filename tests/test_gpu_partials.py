"""GPU parity of the two nodal-assembly modes (reading R27, DESIGN.md §6 "Partials").

Default (partials): stage C sums the contributions of its block's tets to each node of the
block's node list exactly (TwoSum chains) and stores one 48-B partial per (block, node); stage
D adds a node's partials.  CEM_PARTIALS=0: the round-1/2 force slots (96 B per tet), summed by
stage D with the same exact accumulation.  Both must equal the oracle (exact sum rounded once)
bit for bit, on one domain and on P sub-domains, on the staged, persistent and wave launch
paths, and the wide-exponent early steps of a wave problem (where contributions span many
orders of magnitude).
"""
import numpy as np
import pytest

import cem_inputs as ci
from test_gpu_parity import _gpu, assert_parity, run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["1", "0"], ids=["partials", "slots"])
def test_cfg0_both_modes(mode, monkeypatch):
    monkeypatch.setenv("CEM_PARTIALS", mode)
    p = ci.config(0)
    sim, orc = run_pair(p, p.steps, 1, chunks=2)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


@pytest.mark.parametrize("mode", ["1", "0"], ids=["partials", "slots"])
@pytest.mark.parametrize("seed", [3, 4])
def test_random_problems_both_modes(mode, seed, monkeypatch):
    """jittered lattices with inactive tets, a velocity patch and pre-damage, many blocks,
    ragged tail"""
    monkeypatch.setenv("CEM_PARTIALS", mode)
    rng = np.random.default_rng(seed)
    cells = tuple(int(c) for c in rng.integers(7, 19, size=3))
    p = ci.notched_plate(cells=cells, dims=(0.02, 0.015, 0.01), seed=seed, steps=0)
    st = p.tet_state.copy()
    st[rng.random(st.size) < 0.05] = 0
    p.tet_state = st
    p.tet_gc[rng.random(st.size) < 0.01] = 0.0
    sim, orc = run_pair(p, 150, 1, chunks=3)
    assert_parity(sim, orc, p)


def _traction_bar(n=120):
    """a jittered bar pushed at x = 0: ahead of the wave front the nodal forces fall off by
    ~20 orders of magnitude per 10 steps (measured: 1e-135 of the peak after 60 steps)"""
    p = ci.notched_plate(cells=(n, 2, 2), dims=(0.12, 0.002, 0.002), seed=0, notch=False, steps=0, jitter=0.05)
    ijk, X, T = p.node_ijk, p.X, p.tets
    faces = [[T[e, a] for a in range(4) if a != f] for e in range(T.shape[0]) for f in range(4)
             if all(ijk[T[e, a], 0] == 0 for a in range(4) if a != f)]
    return ci.make_problem(X, T, E=p.E, nu=p.nu, rho=p.rho, tet_gc=np.full(T.shape[0], np.inf), tface=faces,
                           tface_t=np.tile([1e6, 0.0, 0.0], (len(faces), 1)))


@pytest.mark.parametrize("mode", ["1", "0"], ids=["partials", "slots"])
def test_wave_front_tails(mode, monkeypatch):
    """The regime where the GPU's TwoSum accumulation is not guaranteed exact (R27): a node's
    contributions span hundreds of orders of magnitude.  Bitwise every 5 steps for 80 steps."""
    monkeypatch.setenv("CEM_PARTIALS", mode)
    p = _traction_bar()
    cem = _gpu()
    import oracle
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    lo = 1.0
    for _ in range(16):
        sim.step(5, 0)
        orc.run(5, 0)
        g, o = sim.state(), orc.state()
        assert np.array_equal(g.u, o["u"]) and np.array_equal(g.v, o["v"]) and np.array_equal(g.a, o["a"])
        x = np.abs(o["a"][o["a"] != 0])
        lo = min(lo, x.min() / x.max())
    assert lo < 1e-100   # the regime is really exercised


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_slots(P, monkeypatch):
    """P sub-domains (loopback halo) with force slots (the default partials are covered by
    tests/test_gpu_dist.py): bitwise equal to the single-domain oracle."""
    monkeypatch.setenv("CEM_PARTIALS", "0")
    from test_gpu_dist import check
    check(ci.config(0), P, 200)


@pytest.mark.parametrize("flags", ["PERSISTENT", "WAVE"])
def test_other_paths_partials(flags, monkeypatch):
    cem = _gpu()
    fl = 0
    if flags == "PERSISTENT":
        fl = cem.CEM_F_PERSISTENT
    else:
        monkeypatch.setenv("CEM_WAVE", "1")
    p = ci.config(0)
    sim, orc = run_pair(p, 200, 1, chunks=2, flags=fl)
    assert_parity(sim, orc, p)
