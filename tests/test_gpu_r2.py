"""GPU parity, round 2: the north-star horizon at full size, the load / criterion options added
this round, and the CEM_DEVICE readback -- all through the C ABI, bitwise against the oracle.

North star (BASELINE.json): "an identical set of split elements on the same seeded inputs, and
nodal displacements within a relative L2 error of 1e-11 per 1000 steps"; configs
0 and 1, config 2 in full, config 3 at P = 1, config 4 for its first 1000 steps.  assert_parity
checks the 1e-11 bound first and then bitwise equality of u, v, a, masses, flags and records.
"""
import os

import numpy as np
import pytest

import cem_inputs as ci
import oracle
from test_gpu_parity import _gpu, assert_parity

pytestmark = pytest.mark.gpu


def _pair(prob, steps, crack_every=1, flags=0, chunks=1):
    cem = _gpu()
    sim = cem.Simulation.from_problem(prob, flags=flags)
    orc = oracle.Oracle(prob, flags=flags & oracle.Oracle.FRONT_BOTH_STRETCHED)
    per = steps // chunks
    for _ in range(chunks):
        sim.step(per, crack_every)
        orc.run(per, crack_every)
    return sim, orc


# ------------------------------------------------------------------ north-star horizons, full size
# The oracle sets the wall time (config 4: 7.68M tets, ~0.5 s per oracle step on 16 cores).  The
# default suite must fit a driver's GPU-test slot, so it runs configs 1 and 3 over the full
# 1000-step horizon, config 2 for 1000 of its 2000 steps and config 4 for its first 100;
# CEM_LONG_TESTS=1 runs SURVEY.md §4's full horizons (config 2 in full, config 4 for 1000 steps:
# ~12 more minutes; logs of those runs on this build: profiles/r02c_pytest_gpu.log, r02d_pytest_gpu.log).
_LONG = os.environ.get("CEM_LONG_TESTS") == "1"
_HORIZONS = [(1, 1000), (3, 1000), (2, 2000 if _LONG else 1000), (4, 1000 if _LONG else 100)]


@pytest.mark.parametrize("cfg,steps", _HORIZONS, ids=[f"cfg{c}-{n}" for c, n in _HORIZONS])
def test_full_size_north_star_horizon(cfg, steps):
    """BASELINE configs at full size over the north star's 1000-step horizon (config 2 in full and
    config 4 for its first 1000 steps with CEM_LONG_TESTS=1), crack criterion and split pass every
    step, in the bench's launch configuration."""
    p = ci.config(cfg)
    sim, orc = _pair(p, steps, 1)
    g = assert_parity(sim, orc, p)
    if cfg in (1, 3):
        assert g.rec_elem.size > 0      # non-vacuous split parity (config 3: pre-damage; 1: notch)


# ------------------------------------------------------------------ loads: body force, nodal forces
def test_body_force_and_nodal_forces_bitwise():
    p = ci.config(0)
    rng = np.random.default_rng(9)
    p.body = (2.0e5, -9.81 * p.rho * 5e3, 1.0e4)
    p.f_nodal = np.zeros((p.n_nodes, 3))
    pick = rng.choice(p.n_nodes, 40, replace=False)
    p.f_nodal[pick] = rng.normal(size=(40, 3)) * 20.0
    sim, orc = _pair(p, 200, 1)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


def test_body_force_only_multiblock():
    """A body force on a plate spanning many blocks, prescribed-velocity load elsewhere."""
    p = ci.edge_impact_plate(cells=(40, 20, 3), dims=(0.04, 0.02, 0.003), steps=200)
    p.body = (0.0, -3.0e7, 0.0)
    sim, orc = _pair(p, 200, 1, chunks=2)
    assert_parity(sim, orc, p)


# ------------------------------------------------------------------ criterion variant R11
@pytest.mark.parametrize("critb_min", ["1024", "0"])
@pytest.mark.parametrize("case", ["cfg0", "predamage"])
def test_front_both_stretched_variant_bitwise(case, critb_min, monkeypatch):
    monkeypatch.setenv("CEM_CRITB_MIN", critb_min)
    cem = _gpu()
    if case == "cfg0":
        p, steps = ci.config(0), 200
    else:
        p, steps = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=300), 300
    sim, orc = _pair(p, steps, 1, flags=cem.CEM_F_FRONT_BOTH_STRETCHED)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0
    if case == "cfg0":
        # the variant is a different reading: on config 0 it changes the records (non-vacuous);
        # on the pre-damaged block (Gc_e = 0) the winning candidates have both fronts stretched
        ref = oracle.Oracle(p).run(steps, 1).records()
        assert not (np.array_equal(ref.elem, g.rec_elem) and np.array_equal(ref.cand, g.rec_cand)
                    and np.array_equal(ref.G, g.rec_G))


@pytest.mark.parametrize("critb_min", ["1024", "0"])
def test_no_early_out_bitwise(critb_min, monkeypatch):
    """CEM_F_NO_EARLY_OUT evaluates every listed tet in full (k_filter passes all of them)."""
    monkeypatch.setenv("CEM_CRITB_MIN", critb_min)
    cem = _gpu()
    p = ci.config(0)
    sim, orc = _pair(p, 200, 1, flags=cem.CEM_F_NO_EARLY_OUT)
    assert assert_parity(sim, orc, p).rec_elem.size > 0


# ------------------------------------------------------------------ CEM_DEVICE readback
def test_device_readback_matches_host_and_oracle():
    p = ci.weak_scaling_block(P=1, cells_per_rank=(24, 20, 5), steps=150)
    sim, orc = _pair(p, 150, 1)
    d = sim.device_state()
    h = sim.state()
    o = orc.state()
    for k in ("u", "v", "a", "mass", "tet_state"):
        arr = d[k].cpu().numpy()
        assert np.array_equal(arr, getattr(h, k)), k
    assert np.array_equal(d["u"].cpu().numpy(), o["u"])
    r = orc.records()
    assert r.elem.size > 0
    assert np.array_equal(d["rec_elem"].cpu().numpy(), r.elem)
    assert np.array_equal(d["rec_step"].cpu().numpy(), r.step)
    assert np.array_equal(d["rec_cand"].cpu().numpy(), r.cand)
    assert np.array_equal(d["rec_G"].cpu().numpy(), r.G)
    assert np.array_equal(d["rec_area"].cpu().numpy(), r.area)
    assert d["dissipated"] == orc.dissipated and d["step"] == 150


def test_user_stream_ordering():
    """Work the caller enqueues on its stream after cem_step sees the stepped state (the library
    runs on a private stream fenced against the caller's, include/cem.h "Asynchrony")."""
    import torch
    cem = _gpu()
    p = ci.config(0)
    s = torch.cuda.Stream()
    sim = cem.Simulation.from_problem(p, stream=s)
    orc = oracle.Oracle(p).run(60, 1)
    sim.step(60, 1)
    d = sim.device_state()
    with torch.cuda.stream(s):
        x = d["u"].clone()      # on the caller's stream, no explicit synchronisation
    s.synchronize()
    assert np.array_equal(x.cpu().numpy(), orc.state()["u"])
