"""GPU parity of the ES-H-FEM hexahedral path (cem_hex.cu, k_hexcrit) through the
C ABI, bitwise against the hex oracle (oracle/cem_oracle_hex.c, pinned by tests/test_oracle_hex.py and
tests/test_oracle_hex_crack.py): u, v, a, the lumped masses, the hex states and the split records
(patterns III-VI, remainder tets) equal bit for bit, and the north-star relative L2 of u first."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from test_gpu_parity import _gpu

pytestmark = pytest.mark.gpu


def _pair(p, steps, chunks=1, crack_every=0, flags=0):
    cem = _gpu()
    sim = cem.Simulation.from_problem(p, flags=flags)
    orc = oracle.HexOracle(p, flags=flags)
    per = steps // chunks
    for _ in range(chunks):
        sim.step(per, crack_every)
        orc.run(per, crack_every)
    return sim, orc


def _assert_bitwise(sim, orc):
    g = sim.state(records=False)
    o = orc.state()
    assert g.dt == orc.dt
    du = np.linalg.norm(g.u - o["u"]) / max(np.linalg.norm(o["u"]), 1e-300)
    assert du <= 1e-11
    assert np.array_equal(g.mass, o["m"])
    for k in ("u", "v", "a"):
        bad = np.nonzero(getattr(g, k) != o[k])
        assert bad[0].size == 0, f"{k} differs at nodes {bad[0][:10]}"
    assert np.abs(o["u"]).max() > 0
    return g


def test_hex_block_traction_bitwise():
    p = ci.hex_block((12, 8, 4), dims=(0.06, 0.04, 0.02), seed=8)
    sim, orc = _pair(p, 400, chunks=2)
    _assert_bitwise(sim, orc)


@pytest.mark.parametrize("cells,seed", [((37, 13, 5), 3), ((3, 2, 1), 4), ((65, 1, 4), 5)])
def test_hex_ragged_distorted_inactive_body_dirichlet(cells, seed):
    """Sizes around block boundaries, strong jitter, inactive hexes, a body force and a
    prescribed-velocity ramp on one face."""
    p = ci.hex_block(cells, dims=(0.002 * cells[0], 0.002 * cells[1], 0.002 * cells[2]), seed=seed, jitter=0.15)
    rng = np.random.default_rng(seed)
    p.tet_state = (rng.uniform(size=p.n_tets) > 0.1).astype(np.uint8)
    p.body = (1.0e5, -3.0e5, 2.0e4)
    face = np.flatnonzero(p.node_ijk[:, 0] == 0)
    p.vbc_node = face.astype(np.int32)
    p.vbc_mask = np.full(face.size, 1, np.uint8)
    p.vbc_v0 = np.tile([0.5, 0.0, 0.0], (face.size, 1))
    p.vbc_t0 = 2e-6
    sim, orc = _pair(p, 300, chunks=3)
    _assert_bitwise(sim, orc)


def test_hex_crack_update_rejected():
    cem = _gpu()
    p = ci.hex_block((4, 3, 2))
    sim = cem.Simulation.from_problem(p)
    with pytest.raises(cem.CemError):
        sim.crack_update()
    sim.step(5, 0)
    assert sim.state(records=False).step == 5


def _assert_cracking(sim, orc, p):
    _assert_bitwise(sim, orc)
    g = sim.state()
    r = orc.records()
    assert r.step.size > 0
    assert np.array_equal(g.rec_step, r.step)
    assert np.array_equal(g.rec_elem, r.elem), "split sets differ"
    assert np.array_equal(g.rec_cand, r.cand)
    assert np.array_equal(g.rec_G, r.G)
    assert np.array_equal(g.rec_area, r.area)
    assert np.array_equal(g.tet_state, orc.elements()["hex_active"])
    assert g.dissipated == orc.dissipated
    return r


def test_hex_cracking_bitwise():
    """Patterns III-VI and remainder-tet splits (R28, R29) on a notched, pulled hex block: 400 steps with
    the criterion every step, every pattern family and tet splits present in the record."""
    p = ci.hex_block((10, 6, 2), dims=(0.05, 0.03, 0.01), seed=2, traction=4e6, gc=2.0, notch=0.3)
    sim, orc = _pair(p, 400, chunks=2, crack_every=1)
    r = _assert_cracking(sim, orc, p)
    hexk = r.cand[r.elem < p.n_tets]
    assert (hexk < 12).any() and ((hexk >= 12) & (hexk < 36)).any()
    assert ((hexk >= 36) & (hexk < 60)).any() and (hexk >= 60).any()
    assert (r.elem >= p.n_tets).any()


@pytest.mark.parametrize("cells,seed,every,flags", [((13, 7, 3), 3, 3, 0), ((9, 5, 2), 4, 1, 0x40)])
def test_hex_cracking_ragged_variants(cells, seed, every, flags):
    """Ragged sizes around the 128/256-thread blocks, strong jitter, a criterion every 3rd step, and the
    R11v variant (both front edges stretched)."""
    p = ci.hex_block(cells, dims=(0.004 * cells[0], 0.004 * cells[1], 0.004 * cells[2]), seed=seed,
                     jitter=0.12, traction=5e6, gc=1.0, notch=0.4)
    sim, orc = _pair(p, 300, chunks=3, crack_every=every, flags=flags)
    _assert_cracking(sim, orc, p)


def test_hex_criterion_without_early_out_bitwise():
    """k_hexcrit skips hexes whose bound max g * max |du| (1 + 1e-6) <= Gc (pinned on the CPU by
    tests/test_early_out_bounds.py); with CEM_F_NO_EARLY_OUT every active hex evaluates its 84
    candidates.  Both equal the oracle (the default path in test_hex_cracking_bitwise)."""
    cem = _gpu()
    p = ci.hex_block((10, 6, 2), dims=(0.05, 0.03, 0.01), seed=2, traction=4e6, gc=2.0, notch=0.3)
    sim = cem.Simulation.from_problem(p, flags=cem.CEM_F_NO_EARLY_OUT)
    orc = oracle.HexOracle(p)
    sim.step(300, 1)
    orc.run(300, 1)
    _assert_cracking(sim, orc, p)


def test_hex_cracked_energy_ledger():
    """cem_energy after splits: strain energy with the mixed smoothing volumes (R29) and U_d."""
    p = ci.hex_block((10, 6, 2), dims=(0.05, 0.03, 0.01), seed=2, traction=4e6, gc=2.0, notch=0.3)
    sim, orc = _pair(p, 200, crack_every=1)
    e = sim.energy()
    o = orc.state()
    assert orc.records().step.size > 0
    assert e["strain"] == pytest.approx(orc.strain_energy(o["u"]), rel=1e-12)
    assert e["kinetic"] == pytest.approx(0.5 * (o["m"][:, None] * o["v"] ** 2).sum(), rel=1e-12)
    assert e["dissipated"] == orc.dissipated


def test_hex_energy_ledger():
    """cem_energy on a hexahedral context: kinetic 1/2 sum m v.v, strain sum psi Vhat/12 (the hex
    oracle's hx_strain_energy), external sum f.u -- equal to the oracle to the rounding of the sums --
    and the discrete balance T + U ~ W of a traction-loaded block."""
    p = ci.hex_block((10, 6, 3), dims=(0.05, 0.03, 0.015), seed=4)
    sim, orc = _pair(p, 300)
    e = sim.energy()
    o = orc.state()
    T = 0.5 * (o["m"][:, None] * o["v"] ** 2).sum()
    W = (orc.fext() * o["u"]).sum()
    U = orc.strain_energy(o["u"])
    assert e["kinetic"] == pytest.approx(T, rel=1e-12)
    assert e["strain"] == pytest.approx(U, rel=1e-12)
    assert e["external"] == pytest.approx(W, rel=1e-12)
    assert e["dissipated"] == 0.0 and e["step"] == 300
    assert abs(e["kinetic"] + e["strain"] - e["external"]) <= 5e-3 * abs(e["external"])
