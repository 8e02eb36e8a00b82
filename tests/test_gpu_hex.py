"""GPU parity of the ES-H-FEM hexahedral path (cem_hex.cu) through the C ABI,
bitwise against the hex oracle (oracle/cem_oracle_hex.c, pinned by tests/test_oracle_hex.py):
u, v, a and the lumped masses equal bit for bit, and the north-star relative L2 of u first."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from test_gpu_parity import _gpu

pytestmark = pytest.mark.gpu


def _pair(p, steps, chunks=1):
    cem = _gpu()
    sim = cem.Simulation.from_problem(p)
    orc = oracle.HexOracle(p)
    per = steps // chunks
    for _ in range(chunks):
        sim.step(per, 0)
        orc.run(per)
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


def test_hex_rejects_cracking():
    cem = _gpu()
    p = ci.hex_block((4, 3, 2))
    sim = cem.Simulation.from_problem(p)
    with pytest.raises(cem.CemError):
        sim.step(5, 1)
    with pytest.raises(cem.CemError):
        sim.crack_update()
    sim.step(5, 0)
    assert sim.state(records=False).step == 5


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
