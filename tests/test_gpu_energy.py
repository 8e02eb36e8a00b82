"""GPU parity of the energy ledger (cem_energy) against the oracle's
orc_energy.

Per-element terms are computed in the oracle's association order; only the final sums differ
(per-block partials in a fixed order vs one sequential sum), so the bar is the rounding bound
of a sum of n terms: |err| <= n * eps * sum|terms|.  For the non-negative kinetic and strain
sums that is a relative bound; for the signed work sums it is taken relative to the larger of
the ledger's magnitudes.  U_d is summed in the same (step, element) order on both sides:
bitwise.  Two GPU runs (and the staged vs persistent paths) agree bitwise."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_04076_b200 as cem
    return cem


def _check(g, o, n_terms):
    tol = 4 * n_terms * EPS
    assert g["kinetic"] == pytest.approx(o["kinetic"], rel=tol, abs=1e-300)
    assert g["strain"] == pytest.approx(o["strain"], rel=tol, abs=1e-300)
    scale = max(abs(o["kinetic"]), abs(o["strain"]), abs(o["external"]), abs(o["reaction"]), 1e-300)
    assert abs(g["external"] - o["external"]) <= tol * scale
    assert abs(g["reaction"] - o["reaction"]) <= tol * scale
    assert g["dissipated"] == o["dissipated"]


@pytest.mark.parametrize("flags", [0, 8])
def test_ledger_traction_with_fracture(flags):
    cem = _gpu()
    p = ci.config(0)
    sim = cem.Simulation.from_problem(p, flags=flags)
    orc = oracle.Oracle(p)
    for _ in range(4):
        sim.step(40, 1)
        orc.run(40, 1)
        g, o = sim.energy(), orc.energy()
        assert g["step"] == orc.step_count
        _check(g, o, p.n_tets * 6)
        assert g["reaction"] == 0.0
    assert o["dissipated"] > 0.0 and o["external"] > 0.0


def test_ledger_prescribed_velocity():
    """Edge-impact stand-in (velocity ramp on x = 0, fracture on): W_R accumulated by the
    node-update kernel."""
    cem = _gpu()
    p = ci.edge_impact_plate(cells=(40, 20, 3), dims=(0.04, 0.02, 0.003), t0=2e-7)
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    for _ in range(3):
        sim.step(50, 1)
        orc.run(50, 1)
        g, o = sim.energy(), orc.energy()
        _check(g, o, p.n_tets * 6)
    assert o["reaction"] > 0.0


def test_ledger_deterministic_and_path_independent():
    cem = _gpu()
    p = ci.edge_impact_plate(cells=(30, 16, 3), dims=(0.03, 0.016, 0.003), t0=2e-7)
    out = []
    for flags in (0, 0, 8):
        sim = cem.Simulation.from_problem(p, flags=flags)
        sim.step(60, 1)
        out.append(sim.energy())
        sim.close()
    assert out[0] == out[1] == out[2]


def test_ledger_full_size_edge_impact():
    """BASELINE.json configs[2] (1.08M tets, Dirichlet-driven) for a few steps."""
    cem = _gpu()
    p = ci.config(2)
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    sim.step(6, 1)
    orc.run(6, 1)
    _check(sim.energy(), orc.energy(), p.n_tets * 6)


def test_ledger_compact_tension():
    """N2 workload: driven and held slot faces both enter the reaction work."""
    cem = _gpu()
    p = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6)
    sim = cem.Simulation.from_problem(p)
    orc = oracle.Oracle(p)
    sim.step(200, 1)
    orc.run(200, 1)
    g, o = sim.energy(), orc.energy()
    _check(g, o, p.n_tets * 6)
    assert o["reaction"] > 0.0
