"""Pins of the oracle's energy ledger (oracle/cem_oracle.c orc_energy) against
closed forms and the discrete energy balance.  CPU only."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle


def _block(cells=(6, 4, 3), dims=(0.06, 0.04, 0.03), seed=11, **kw):
    X, T, ijk = ci.kuhn_lattice(cells, dims, seed)
    return X, T, ijk, float(np.prod(dims))


def test_kinetic_rigid_translation():
    """T = 1/2 M s^2 with M = rho * volume (lumped masses partition the mass exactly)."""
    X, T, _, vol = _block()
    p = ci.make_problem(X, T, tet_gc=np.full(T.shape[0], np.inf))
    o = oracle.Oracle(p)
    s = np.array([3.0, -1.5, 0.5])
    o.set_state(u=np.zeros_like(X), v=np.tile(s, (X.shape[0], 1)), a=np.zeros_like(X))
    e = o.energy()
    assert e["kinetic"] == pytest.approx(0.5 * p.rho * vol * float(s @ s), rel=1e-12)
    assert e["strain"] == 0.0 and e["external"] == 0.0 and e["reaction"] == 0.0 and e["dissipated"] == 0.0


@pytest.mark.parametrize("mode", ["uniaxial", "shear"])
def test_strain_energy_uniform_field(mode):
    """Affine u = G X: every smoothing domain carries the exact strain, U = psi * volume with
    psi = 1/2 (lam + 2 mu) eps^2 (uniaxial strain) or 1/2 mu gamma^2 (simple shear)."""
    X, T, _, vol = _block()
    p = ci.make_problem(X, T, E=30e9, nu=0.25, tet_gc=np.full(T.shape[0], np.inf))
    o = oracle.Oracle(p)
    lam, mu = o.lame()
    u = np.zeros_like(X)
    g = 1e-4
    if mode == "uniaxial":
        u[:, 0] = g * X[:, 0]
        psi = 0.5 * (lam + 2 * mu) * g * g
    else:
        u[:, 0] = g * X[:, 1]
        psi = 0.5 * mu * g * g
    o.set_state(u=u, v=np.zeros_like(X), a=np.zeros_like(X))
    assert o.energy()["strain"] == pytest.approx(psi * vol, rel=1e-9)


def test_external_work_rigid_translation():
    """One loaded face (traction t on y = 0): W = d . (t * area) for a rigid translation d."""
    cells, dims = (5, 3, 2), (0.05, 0.03, 0.02)
    X, T, ijk = ci.kuhn_lattice(cells, dims, 4)
    state = np.ones(T.shape[0], np.uint8)
    t = np.array([0.0, -2e6, 5e5])
    faces, tr, _ = ci._loaded_faces(T, state, ijk, 1, 0, tuple(t))
    p = ci.make_problem(X, T, tet_gc=np.full(T.shape[0], np.inf), tface=faces, tface_t=tr)
    o = oracle.Oracle(p)
    d = np.array([1e-5, 2e-5, -3e-5])
    o.set_state(u=np.tile(d, (X.shape[0], 1)), v=np.zeros_like(X), a=np.zeros_like(X))
    area = dims[0] * dims[2]
    assert o.energy()["external"] == pytest.approx(float(d @ t) * area, rel=1e-12)


def test_reaction_work_equals_kinetic_energy_in_a_rigid_ramp():
    """Every node driven in x by the ramp v = (t/t0) v0, no loads: the body stays unstrained,
    the support force is m a, and the trapezoidal work over the ramp equals 1/2 M v(t)^2."""
    X, T, _, vol = _block(cells=(3, 2, 2), dims=(0.03, 0.02, 0.02))
    n = X.shape[0]
    v0 = 5.0
    vbc = (np.arange(n, dtype=np.int32), np.full(n, 1, np.uint8), np.tile([v0, 0.0, 0.0], (n, 1)), 0.0)
    p0 = ci.make_problem(X, T, tet_gc=np.full(T.shape[0], np.inf), vbc=vbc)
    dt = oracle.Oracle(p0).dt
    t0 = 40 * dt
    vbc = (vbc[0], vbc[1], vbc[2], t0)
    p = ci.make_problem(X, T, tet_gc=np.full(T.shape[0], np.inf), vbc=vbc)
    o = oracle.Oracle(p)
    o.run(25, 0)
    e = o.energy()
    vt = 25 * o.dt / t0 * v0
    M = p.rho * vol
    assert e["kinetic"] == pytest.approx(0.5 * M * vt * vt, rel=1e-9)
    assert e["reaction"] == pytest.approx(e["kinetic"], rel=1e-9)


def test_energy_balance_with_prescribed_velocity():
    """Edge-impact stand-in without fracture, velocity ramp over ~40 steps: T + U = W_ext + W_R
    along the run to 1e-4 of the peak input work (discrete balance of the central-difference
    scheme; a ramp that ends between two steps leaves an O(dt) offset at the jump of the
    prescribed acceleration, hence the smooth ramp here)."""
    p = ci.edge_impact_plate(cells=(12, 8, 2), dims=(0.024, 0.016, 0.004), t0=4e-6).with_gc(np.inf)
    o = oracle.Oracle(p)
    hist = []
    for _ in range(30):
        o.run(20, 0)
        e = o.energy()
        hist.append((e["kinetic"], e["strain"], e["external"], e["reaction"]))
    h = np.array(hist)
    peak = np.abs(h[:, 3]).max()
    assert peak > 0
    assert np.abs(h[:, 0] + h[:, 1] - h[:, 2] - h[:, 3]).max() <= 2e-4 * peak


def test_energy_balance_with_traction():
    """Notched plate under constant traction, no fracture: T + U = W_ext (W_R = 0)."""
    p = ci.notched_plate(cells=(10, 4, 2), dims=(0.05, 0.02, 0.005), seed=5, steps=0).with_gc(np.inf)
    o = oracle.Oracle(p)
    hist = []
    for _ in range(20):
        o.run(50, 0)
        e = o.energy()
        assert e["reaction"] == 0.0
        hist.append((e["kinetic"], e["strain"], e["external"]))
    h = np.array(hist)
    assert np.abs(h[:, 0] + h[:, 1] - h[:, 2]).max() <= 1e-3 * np.abs(h[:, 2]).max()


def test_dissipated_matches_records():
    """U_d of the ledger = sum Gc_e A_e over the split records."""
    p = ci.config(0)
    o = oracle.Oracle(p)
    o.run(120, 1)
    r = o.records()
    assert r.elem.size > 0
    ud = 0.0
    for e, a in zip(r.elem, r.area):
        ud = ud + p.tet_gc[e] * a
    assert o.energy()["dissipated"] == pytest.approx(ud, rel=1e-12)
