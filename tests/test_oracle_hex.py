"""Pins of the ES-H-FEM hexahedral oracle (oracle/cem_oracle_hex.c; SURVEY.md §8(f) N3;
PAPER.md:L311-L338 eq:hex_strain_discretization, L368-L390 eq:hex_fint_discretization;
readings R23-R26 in DESIGN.md) against closed forms, invariants, numpy and the literal
assembled-B̃ form (oracle/l0_literal.py hex_B with its own quadrature and matrix inverse).
A plausible mistake anywhere -- a wrong shape-function sign or node order, the Jacobian
transposed, 1/6 instead of 1/12, V/4 instead of V/8, a missing weight -- fails one of them."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from oracle import l0_literal as L0

XI = L0.HEX_XI


def _cube(h=1.0, x0=(0.0, 0.0, 0.0)):
    return np.asarray(x0) + (XI + 1.0) / 2.0 * h


def test_unit_cube_geometry():
    V, g = oracle.hex_geometry(_cube())
    assert V == pytest.approx(1.0, rel=1e-15)
    assert np.allclose(g, XI / 4.0, rtol=0, atol=1e-16)   # dN_i/dx at the centre = xi_i / 4


@pytest.mark.parametrize("seed", range(5))
def test_parallelepiped_closed_form(seed):
    rng = np.random.default_rng(seed)
    A = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
    if np.linalg.det(A) < 0:
        A[:, 0] *= -1
    x0 = rng.normal(size=3)
    X8 = x0 + ((XI + 1.0) / 2.0) @ A.T                    # x = x0 + A (xi + 1) / 2
    V, g = oracle.hex_geometry(X8)
    assert V == pytest.approx(np.linalg.det(A), rel=1e-13)
    assert np.allclose(g, (XI / 4.0) @ np.linalg.inv(A), rtol=0, atol=1e-13 * np.abs(g).max())


@pytest.mark.parametrize("seed", range(8))
def test_distorted_hex_vs_numpy(seed):
    rng = np.random.default_rng(10 + seed)
    X8 = _cube(0.01) + rng.uniform(-0.002, 0.002, size=(8, 3))
    V, g = oracle.hex_geometry(X8)
    Vn, B = L0.hex_B(X8)
    assert V == pytest.approx(Vn, rel=1e-13)               # 2x2x2 (oracle) == 3x3x3 (numpy): both exact
    gn = np.stack([B[0, 0::3], B[1, 1::3], B[2, 2::3]], axis=1)
    assert np.allclose(g, gn, rtol=0, atol=1e-12 * np.abs(gn).max())
    assert np.allclose(X8.T @ g, np.eye(3), atol=1e-12)    # linear fields reproduced by the mean gradients
    assert np.allclose(g.sum(axis=0), 0.0, atol=1e-10)


def test_inverted_hex_rejected():
    X8 = _cube()[[1, 0, 3, 2, 5, 4, 7, 6]]                 # mirrored node order: negative Jacobian
    assert oracle.hex_geometry(X8) is None
    p = ci.hex_block((2, 2, 1))
    p.tets = p.tets[:, [1, 0, 3, 2, 5, 4, 7, 6]].copy()
    with pytest.raises(ValueError):
        oracle.HexOracle(p)


@pytest.fixture(scope="module")
def block():
    p = ci.hex_block((4, 3, 3), dims=(0.04, 0.03, 0.03), seed=5, jitter=0.12)
    return p, oracle.HexOracle(p)


def _voigt_sym(A):
    S = 0.5 * (A + A.T)
    return np.array([S[0, 0], S[1, 1], S[2, 2], 2 * S[0, 1], 2 * S[1, 2], 2 * S[0, 2]])


def test_patch_test(block):
    p, o = block
    rng = np.random.default_rng(1)
    A = rng.normal(size=(3, 3)) * 1e-4
    u = p.X @ A.T
    sig, vh, _ = o.edge_stress(u)
    want = L0.D_matrix(p.E, p.nu) @ _voigt_sym(A)
    assert np.abs(sig - want[None, :]).max() <= 1e-10 * np.abs(want).max()
    assert np.all(vh > 0)


def test_linear_field_forces_and_invariants(block):
    p, o = block
    rng = np.random.default_rng(2)
    A = rng.normal(size=(3, 3)) * 1e-4
    f = o.internal_force(p.X @ A.T)
    ijk = p.node_ijk
    interior = np.all((ijk > 0) & (ijk < np.array(p.cells)[None, :]), axis=1)
    assert interior.any()
    assert np.abs(f[interior]).max() <= 1e-9 * np.abs(f).max()
    u = rng.normal(size=p.X.shape) * 1e-6
    w = rng.normal(size=p.X.shape) * 1e-6
    fu, fw = o.internal_force(u), o.internal_force(w)
    assert np.abs(fu.sum(axis=0)).max() <= 1e-12 * np.abs(fu).max()           # sum of forces 0
    assert (w * fu).sum() == pytest.approx((u * fw).sum(), rel=1e-11)           # reciprocity
    assert (u * fu).sum() == pytest.approx(2 * o.strain_energy(u), rel=1e-11)   # u.f = 2U


@pytest.mark.parametrize("seed", range(3))
def test_factored_equals_literal(seed):
    p = ci.hex_block((3, 2, 2), dims=(0.03, 0.02, 0.02), seed=20 + seed, jitter=0.15)
    rng = np.random.default_rng(seed)
    p.tet_state = (rng.uniform(size=p.n_tets) > 0.2).astype(np.uint8)
    o = oracle.HexOracle(p)
    u = rng.normal(size=p.X.shape) * 1e-5
    f = o.internal_force(u)
    fl = L0.internal_force(p.X, p.tets, p.tet_state.astype(bool), u, p.E, p.nu)
    assert np.abs(f - fl).max() <= 1e-13 * np.abs(fl).max()
    assert o.strain_energy(u) == pytest.approx(L0.strain_energy(p.X, p.tets, p.tet_state.astype(bool), u, p.E, p.nu),
                                               rel=1e-12)


def test_mass_and_timestep_closed_forms():
    h = (0.004, 0.003, 0.005)
    p = ci.hex_block((3, 2, 2), dims=(3 * h[0], 2 * h[1], 2 * h[2]), jitter=0.0)
    o = oracle.HexOracle(p)
    m = o.state()["m"]
    Vc = h[0] * h[1] * h[2]
    assert m.sum() == pytest.approx(p.rho * Vc * p.n_tets, rel=1e-13)
    corner = np.flatnonzero((p.node_ijk == 0).all(axis=1))[0]
    assert m[corner] == pytest.approx(p.rho * Vc / 8.0, rel=1e-14)              # R24: rho V / 8
    lam = p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)); mu = p.E / (2 * (1 + p.nu))
    cd = np.sqrt((lam + 2 * mu) / p.rho)
    assert o.dt == pytest.approx(0.5 * min(h) / cd, rel=1e-13)                  # R25: V / A_max = min h


def test_traction_and_body_force_resultants():
    p = ci.hex_block((4, 2, 2), dims=(0.04, 0.02, 0.02), jitter=0.1)
    p.body = (0.0, 0.0, -2.0e4)
    o = oracle.HexOracle(p)
    f = o.fext()
    V, _ = o.geometry()
    top = p.node_ijk[:, 1] == p.cells[1]
    assert f[top, 1].sum() == pytest.approx(1e6 * 0.04 * 0.02, rel=1e-12)
    assert f[:, 2].sum() == pytest.approx(-2.0e4 * V.sum(), rel=1e-12)


def _energy_error(p, dt, t_end, checks=15):
    o = oracle.HexOracle(p, dt=dt)
    f = o.fext()
    n = int(round(t_end / dt)) // checks
    worst, peak = 0.0, 0.0
    for _ in range(checks):
        o.run(n)
        s = o.state()
        T = 0.5 * (s["m"][:, None] * s["v"] ** 2).sum()
        U = o.strain_energy(s["u"])
        W = (f * s["u"]).sum()
        worst = max(worst, abs(T + U - W))
        peak = max(peak, abs(W))
    return worst, peak


def test_energy_balance_no_fracture():
    """Central differences conserve T + U - W only to O(dt^2): the balance error is small and
    falls about fourfold when dt is halved (the traction is constant from t = 0, u_0 = 0)."""
    p = ci.hex_block((6, 4, 2), dims=(0.06, 0.04, 0.02), seed=3)
    dt0 = oracle.HexOracle(p).dt
    e1, peak = _energy_error(p, dt0, 1500 * dt0)
    e2, _ = _energy_error(p, dt0 / 2, 1500 * dt0)
    assert peak > 0
    assert e1 <= 5e-3 * peak
    assert e2 <= e1 / 3.0
