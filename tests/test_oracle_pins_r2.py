"""Oracle pins for the parts the round-1 review found unpinned, and for the load/criterion
options added in round 2.  Each test checks the oracle against something other than itself
(closed forms, numpy / LAPACK, the literal assembled-B form in oracle/l0_literal.py) and is
chosen so that a plausible mistake fails it:

- time step R12 (BASELINE.json "dt=0.5xCFL"; SURVEY.md §8(c) Init 5): closed-form altitudes of
  a right and a regular tet (fails for 2V/A, min edge, min face), inactive tets ignored, and
  dt below the ES-FEM stability limit 2/omega_max of the literal stiffness with a numpy lumped
  mass;
- lumped mass after splits (PAPER.md:L392-L407 with L151 "excluded from subsequent
  computations", R2/R15): every node's mass equals a numpy sum over its active tets after a
  cracking run (fails if the split pass does not recompute it);
- sigma_G . n for a degenerate top eigenspace (R8): closed form
  s ||P m|| for sigma = R diag(s, s, t) R^T (fails without the square root or with the
  single-eigenvector rule);
- external force with a body force and nodal point forces: resultants and
  the single-tet consistent lumping b V/4;
- the Q11 / R11 criterion variant ("whose tensile stretches at two edges"):
  candidates whose front is not stretched at both edges are zero, the others unchanged;
  stretch flags computed independently with the square-root length ratio of eq:stretch-delta.
"""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from oracle import l0_literal as L0


def _cd(E, nu, rho):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return np.sqrt((lam + 2 * mu) / rho)


# ------------------------------------------------------------------ time step (R12)
def test_dt_right_tet_closed_form():
    """Unit right tet scaled by L: V = L^3/6, largest face the slanted one (sqrt(3)/2 L^2),
    altitude 3V/A_max = L/sqrt(3); dt = 0.5 * L/sqrt(3) / c_d."""
    L = 0.004
    X, T = ci.single_tet(L)
    p = ci.make_problem(X, T)
    dt = oracle.Oracle(p).dt
    want = 0.5 * (L / np.sqrt(3.0)) / _cd(p.E, p.nu, p.rho)
    assert dt == pytest.approx(want, rel=1e-14)
    # plausible mistakes: 2V/A_max, min edge, min face area
    assert abs(dt - 0.5 * (2 * L / (3 * np.sqrt(3))) / _cd(p.E, p.nu, p.rho)) > 1e-3 * want
    assert abs(dt - 0.5 * L / _cd(p.E, p.nu, p.rho)) > 1e-3 * want


def test_dt_regular_tet_closed_form():
    """Regular tet of edge a: V = a^3/(6 sqrt 2), face sqrt(3)/4 a^2, altitude a sqrt(2/3)."""
    s = 0.002
    X = s * np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=np.float64)
    T = np.array([[0, 1, 2, 3]], np.int32)
    if np.linalg.det(X[1:] - X[0]) < 0:
        T = T[:, [0, 1, 3, 2]]
    a = np.linalg.norm(X[1] - X[0])
    p = ci.make_problem(X, T, E=190e9, nu=0.3, rho=8000.0)
    dt = oracle.Oracle(p).dt
    assert dt == pytest.approx(0.5 * a * np.sqrt(2.0 / 3.0) / _cd(190e9, 0.3, 8000.0), rel=1e-14)


def test_dt_ignores_inactive_tets():
    """A flattened inactive tet does not set the step: dt comes from the active one only."""
    L = 0.01
    X = np.array([[0, 0, 0], [L, 0, 0], [0, L, 0], [0, 0, L], [0.5 * L, 0.5 * L, 0.02 * L]], dtype=np.float64)  # 4 just off face 123
    T = np.array([[0, 1, 2, 3], [1, 4, 2, 3]], np.int32)
    for e in range(2):
        if np.linalg.det(X[T[e, 1:]] - X[T[e, 0]]) < 0:
            T[e, [2, 3]] = T[e, [3, 2]]
    full = oracle.Oracle(ci.make_problem(X, T)).dt
    only0 = oracle.Oracle(ci.make_problem(X, T, tet_state=[1, 0])).dt
    assert only0 == pytest.approx(0.5 * (L / np.sqrt(3.0)) / _cd(32e9, 0.2, 2450.0), rel=1e-14)
    assert full < 0.5 * only0   # the flat tet's altitude is much smaller


def test_dt_below_stability_limit():
    """P7: central differences are stable for dt < 2/omega_max.  omega_max from the literal
    ES-FEM stiffness (l0_literal.stiffness) and a numpy lumped mass, dense eigen-solve."""
    X, T, _ = ci.kuhn_lattice((3, 3, 2), (0.03, 0.03, 0.02), seed=7, jitter=0.05)
    p = ci.make_problem(X, T)
    act = np.ones(len(T), bool)
    K = L0.stiffness(X, T, act, p.E, p.nu)
    V = np.array([np.linalg.det(X[t[1:]] - X[t[0]]) / 6.0 for t in T])
    m = np.zeros(len(X))
    for e, t in enumerate(T):
        m[t] += p.rho * V[e] / 4.0
    minv = 1.0 / np.sqrt(np.repeat(m, 3))
    w2 = np.linalg.eigvalsh(minv[:, None] * K * minv[None, :]).max()
    dt_crit = 2.0 / np.sqrt(w2)
    o = oracle.Oracle(p)
    assert o.dt < dt_crit
    # the altitude rule at cfl = 1 is itself below the ES-FEM limit
    assert 2.0 * o.dt < dt_crit
    assert 0.3 * dt_crit < o.dt     # and not absurdly small (0.5 x CFL ~ 0.38-0.43 of critical)


# ------------------------------------------------------------------ mass after splits
def test_mass_after_splits_matches_active_volume(cfg0):
    o = oracle.Oracle(cfg0)
    m0 = o.state()["m"].copy()
    o.run(200, 1)
    s = o.state()
    assert len(o.records().elem) > 0
    X, T = cfg0.X, cfg0.tets
    V = np.array([np.linalg.det(X[t[1:]] - X[t[0]]) / 6.0 for t in T])
    act = s["state"] == 1
    want = np.zeros(len(X))
    for e in np.flatnonzero(act):
        want[T[e]] += cfg0.rho * V[e] / 4.0
    assert np.allclose(s["m"], want, rtol=1e-13, atol=0.0)
    assert s["m"].sum() == pytest.approx(cfg0.rho * V[act].sum(), rel=1e-12)
    changed = np.flatnonzero(s["m"] != m0)
    assert changed.size > 0                       # the splits changed some masses (non-vacuous)
    touched = np.unique(T[o.records().elem].ravel())
    assert set(changed.tolist()) <= set(touched.tolist())
    has_active = np.zeros(len(X), bool)
    has_active[T[act].ravel()] = True
    assert np.array_equal(s["m"] == 0.0, ~has_active)


# ------------------------------------------------------------------ sigma_G . n (R8)
def _rot(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(3, 3)))
    return q * np.sign(np.linalg.det(q))


def _s6(A):
    return np.array([A[0, 0], A[1, 1], A[2, 2], A[0, 1], A[1, 2], A[0, 2]])


@pytest.mark.parametrize("seed", range(6))
def test_sig_proj_degenerate_top_closed_form(seed):
    rng = np.random.default_rng(100 + seed)
    R = _rot(seed)
    s, t = 2.5e6, -0.7e6
    sig = R @ np.diag([s, s, t]) @ R.T
    m = rng.normal(size=3) * 1e-5
    r3 = R[:, 2]
    want = s * np.linalg.norm(m - (m @ r3) * r3)           # s ||projection of m on the top plane||
    got = oracle.sig_proj(_s6(sig), m)
    assert got == pytest.approx(want, rel=1e-10)
    assert abs(got - s * np.linalg.norm(m - (m @ r3) * r3) ** 2) > 1e-6 * want   # sqrt dropped


def test_sig_proj_nondegenerate_and_hydrostatic():
    R = _rot(11)
    m = np.array([0.3, -0.2, 0.7])
    sig = R @ np.diag([1.0e6, 3.0e6, 2.0e6]) @ R.T
    assert oracle.sig_proj(_s6(sig), m) == pytest.approx(3.0e6 * abs(m @ R[:, 1]), rel=1e-10)
    assert oracle.sig_proj(_s6(4e5 * np.eye(3)), m) == pytest.approx(4e5 * np.linalg.norm(m), rel=1e-14)
    # top eigenvalue t > s: not degenerate, single eigenvector rule
    sig = R @ np.diag([1.0e6, 1.0e6, 2.0e6]) @ R.T
    assert oracle.sig_proj(_s6(sig), m) == pytest.approx(2.0e6 * abs(m @ R[:, 2]), rel=1e-10)
    # within the 1e-10 relative degeneracy band -> projector norm over both
    sig = np.diag([1.0e6, 1.0e6 * (1 - 1e-13), -3e5])
    assert oracle.sig_proj(_s6(sig), m) == pytest.approx(1.0e6 * np.hypot(m[0], m[1]), rel=1e-12)


# ------------------------------------------------------------------ body force, nodal forces
def test_body_force_single_tet_consistent_lumping():
    X, T = ci.single_tet(0.01)
    p = ci.make_problem(X, T)
    p.body = (0.0, -9.81 * p.rho, 2.0)
    f = oracle.Oracle(p).fext()
    V = 0.01 ** 3 / 6
    assert np.allclose(f, np.tile(np.array(p.body) * V / 4, (4, 1)), rtol=1e-14, atol=0)


def test_external_force_resultant_body_traction_nodal(cfg0):
    p = ci.config(0)
    rng = np.random.default_rng(4)
    p.body = (1.5e3, -2.4e4, 7.0e2)
    p.f_nodal = rng.normal(size=(p.n_nodes, 3)) * 10.0
    f = oracle.Oracle(p).fext()
    f_tr = oracle.Oracle(cfg0).fext()
    X, T = p.X, p.tets
    V = np.array([np.linalg.det(X[t[1:]] - X[t[0]]) / 6.0 for t in T])
    Vact = V[p.tet_state == 1].sum()
    want = np.array(p.body) * Vact + f_tr.sum(axis=0) + p.f_nodal.sum(axis=0)
    assert np.allclose(f.sum(axis=0), want, rtol=1e-9, atol=1e-12)
    # nodes touching no active tet get no body force; a node with only inactive tets
    body_only = f - f_tr - p.f_nodal
    w = np.zeros(len(X))
    for e in np.flatnonzero(p.tet_state == 1):
        w[T[e]] += V[e] / 4
    assert np.allclose(body_only, w[:, None] * np.array(p.body)[None, :], rtol=1e-9, atol=1e-12)


# ------------------------------------------------------------------ Q11 / R11 variant
def _stretched(X, u, a, b):
    """eq:stretch-delta's Heaviside with the square-root length ratio (H(0) = 0)."""
    return np.linalg.norm((X[b] + u[b]) - (X[a] + u[a])) / np.linalg.norm(X[b] - X[a]) > 1.0


@pytest.mark.parametrize("seed", range(4))
def test_front_both_stretched_variant(seed):
    X, T, _ = ci.random_tet_mesh(seed)
    p = ci.make_problem(X, T)
    rng = np.random.default_rng(seed)
    u = rng.normal(size=X.shape) * 1e-4
    o0 = oracle.Oracle(p)
    o1 = oracle.Oracle(p, flags=oracle.Oracle.FRONT_BOTH_STRETCHED)
    checked = zeroed = 0
    for e in range(0, len(T), 3):
        G0, A0 = o0.candidates(u, e)
        G1, A1 = o1.candidates(u, e)
        assert np.array_equal(A0, A1)
        t = T[e]
        for c in range(4):
            o = [b for b in range(4) if b != c]
            for f, (ip, iq) in enumerate([(0, 1), (0, 2), (1, 2)]):
                p_, q_ = o[ip], o[iq]
                both = _stretched(X, u, t[c], t[p_]) and _stretched(X, u, t[c], t[q_])
                for tt in range(2):
                    k = 6 * c + 2 * f + tt
                    checked += 1
                    if both:
                        assert G1[k] == G0[k]
                    else:
                        assert G1[k] == 0.0
                        zeroed += G0[k] != 0.0
    assert checked > 0 and zeroed > 0
