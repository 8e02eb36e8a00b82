"""Oracle pins for ES-FEM strain, stress, internal force, mass and external force.

P2 patch test (u = A X -> eps~_s = Voigt(sym A) on every edge);
   rigid translation / infinitesimal rotation -> zero strain.
P3 interior forces vanish for linear fields; sum_k f_k = 0; reciprocity w.f(u) = u.f(w);
   energy identity u.f(u) = 2U; central finite differences dU/du = f;
   single tet = standard FEM B^T sigma V.
P4 factored oracle == literal assembled-B̃ form (oracle/l0_literal.py) to 1e-13 relative,
   including meshes with inactive tets.
P5 mass: sum m = rho * active volume, single tet rho V/4;
   traction: unit-area triangle with t = (0,3,0) -> (0,1,0) per node.
"""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from oracle import l0_literal as L0


def voigt_sym(A):
    return np.array([A[0, 0], A[1, 1], A[2, 2], A[0, 1] + A[1, 0], A[1, 2] + A[2, 1], A[0, 2] + A[2, 0]])


def stress_of(eps, E, nu):
    return L0.D_matrix(E, nu) @ eps


@pytest.fixture(scope="module")
def small():
    p = ci.notched_plate(cells=(6, 4, 2), dims=(0.03, 0.02, 0.01), seed=11, steps=0)
    return p, oracle.Oracle(p)


def test_patch_test(small):
    p, o = small
    rng = np.random.default_rng(0)
    A = rng.standard_normal((3, 3)) * 1e-4
    u = p.X @ A.T
    sig, vh = o.edge_stress(u)
    en, _ = o.edges()
    live = vh > 0
    target = stress_of(voigt_sym(A), p.E, p.nu)
    err = np.abs(sig[live] - target[None, :]).max() / np.abs(target).max()
    assert err < 1e-10
    assert np.all(sig[~live] == 0)
    # rigid translation + infinitesimal rotation: zero strain
    W = np.array([[0, -1, 2], [1, 0, -3], [-2, 3, 0]]) * 1e-5
    u = p.X @ W.T + np.array([1e-3, -2e-3, 5e-4])
    sig, _ = o.edge_stress(u)
    assert np.abs(sig).max() < 1e-9 * np.abs(target).max()


def test_linear_field_interior_force_zero(small):
    p, o = small
    rng = np.random.default_rng(1)
    A = rng.standard_normal((3, 3)) * 1e-4
    f = o.internal_force(p.X @ A.T)
    cells = np.array(p.cells)
    interior = np.all((p.node_ijk > 0) & (p.node_ijk < cells[None, :]), axis=1)
    # nodes touching the notch see a free surface: exclude nodes of inactive tets
    near_notch = np.zeros(p.n_nodes, bool)
    near_notch[p.tets[p.tet_state == 0].ravel()] = True
    sel = interior & ~near_notch
    assert sel.sum() >= 5
    scale = np.abs(f).max()
    assert np.abs(f[sel]).max() < 1e-12 * scale


def test_force_sum_zero_reciprocity_energy(small):
    p, o = small
    rng = np.random.default_rng(2)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-6
    w = rng.standard_normal((p.n_nodes, 3)) * 1e-6
    fu = o.internal_force(u); fw = o.internal_force(w)
    scale = np.abs(fu).max()
    assert np.abs(fu.sum(axis=0)).max() < 1e-12 * scale * p.n_nodes
    assert np.vdot(w, fu) == pytest.approx(np.vdot(u, fw), rel=1e-12)
    U = o.strain_energy(u)
    assert np.vdot(u, fu) == pytest.approx(2 * U, rel=1e-12)
    # rigid rotation -> f = 0
    Wk = np.array([[0, -1, 2], [1, 0, -3], [-2, 3, 0]]) * 1e-6
    assert np.abs(o.internal_force(p.X @ Wk.T)).max() < 1e-9 * scale


def test_finite_difference_gradient(small):
    p, o = small
    rng = np.random.default_rng(3)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-6
    f = o.internal_force(u)
    h = 1e-9
    for _ in range(20):
        k = rng.integers(p.n_nodes); c = rng.integers(3)
        up = u.copy(); up[k, c] += h
        um = u.copy(); um[k, c] -= h
        fd = (o.strain_energy(up) - o.strain_energy(um)) / (2 * h)
        assert fd == pytest.approx(f[k, c], rel=1e-5, abs=1e-5 * np.abs(f).max())


def test_single_tet_equals_standard_fem():
    X, T = ci.single_tet(0.01)
    X = X + np.random.default_rng(4).standard_normal(X.shape) * 1e-3
    p = ci.make_problem(X, T)
    o = oracle.Oracle(p)
    u = np.random.default_rng(5).standard_normal((4, 3)) * 1e-6
    V, B = L0.tet_B(X)
    D = L0.D_matrix(p.E, p.nu)
    fstd = (B.T @ D @ B @ u.ravel() * V).reshape(4, 3)
    assert np.allclose(o.internal_force(u), fstd, rtol=0, atol=1e-13 * np.abs(fstd).max())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_factored_equals_literal(seed):
    rng = np.random.default_rng(seed)
    X, T, ijk = ci.random_tet_mesh(seed, n_cells=(3, 2, 2), jitter=0.2)
    st = (rng.random(T.shape[0]) > 0.25).astype(np.uint8)
    p = ci.make_problem(X, T, tet_state=st)
    o = oracle.Oracle(p)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-5
    f1 = o.internal_force(u)
    f0 = L0.internal_force(p.X, p.tets, st, u, p.E, p.nu)
    assert np.abs(f1 - f0).max() <= 1e-13 * np.abs(f0).max()
    # edge stresses: same edge order (sorted (min,max) pairs)
    sig1, vh = o.edge_stress(u)
    en, _ = o.edges()
    ref = L0.edge_strain_stress(p.X, p.tets, st, u, p.E, p.nu)
    sig0 = np.array([ref[(int(a), int(b))][1] for a, b in en])
    assert np.abs(sig1 - sig0).max() <= 1e-12 * np.abs(sig0).max()
    assert o.strain_energy(u) == pytest.approx(L0.strain_energy(p.X, p.tets, st, u, p.E, p.nu), rel=1e-12)


def test_mass_lumping(small):
    p, o = small
    m = o.state()["m"]
    V, _ = o.geometry()
    assert m.sum() == pytest.approx(p.rho * V[p.tet_state == 1].sum(), rel=1e-12)
    X, T = ci.single_tet(2.0)
    q = ci.make_problem(X, T, rho=3.0)
    mq = oracle.Oracle(q).state()["m"]
    assert np.allclose(mq, 3.0 * (8 / 6) / 4, rtol=1e-15)


def test_traction_unit_triangle():
    X = np.array([[0, 0, 0], [np.sqrt(2), 0, 0], [0, np.sqrt(2), 0], [0, 0, 1.0]])
    T = np.array([[0, 1, 2, 3]], np.int32)
    p = ci.make_problem(X, T, tface=[[0, 1, 2]], tface_t=[[0.0, 3.0, 0.0]])
    f = oracle.Oracle(p).fext()
    assert np.allclose(f[:3], [[0, 1, 0]] * 3, rtol=1e-14)
    assert np.all(f[3] == 0)


def test_traction_total_force_cfg0(cfg0):
    o = oracle.Oracle(cfg0)
    f = o.fext()
    Lx, Ly, Lz = cfg0.dims
    # equal and opposite resultants of magnitude t * Lx * Lz
    top = cfg0.node_ijk[:, 1] == cfg0.cells[1]
    assert f[top, 1].sum() == pytest.approx(1e6 * Lx * Lz, rel=1e-12)
    assert f.sum(axis=0) == pytest.approx(np.zeros(3), abs=1e-9)
