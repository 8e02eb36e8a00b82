"""Oracle pins: tet geometry, Lamé constants, principal stress, crack-plane geometry.

P1  unit tet gradients / volume, partition of unity, linear reproduction.
P8  principal stress: diagonal, degenerate, random vs numpy.linalg.eigh, frame invariance.
P10 Appendix I coplanarity and the closed-form crack-plane normals.
Material: Lamé values and Rayleigh speeds printed in the paper
(tests/golden/paper_values.txt: PAPER.md:L571 2803 m/s, L984 1237.5 m/s).
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_unit_tet():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    V, g = oracle.tet_geometry(X)
    assert V == pytest.approx(1 / 6, rel=1e-15)
    assert np.array_equal(g, np.array([[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float))
    V2, g2 = oracle.tet_geometry(2 * X)
    assert V2 == pytest.approx(8 / 6, rel=1e-15)
    assert np.allclose(g2, g / 2, rtol=0, atol=1e-16)


def test_random_tets_linear_reproduction():
    rng = np.random.default_rng(1)
    for _ in range(200):
        X = rng.standard_normal((4, 3))
        d = np.linalg.det(np.hstack([np.ones((4, 1)), X]))
        if d < 0:
            X[[2, 3]] = X[[3, 2]]
        V, g = oracle.tet_geometry(X)
        # volume vs numpy determinant
        assert V == pytest.approx(abs(d) / 6, rel=1e-12)
        # sum of gradients = 0; grad N_a . (X_b - X_0) = delta_ab - delta_a0
        assert np.abs(g.sum(axis=0)).max() < 1e-12 * np.abs(g).max()
        M = np.array([[g[a] @ (X[b] - X[0]) for b in range(4)] for a in range(4)])
        target = np.eye(4); target[0, :] -= 1; target[:, 0] = 0
        target[0, 0] = 0
        assert np.allclose(M, target, atol=1e-11)


def test_lame():
    lam, mu = oracle.lame(190e9, 0.3)
    assert lam == pytest.approx(1.09615e11, rel=1e-5) and mu == pytest.approx(7.30769e10, rel=1e-5)
    lam, mu = oracle.lame(1.0, 0.0)
    assert lam == 0.0 and mu == 0.5
    lam, mu = oracle.lame(5.76e9, 0.42)
    assert mu == pytest.approx(2.0282e9, rel=1e-4)


def _golden_values():
    vals = {}
    with open(os.path.join(GOLDEN, "paper_values.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                k, v = line.split("=")
                vals[k.strip()] = float(v)
    return vals


def test_rayleigh_speed_matches_paper():
    """v_R = c_s (0.862 + 1.14 nu)/(1+nu) from the oracle's Lamé mu vs the paper's printed values."""
    g = _golden_values()
    for E, nu, rho, key in [(190e9, 0.3, 8000.0, "kalthoff_vR"), (5.76e9, 0.42, 1180.0, "pmma_vR")]:
        lam, mu = oracle.lame(E, nu)
        cs = np.sqrt(mu / rho)
        vR = cs * (0.862 + 1.14 * nu) / (1 + nu)
        assert vR == pytest.approx(g[key], rel=0.01)


# ------------------------------------------------------------------ principal stress (P8)
def test_principal_diagonal():
    lam, vec, k1, deg = oracle.principal([3, 1, 2, 0, 0, 0])
    assert lam[k1] == 3.0 and deg == 1 << k1
    assert np.array_equal(np.abs(vec[:, k1]), [1, 0, 0])


def test_principal_hydrostatic_degenerate():
    lam, vec, k1, deg = oracle.principal([5, 5, 5, 0, 0, 0])
    assert lam[k1] == 5.0 and deg == 7


def test_principal_zero():
    lam, vec, k1, deg = oracle.principal([0, 0, 0, 0, 0, 0])
    assert np.all(lam == 0) and deg == 7


def test_principal_random_vs_eigh():
    rng = np.random.default_rng(2)
    for _ in range(2000):
        s = rng.standard_normal(6) * 10 ** rng.uniform(-3, 8)
        A = np.array([[s[0], s[3], s[5]], [s[3], s[1], s[4]], [s[5], s[4], s[2]]])
        w, Q = np.linalg.eigh(A)
        lam, vec, k1, deg = oracle.principal(s)
        scale = np.abs(w).max()
        assert np.allclose(np.sort(lam), w, rtol=0, atol=1e-13 * scale)
        assert np.allclose(vec.T @ vec, np.eye(3), atol=1e-13)
        # A v = lam v
        assert np.allclose(A @ vec, vec * lam[None, :], atol=1e-12 * scale)
        assert lam[k1] == lam.max()


def test_principal_frame_invariance():
    rng = np.random.default_rng(3)
    for _ in range(200):
        s = rng.standard_normal(6)
        A = np.array([[s[0], s[3], s[5]], [s[3], s[1], s[4]], [s[5], s[4], s[2]]])
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        B = Q @ A @ Q.T
        lam1, v1, k1, _ = oracle.principal(s)
        lam2, v2, k2, _ = oracle.principal([B[0, 0], B[1, 1], B[2, 2], B[0, 1], B[1, 2], B[0, 2]])
        assert lam1[k1] == pytest.approx(lam2[k2], rel=1e-12, abs=1e-14)
        assert abs(abs((Q @ v1[:, k1]) @ v2[:, k2]) - 1) < 1e-9


# ------------------------------------------------------------------ crack-plane geometry (P10)
def _mid(X, a, b):
    return 0.5 * (X[a] + X[b])


def test_appendix_I_coplanarity_random():
    """Appendix I: midpoints of N1N2, N2N3, N1N4, N3N4 are coplanar."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((10000, 4, 3))
    G1 = 0.5 * (X[:, 0] + X[:, 1]); G2 = 0.5 * (X[:, 1] + X[:, 2])
    G3 = 0.5 * (X[:, 0] + X[:, 3]); G4 = 0.5 * (X[:, 2] + X[:, 3])
    mixed = np.einsum("ij,ij->i", G1 - G4, np.cross(G2 - G4, G3 - G4))
    scale = np.abs(X).max(axis=(1, 2)) ** 3
    assert np.all(np.abs(mixed) <= 1e-12 * scale)
    # and a generic 4th point is not coplanar
    mixed2 = np.einsum("ij,ij->i", G1 - X[:, 3], np.cross(G2 - X[:, 3], G3 - X[:, 3]))
    assert np.median(np.abs(mixed2) / scale) > 1e-3


def test_crack_plane_normals_closed_form():
    """Quad normal ∝ (X_q-X_p) x (X_r-X_c), area |.|/4; corner triangle ∥ face pqr, area face/4."""
    rng = np.random.default_rng(5)
    for _ in range(500):
        X = rng.standard_normal((4, 3))
        c, p, q, r = rng.permutation(4)
        quad = [_mid(X, c, p), _mid(X, c, q), _mid(X, q, r), _mid(X, p, r)]
        nq = np.cross(quad[2] - quad[0], quad[3] - quad[1])          # diagonals
        m = np.cross(X[q] - X[p], X[r] - X[c])
        assert np.linalg.norm(np.cross(nq, m)) <= 1e-12 * np.linalg.norm(nq) * np.linalg.norm(m)
        assert 0.5 * np.linalg.norm(nq) == pytest.approx(np.linalg.norm(m) / 4, rel=1e-12)
        tri = [_mid(X, c, p), _mid(X, c, q), _mid(X, c, r)]
        nt = np.cross(tri[1] - tri[0], tri[2] - tri[0])
        m2 = np.cross(X[q] - X[p], X[r] - X[p])
        assert np.linalg.norm(np.cross(nt, m2)) <= 1e-12 * np.linalg.norm(nt) * np.linalg.norm(m2)
        assert 0.5 * np.linalg.norm(nt) == pytest.approx(np.linalg.norm(m2) / 8, rel=1e-12)
