"""Oracle pins for the crack criterion and the split pass.

Independent evaluation: `brute_candidates` below recomputes the 24 candidate energy
release rates of a tet directly from the paper's construction -- crack surfaces through
the actual edge midpoints (Fig. 5 caption L455, Appendix I), unit normals
from an SVD of those midpoints, the stretch of eq:stretch-delta with the square-root
length ratio, principal stresses from numpy.linalg.eigh and
eq:G-I / eq:G-II -- and compares with the oracle, which uses the
closed-form cross-product normals, the cancellation-free Heaviside test and cyclic
Jacobi (R6-R9).  Edge stresses come from the literal assembled form L0.

P9  exact rationals on the scaled unit tet: G_e = (lam+2mu) e^2 L.
P11 threshold brute force (Gc = G (1 +- 1e-6)), monotonicity, irreversibility.
P12 U_d = sum Gc * area over records, non-decreasing; active count non-increasing.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import cem_inputs as ci
import oracle
from oracle import l0_literal as L0

LOCAL_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def plane_normal(pts):
    P = np.asarray(pts) - np.mean(pts, axis=0)
    return np.linalg.svd(P)[2][-1]


def sig_dot_n(s6, n):
    A = np.array([[s6[0], s6[3], s6[5]], [s6[3], s6[1], s6[4]], [s6[5], s6[4], s6[2]]])
    w, Q = np.linalg.eigh(A)
    top = w[-1]
    D = [k for k in range(3) if top - w[k] <= 1e-10 * abs(top)]
    return top * np.sqrt(sum((Q[:, k] @ n) ** 2 for k in D))


def stretch_dot_n(Xa, Xb, ua, ub, n):
    """delta = (u_b - u_a) H(|x_b-x_a|/|X_b-X_a| - 1), projected on n oriented a -> b."""
    ratio = np.linalg.norm((Xb + ub) - (Xa + ua)) / np.linalg.norm(Xb - Xa)
    if not ratio > 1.0:
        return 0.0
    nn = n if (Xb - Xa) @ n > 0 else -n
    return (ub - ua) @ nn


def brute_candidates(X, u, sig_edge):
    """X,u: [4,3] of one tet; sig_edge: dict (p,q)->s6 for local edges p<q."""
    mid = lambda a, b: 0.5 * (X[a] + X[b])
    S = lambda a, b: sig_edge[(min(a, b), max(a, b))]
    G = np.zeros(24); A = np.zeros(24)
    for c in range(4):
        o = [b for b in range(4) if b != c]
        for f, (ip, iq, ir) in enumerate([(0, 1, 2), (0, 2, 1), (1, 2, 0)]):
            p, q, r = o[ip], o[iq], o[ir]
            quad = [mid(c, p), mid(c, q), mid(q, r), mid(p, r)]
            n = plane_normal(quad)
            d1 = stretch_dot_n(X[c], X[p], u[c], u[p], n)
            d2 = stretch_dot_n(X[c], X[q], u[c], u[q], n)
            G[6 * c + 2 * f] = 0.5 * (sig_dot_n(S(p, r), n) * d1 + sig_dot_n(S(q, r), n) * d2)
            A[6 * c + 2 * f] = 0.5 * np.linalg.norm(np.cross(quad[2] - quad[0], quad[3] - quad[1]))
            tri = [mid(c, p), mid(c, q), mid(c, r)]
            n = plane_normal(tri)
            d1 = stretch_dot_n(X[c], X[p], u[c], u[p], n)
            d2 = stretch_dot_n(X[c], X[q], u[c], u[q], n)
            G[6 * c + 2 * f + 1] = 0.5 * sig_dot_n(S(c, r), n) * (d1 + d2)
            A[6 * c + 2 * f + 1] = 0.5 * np.linalg.norm(np.cross(tri[1] - tri[0], tri[2] - tri[0]))
    return G, A


def tet_edge_stresses(p, u, e):
    ref = L0.edge_strain_stress(p.X, p.tets, p.tet_state, u, p.E, p.nu)
    t = p.tets[e]
    out = {}
    for a, b in LOCAL_EDGES:
        i, j = int(t[a]), int(t[b])
        out[(a, b)] = ref[(min(i, j), max(i, j))][1]
    return out


@pytest.mark.parametrize("seed", range(4))
def test_candidates_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    X, T, _ = ci.random_tet_mesh(seed, n_cells=(2, 2, 1), jitter=0.2)
    p = ci.make_problem(X, T)
    o = oracle.Oracle(p)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-4
    for e in range(0, p.n_tets, 3):
        G, A = o.candidates(u, e)
        Gb, Ab = brute_candidates(p.X[p.tets[e]], u[p.tets[e]], tet_edge_stresses(p, u, e))
        scale = np.abs(Gb).max()
        assert scale > 0
        assert np.abs(G - Gb).max() <= 1e-9 * scale
        assert np.allclose(A, Ab, rtol=1e-12)


def test_single_tet_exact_rationals():
    """P9: unit right tet scaled by L = 5 mm, u = e z z^ (e = 1e-4), E = 32 GPa, nu = 0.2."""
    Lf, ef = Fr(1, 200), Fr(1, 10000)
    lam = Fr(32 * 10 ** 9) * Fr(1, 5) / ((1 + Fr(1, 5)) * (1 - Fr(2, 5)))
    mu = Fr(32 * 10 ** 9) / (2 * (1 + Fr(1, 5)))
    s1 = (lam + 2 * mu) * ef                       # sigma_1, e_1 = z^
    Xf = [(0, 0, 0), (Lf, 0, 0), (0, Lf, 0), (0, 0, Lf)]
    uf = [(0, 0, 0), (0, 0, 0), (0, 0, 0), (0, 0, ef * Lf)]
    sub = lambda a, b: tuple(x - y for x, y in zip(a, b))
    dot = lambda a, b: sum(x * y for x, y in zip(a, b))
    cross = lambda a, b: (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])

    def Dd(a, b, m):
        du = sub(uf[b], uf[a]); dX = sub(Xf[b], Xf[a])
        if not dot(du, tuple(2 * x + y for x, y in zip(dX, du))) > 0:
            return Fr(0)
        s = dot(dX, m)
        return dot(du, m) * (1 if s > 0 else (-1 if s < 0 else 0))

    exact = []
    for c in range(4):
        o = [b for b in range(4) if b != c]
        for ip, iq, ir in [(0, 1, 2), (0, 2, 1), (1, 2, 0)]:
            p, q, r = o[ip], o[iq], o[ir]
            m = cross(sub(Xf[q], Xf[p]), sub(Xf[r], Xf[c]))
            S = s1 * abs(m[2])
            exact.append(Fr(1, 2) * (S * Dd(c, p, m) + S * Dd(c, q, m)) / dot(m, m))
            m = cross(sub(Xf[q], Xf[p]), sub(Xf[r], Xf[p]))
            S = s1 * abs(m[2])
            exact.append(Fr(1, 2) * S * (Dd(c, p, m) + Dd(c, q, m)) / dot(m, m))
    assert set(exact) <= {Fr(0), Fr(8, 27), Fr(4, 9), Fr(8, 9), Fr(16, 9)}
    assert max(exact) == (lam + 2 * mu) * ef * ef * Lf == Fr(16, 9)
    X, T = ci.single_tet(0.005)
    prob = ci.make_problem(X, T, Gc=3.0)
    orc = oracle.Oracle(prob)
    u = np.zeros((4, 3)); u[3, 2] = 1e-4 * 0.005
    G, A = orc.candidates(u, 0)
    assert np.allclose(G, [float(x) for x in exact], rtol=1e-12, atol=1e-15)
    Ge, k, area, flag = orc.criterion(u)
    best = max(range(24), key=lambda i: (exact[i], float(A[i]), -i))
    assert k[0] == best == 19 and Ge[0] == pytest.approx(16 / 9, rel=1e-13) and flag[0] == 0
    prob2 = ci.make_problem(X, T, Gc=1.7)                 # 16/9 = 1.777... > 1.7 -> split
    assert oracle.Oracle(prob2).criterion(u)[3][0] == 1


def test_perpendicular_and_homogeneity():
    X, T = ci.single_tet(0.005)
    o = oracle.Oracle(ci.make_problem(X, T))
    u = np.zeros((4, 3)); u[3, 2] = 5e-7
    G1, _ = o.candidates(u, 0)
    G2, _ = o.candidates(3.0 * u, 0)
    # G ~ sigma * delta: quadratic in u (H unchanged by positive scaling here)
    assert np.allclose(G2, 9.0 * G1, rtol=1e-12)
    # pure in-plane shear of the z=0 face opens nothing normal to a z-normal plane
    u2 = np.zeros((4, 3)); u2[1, 1] = 1e-7
    G3, _ = o.candidates(u2, 0)
    assert np.all(np.isfinite(G3))


@pytest.mark.parametrize("seed", [0, 1])
def test_threshold_bruteforce(seed):
    rng = np.random.default_rng(seed + 10)
    p = ci.notched_plate(cells=(3, 2, 1), dims=(0.015, 0.01, 0.005), seed=seed, steps=0)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-7
    Gb = np.zeros(p.n_tets)
    for e in range(p.n_tets):
        if p.tet_state[e]:
            Gb[e] = brute_candidates(p.X[p.tets[e]], u[p.tets[e]], tet_edge_stresses(p, u, e))[0].max()
    act = p.tet_state == 1
    for fac, expect_split in [(1 + 1e-6, False), (1 - 1e-6, True)]:
        gc = np.where(act, np.abs(Gb) * fac, 1.0)
        q = ci.make_problem(p.X, p.tets, tet_state=p.tet_state, tet_gc=gc)
        G, k, A, fl = oracle.Oracle(q).criterion(u)
        want = act & (Gb > 0) if expect_split else np.zeros(p.n_tets, bool)
        assert np.array_equal(fl.astype(bool), want)
        assert np.allclose(G[act], Gb[act], rtol=1e-9, atol=1e-12 * np.abs(Gb).max())


def test_monotone_in_gc():
    rng = np.random.default_rng(7)
    p = ci.notched_plate(cells=(4, 3, 1), dims=(0.02, 0.015, 0.005), seed=3, steps=0)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-7
    prev = None
    for gc in [1e-3, 1e-2, 1e-1, 1.0]:
        fl = oracle.Oracle(p.with_gc(gc)).criterion(u)[3].astype(bool)
        if prev is not None:
            assert not np.any(fl & ~prev)
        prev = fl


def test_run_bookkeeping_and_irreversibility(cfg0):
    o = oracle.Oracle(cfg0)
    act_prev = o.state()["state"].copy()
    ud_prev = 0.0
    for _ in range(8):
        o.run(25, 1)
        st = o.state()["state"]
        assert not np.any(st > act_prev)             # irreversibility
        assert o.dissipated >= ud_prev
        act_prev, ud_prev = st.copy(), o.dissipated
    r = o.records()
    assert len(r.elem) > 0                           # config 0 cracks (non-vacuous split parity)
    assert np.all(np.diff(r.step) >= 0)
    assert len(set(r.elem.tolist())) == len(r.elem)
    assert np.all(st[r.elem] == 0)
    assert np.all(r.G > cfg0.tet_gc[r.elem])
    Ud = 0.0
    for e, a in zip(r.elem, r.area):
        Ud = Ud + cfg0.tet_gc[e] * a
    assert o.dissipated == pytest.approx(Ud, rel=1e-12)
    # frozen nodes (all incident tets inactive) have zero mass, velocity, acceleration
    s = o.state()
    frozen = s["m"] == 0
    assert np.all(s["v"][frozen] == 0) and np.all(s["a"][frozen] == 0)


def test_no_fracture_with_infinite_gc(cfg0):
    o = oracle.Oracle(cfg0.with_gc(np.inf))
    o.run(100, 1)
    assert len(o.records().elem) == 0
