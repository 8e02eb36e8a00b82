"""Pins of the hexahedral crack patterns III-VI and the prism remainder in the hex oracle
(oracle/cem_oracle_hex.c, readings R28-R29 in DESIGN.md §3).

The oracle is pinned against values fixed by the geometry and the mathematics, not by retyping it:
- closed forms on a cube under uniaxial stretch (the crack plane's normal, the projected stress
  and stretch, and the section areas worked out by hand for each pattern);
- invariance of the 84 candidate values under a rigid rotation of the element and its fields, and
  under every orientation-preserving relabelling of the cube's nodes (catches a wrong partner,
  front or far-edge table);
- the remainder prism: three positive tets of total volume V/2 on a parallelepiped, covering the six
  prism nodes; lumped masses after splits sum to rho times the active volume;
- the mixed-mesh patch test (affine u gives sigma = D eps on every edge with a live smoothing
  domain, zero force sum, zero force at nodes away from the splits);
- whole cracking runs: every record strictly above Gc, each remainder equal to its candidate's
  prism, U_d = sum Gc * area.
"""
import itertools

import numpy as np
import pytest

import cem_inputs as ci
import oracle
from oracle import l0_literal as L0

XI = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
               [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)


def one_hex(X8, gc=np.inf, E=32e9, nu=0.2):
    X8 = np.asarray(X8, float)
    return ci.Problem(name="one_hex", X=X8.copy(), tets=np.arange(8, dtype=np.int32)[None, :],
                      tet_state=np.ones(1, np.uint8), tet_gc=np.full(1, gc), E=E, nu=nu, rho=2450.0, Gc=gc,
                      tface=np.zeros((0, 3), np.int32), tface_t=np.zeros((0, 3)),
                      vbc_node=np.zeros(0, np.int32), vbc_mask=np.zeros(0, np.uint8), vbc_v0=np.zeros((0, 3)))


def cube(h=1.0):
    return (XI + 1.0) * 0.5 * h


def test_closed_forms_uniaxial_cube():
    """u = (eps x, 0, 0) on a cube of side h: sigma uniform, sigma_1 = (lam + 2 mu) eps along x.
    III (x mid-plane): G = s1 eps h, area h^2; IV (plane through the bottom front and the top edge
    x = 0): n = (1, 0, 1/2)/|.|, G = s1 eps h / 1.25, area h^2 sqrt(1.25); V (corner 0, plane at 45
    degrees): G = s1 eps h / 4, area h^2/sqrt 2; VI (corner triangle): G = s1 eps h / 6, area sqrt3 h^2/8;
    fronts along y see no stretch (H = 0): G = 0."""
    h, eps = 0.01, 1e-4
    p = one_hex(cube(h))
    o = oracle.HexOracle(p)
    lam = p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)); mu = p.E / (2 * (1 + p.nu))
    s1 = (lam + 2 * mu) * eps
    u = np.zeros((8, 3)); u[:, 0] = eps * p.X[:, 0]
    G, A, P = o.candidates(u, 0)
    ref = s1 * eps * h
    r = dict(rel=1e-12, abs=1e-12 * ref)
    # face 0 = (0,1,2,3): front j=0 joins edges (0,1) and (3,2) (x-edges), j=1 the y-edges
    assert G[0] == pytest.approx(ref, **r) and A[0] == pytest.approx(h * h, rel=1e-12)
    assert G[1] == 0.0
    assert (P[:12] == -1).all()                                   # III: no remainder
    assert G[12] == pytest.approx(ref / 1.25, **r) and A[12] == pytest.approx(h * h * np.sqrt(1.25), rel=1e-12)
    assert sorted(P[12]) == [1, 2, 4, 5, 6, 7]                    # half-hex prism away from edge (0,3)
    assert G[36] == pytest.approx(ref / 4, **r) and A[36] == pytest.approx(h * h / np.sqrt(2), rel=1e-12)
    assert G[60] == pytest.approx(ref / 6, **r) and A[60] == pytest.approx(np.sqrt(3) * h * h / 8, rel=1e-12)
    assert sorted(P[36]) == sorted(P[60]) == [1, 2, 3, 5, 6, 7]   # half-hex away from edge (0,4)
    # the largest is a mid-plane x candidate, and the lowest such k wins (R14)
    assert G.max() == pytest.approx(ref, **r)
    assert np.isclose(G, ref, rtol=1e-12).sum() == 4             # the x mid-plane from 4 faces


def _rot(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(3, 3)))
    return q * np.sign(np.linalg.det(q))


def _distorted(seed, jit=0.12):
    rng = np.random.default_rng(seed)
    A = np.eye(3) + 0.2 * rng.normal(size=(3, 3))
    if np.linalg.det(A) < 0:
        A[:, 0] *= -1
    return cube(0.01) @ A.T + jit * 0.01 * rng.uniform(-1, 1, size=(8, 3))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_rotation_invariance(seed):
    X = _distorted(seed)
    rng = np.random.default_rng(seed + 10)
    u = rng.normal(size=(8, 3)) * 1e-5
    R = _rot(seed)
    G, A, P = oracle.HexOracle(one_hex(X)).candidates(u, 0)
    G2, A2, P2 = oracle.HexOracle(one_hex(X @ R.T)).candidates(u @ R.T, 0)
    scale = np.abs(G).max()
    assert scale > 0
    assert np.abs(G - G2).max() <= 1e-10 * scale
    assert np.abs(A - A2).max() <= 1e-12 * A.max()
    assert (P == P2).all()


def _cube_rotations():
    out = []
    for perm in itertools.permutations(range(3)):
        for sg in itertools.product((1, -1), repeat=3):
            R = np.zeros((3, 3))
            for i in range(3):
                R[i, perm[i]] = sg[i]
            if np.linalg.det(R) > 0:
                out.append(R)
    return out


@pytest.mark.parametrize("seed", [4, 5])
def test_relabelling_invariance(seed):
    """The 24 rotations of the cube relabel the local nodes; the multiset of (G, area) pairs and of
    remainder prisms (as node sets) must not change -- every face, front, partner and far edge is
    then defined symmetrically."""
    X = _distorted(seed, jit=0.08)
    u = np.random.default_rng(seed).normal(size=(8, 3)) * 1e-5
    p = one_hex(X)
    G0, A0, P0 = oracle.HexOracle(p).candidates(u, 0)
    key0 = sorted(zip(np.round(G0 / np.abs(G0).max(), 9), np.round(A0 / A0.max(), 9)))
    prisms0 = sorted(tuple(sorted(p.tets[0][P0[k]])) for k in range(84) if P0[k, 0] >= 0)
    rots = _cube_rotations()
    assert len(rots) == 24
    for R in rots:
        perm = [int(np.nonzero((XI == R @ XI[i]).all(axis=1))[0][0]) for i in range(8)]
        H = np.empty(8, np.int32)
        H[perm] = np.arange(8)           # new local node perm[i] is the old local node i
        q = one_hex(X); q.tets = H[None, :]
        G, A, P = oracle.HexOracle(q).candidates(u, 0)
        key = sorted(zip(np.round(G / np.abs(G0).max(), 9), np.round(A / A0.max(), 9)))
        assert key == key0
        prisms = sorted(tuple(sorted(H[P[k]])) for k in range(84) if P[k, 0] >= 0)
        assert prisms == prisms0


@pytest.mark.parametrize("seed", [6, 7])
def test_remainder_prism_tets(seed):
    """Every remainder candidate of a parallelepiped: three tets of positive volume summing to V/2 whose
    nodes are the prism's six nodes; the hex's lost nodes keep no mass."""
    rng = np.random.default_rng(seed)
    A = np.eye(3) + 0.25 * rng.normal(size=(3, 3))
    if np.linalg.det(A) < 0:
        A[:, 0] *= -1
    X = cube(0.02) @ A.T
    p = one_hex(X)
    V = abs(np.linalg.det(A)) * 0.02 ** 3
    _, _, P = oracle.HexOracle(p).candidates(np.zeros((8, 3)), 0)
    for k in range(12, 84):
        o = oracle.HexOracle(p)
        o.force_split(0, k)
        el = o.elements()
        assert el["hex_active"][0] == 0 and el["tet_active"][0].all()
        tv = el["tet_V"][0]
        assert (tv > 0).all()
        assert tv.sum() == pytest.approx(V / 2, rel=1e-12)
        assert set(el["tet_nodes"][0].ravel()) == set(P[k])
        # tets are distinct and each is a 4-subset of the prism
        assert len({tuple(sorted(t)) for t in el["tet_nodes"][0]}) == 3
        m = o.state()["m"]
        assert m.sum() == pytest.approx(p.rho * V / 2, rel=1e-12)
        lost = sorted(set(range(8)) - set(P[k]))
        assert len(lost) == 2 and (m[lost] == 0).all()
    o = oracle.HexOracle(p)
    o.force_split(0, 3)                                 # pattern III: fully cracked
    el = o.elements()
    assert el["hex_active"][0] == 0 and not el["tet_active"].any()
    assert (o.state()["m"] == 0).all()


def _split_block(seed=3):
    p = ci.hex_block((5, 4, 3), dims=(0.025, 0.02, 0.015), seed=seed, jitter=0.1)
    o = oracle.HexOracle(p)
    rng = np.random.default_rng(seed)
    for e in rng.choice(p.n_tets, size=12, replace=False):
        o.force_split(int(e), int(rng.integers(0, 84)))
    return p, o


def test_mass_after_splits():
    p, o = _split_block()
    el = o.elements()
    V, _ = o.geometry()
    vol = (V * el["hex_active"]).sum() + (el["tet_V"] * el["tet_active"]).sum()
    assert o.state()["m"].sum() == pytest.approx(p.rho * vol, rel=1e-12)
    assert el["tet_active"].any() and (el["hex_active"] == 0).any()


def test_mixed_patch_test():
    """Affine u on a mesh with remainder tets: sigma = D sym(A) on every edge with a live smoothing
    domain (the tets' strain and the mixed edge gather), internal forces sum to zero, and nodes whose
    elements were not split and are inside the block carry no force."""
    p, o = _split_block(5)
    A = np.random.default_rng(2).normal(size=(3, 3)) * 1e-4
    u = p.X @ A.T
    sig, vh, en = o.edge_stress_all(u)
    Sy = 0.5 * (A + A.T)
    want = L0.D_matrix(p.E, p.nu) @ np.array([Sy[0, 0], Sy[1, 1], Sy[2, 2], 2 * Sy[0, 1], 2 * Sy[1, 2], 2 * Sy[0, 2]])
    live = vh > 0
    assert live[o.S:].any()                             # some diagonal edges carry remainder tets
    assert np.abs(sig[live] - want[None, :]).max() <= 1e-10 * np.abs(want).max()
    assert (sig[~live] == 0).all()
    f = o.internal_force(u)
    assert np.abs(f.sum(axis=0)).max() <= 1e-12 * np.abs(f).max()
    el = o.elements()
    touched = np.zeros(p.n_nodes, bool)
    touched[p.tets[el["hex_active"] == 0].ravel()] = True
    ijk = p.node_ijk
    inside = np.all((ijk > 0) & (ijk < np.array(p.cells)[None, :]), axis=1)
    sel = inside & ~touched
    assert sel.any()
    assert np.abs(f[sel]).max() <= 1e-9 * np.abs(f).max()


def test_cracking_run_invariants():
    p = ci.hex_block((10, 6, 2), dims=(0.05, 0.03, 0.01), seed=2, traction=4e6, gc=2.0, notch=0.3)
    o = oracle.HexOracle(p)
    o.run(400, crack_every=1)
    r = o.records()
    assert r.step.size >= 3
    E = p.n_tets
    assert (r.G > 2.0).all()
    assert np.all(np.diff(r.step) >= 0)
    assert o.dissipated == pytest.approx((2.0 * r.area).sum(), rel=1e-12)
    el = o.elements()
    hexes = r.elem < E
    assert (el["hex_active"][r.elem[hexes]] == 0).all()
    for e, k in zip(r.elem[hexes], r.cand[hexes]):
        if k >= 12:   # a remainder: its tets' nodes are the candidate's prism (as global ids)
            assert el["tet_nodes"][e].min() >= 0
        else:
            assert (el["tet_nodes"][e] == -1).all()
    tets = r.elem[~hexes] - E
    assert (el["tet_active"][tets // 3, tets % 3] == 0).all()
    V, _ = o.geometry()
    vol = (V * el["hex_active"]).sum() + (el["tet_V"] * el["tet_active"]).sum()
    assert o.state()["m"].sum() == pytest.approx(p.rho * vol, rel=1e-12)
