"""The criterion's early-out bounds ("Long criterion lists") against the
oracle's 24 candidate energy release rates.

Stage C skips a tet when  max_l g_l * max_l |du_l| (1 + 1e-6) <= Gc_e  (g_l: Gershgorin bound of
sigma at edge l); k_filter keeps a listed tet unless every candidate has N_k / |m| below Gc_e, with
N_k = 1/2 (g_pr H_cp |du_cp.m| + g_qr H_cq |du_cq.m|)  (pattern I) or 1/2 g_cr (H_cp |du_cp.m| +
H_cq |du_cq.m|)  (pattern II).  Both rest on |S(s,m)| <= |sigma_1| |m| <= g_s |m| and
|Dd(a,b,m)| = H_ab |du_ab . m|.  Pinned here: |G_k| <= N_k/|m| <= the stage-C bound for every
candidate of random tets under random displacements (tension, compression, shear, rigid
motions), with the oracle's G_k (PAPER.md eq:G-I, eq:G-II) and the oracle's edge stresses."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle

LOCAL_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
LID = {}
for _l, (_a, _b) in enumerate(LOCAL_EDGES):
    LID[(_a, _b)] = LID[(_b, _a)] = _l


def gershgorin(s6):
    return max(abs(s6[0]) + abs(s6[3]) + abs(s6[5]), abs(s6[1]) + abs(s6[3]) + abs(s6[4]),
               abs(s6[2]) + abs(s6[4]) + abs(s6[5]))


def bounds(X, u, s6l):
    """(per-candidate bound b[24], stage-C bound B0) of one tet: X, u [4,3]; s6l [6][6]."""
    g = [gershgorin(s) for s in s6l]
    du = [u[b] - u[a] for a, b in LOCAL_EDGES]
    H = [du[l] @ (2 * (X[b] - X[a]) + du[l]) > 0 for l, (a, b) in enumerate(LOCAL_EDGES)]
    B0 = max(g) * max(np.linalg.norm(d) for d in du)
    b = np.zeros(24)
    for k in range(24):
        c, f, t = k // 6, (k % 6) // 2, k & 1
        o = [x for x in range(4) if x != c]
        p, q, r = o[1 if f == 2 else 0], o[1 if f == 0 else 2], o[2 - f]
        m = np.cross(X[q] - X[p], (X[r] - X[c]) if t == 0 else (X[r] - X[p]))
        ap = abs((u[p] - u[c]) @ m) if H[LID[(c, p)]] else 0.0
        aq = abs((u[q] - u[c]) @ m) if H[LID[(c, q)]] else 0.0
        N = 0.5 * (g[LID[(p, r)]] * ap + g[LID[(q, r)]] * aq) if t == 0 else 0.5 * g[LID[(c, r)]] * (ap + aq)
        b[k] = N / np.linalg.norm(m)
    return b, B0


def fields(kind, X, rng):
    c = X.mean(axis=0)
    if kind == "random":
        return rng.standard_normal(X.shape) * 1e-4
    if kind == "tension":
        return (X - c) * np.array([2e-4, -4e-5, -4e-5]) + rng.standard_normal(X.shape) * 1e-6
    if kind == "compression":
        return (X - c) * -3e-4 + rng.standard_normal(X.shape) * 1e-6
    if kind == "shear":
        return np.stack([3e-4 * (X[:, 1] - c[1]), np.zeros(len(X)), np.zeros(len(X))], 1)
    # rigid rotation + translation (no strain, stretches from the rotation's second-order term)
    th = 1e-3
    R = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.0], [0.0, 0.0, 1.0]])
    return (X - c) @ R.T + c - X + 1e-3


@pytest.mark.parametrize("kind", ["random", "tension", "compression", "shear", "rigid"])
@pytest.mark.parametrize("seed", range(3))
def test_candidate_bounds_hold(kind, seed):
    rng = np.random.default_rng(100 + seed)
    X, T, _ = ci.random_tet_mesh(seed, n_cells=(2, 2, 2), jitter=0.25)
    p = ci.make_problem(X, T)
    o = oracle.Oracle(p)
    u = fields(kind, p.X, rng)
    sig, _ = o.edge_stress(u)
    en, _ = o.edges()
    eid = {(int(min(a, b)), int(max(a, b))): s for s, (a, b) in enumerate(en)}
    nontrivial = 0
    for e in range(p.n_tets):
        t = p.tets[e]
        s6l = [sig[eid[(int(min(t[a], t[b])), int(max(t[a], t[b])))]] for a, b in LOCAL_EDGES]
        G, _ = o.candidates(u, e)
        b, B0 = bounds(p.X[t], u[t], s6l)
        assert np.all(np.abs(G) <= b * (1 + 1e-12) + 1e-300), (e, np.abs(G) - b)
        assert np.all(b <= B0 * (1 + 1e-12) + 1e-300)
        nontrivial += int(np.abs(G).max() > 0)
    if kind != "compression":
        assert nontrivial > 0


def test_refined_bound_is_tighter_on_a_cracking_state():
    """On a config-0 state mid-run the refined bound discards most tets stage C lists."""
    p = ci.config(0)
    o = oracle.Oracle(p)
    o.run(120, 1)
    u = o.state()["u"]
    act = o.state()["state"].astype(bool)
    sig, _ = o.edge_stress(u)
    en, _ = o.edges()
    eid = {(int(min(a, b)), int(max(a, b))): s for s, (a, b) in enumerate(en)}
    gc = p.tet_gc
    listed = kept = 0
    for e in np.nonzero(act)[0]:
        t = p.tets[e]
        s6l = [sig[eid[(int(min(t[a], t[b])), int(max(t[a], t[b])))]] for a, b in LOCAL_EDGES]
        b, B0 = bounds(p.X[t], u[t], s6l)
        if B0 * (1 + 1e-6) > gc[e]:
            listed += 1
            kept += int(b.max() * (1 + 1e-6) > gc[e])
    assert listed > 0 and kept < listed


# ------------------------------------------------------------------ hexahedra (patterns III-VI)
HEX_EDGES = [(0, 1), (1, 2), (2, 3), (0, 3), (4, 5), (5, 6), (6, 7), (4, 7), (0, 4), (1, 5), (2, 6), (3, 7)]


@pytest.mark.parametrize("kind", ["random", "tension", "compression", "shear", "rigid"])
def test_hex_early_out_bound_dominates_all_84_candidates(kind):
    """k_hexcrit skips an active hex when  max_l g_l * max_l |du_l| (1 + 1e-6) <= Gc_e  over the
    hex's 12 edges (g_l: Gershgorin bound of the edge stress).  Every pattern III-VI candidate is
    1/2 (S_1 Dd_1 + S_2 Dd_2)/|m|^2 with S_i the projected stress of one of those edges and Dd_i the
    stretch of one of them along m (R28), so the bound dominates all 84 values
    of the hex oracle -- checked on every hex of jittered blocks under five kinds of fields."""
    rng = np.random.default_rng({"random": 1, "tension": 2, "compression": 3, "shear": 4, "rigid": 5}[kind])
    p = ci.hex_block((3, 3, 2), dims=(0.03, 0.03, 0.02), seed=7, jitter=0.15)
    o = oracle.HexOracle(p)
    u = fields(kind, p.X, rng)
    s, vh, en = o.edge_stress(u)
    eid = {(min(a, b), max(a, b)): i for i, (a, b) in enumerate(en)}
    worst = 0.0
    for e in range(p.n_tets):
        nd = p.tets[e]
        g = max(gershgorin(s[eid[(min(nd[a], nd[b]), max(nd[a], nd[b]))]]) for a, b in HEX_EDGES)
        dmax = max(np.linalg.norm(u[nd[b]] - u[nd[a]]) for a, b in HEX_EDGES)
        G, A, P = o.candidates(u, e)
        B0 = g * dmax
        assert np.all(np.abs(G) <= B0 * (1 + 1e-9) + 1e-300), (e, np.abs(G).max(), B0)
        if B0 > 0:
            worst = max(worst, np.abs(G).max() / B0)
    assert kind == "rigid" or worst > 1e-3     # the bound is not vacuous (same order as the largest |G|)
