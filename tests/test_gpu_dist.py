"""Multi-rank GPU path on one B200 (loopback transport): P sub-domain contexts with the
2-ring ghost layer, owner-only updates/records, pack -> device copy -> unpack halo exchange
after every step.  The assembled result must equal the single-domain oracle BIT FOR BIT
(P-invariance)."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle

pytestmark = pytest.mark.gpu


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_04076_b200.dist as dist
    return dist


def check(prob, P, steps, crack_every=1, chunks=2):
    dist = _gpu()
    grp = dist.LoopbackGroup(prob, P)
    orc = oracle.Oracle(prob)
    for _ in range(chunks):
        grp.step(steps // chunks, crack_every)
        orc.run(steps // chunks, crack_every)
    g, o, r = grp.state(), orc.state(), orc.records()
    for k in ("u", "v", "a"):
        assert np.array_equal(g[k], o[k]), k
    assert np.array_equal(g["mass"], o["m"])
    assert np.array_equal(g["tet_state"], o["state"])
    assert np.array_equal(g["rec_elem"], r.elem) and np.array_equal(g["rec_step"], r.step)
    assert np.array_equal(g["rec_G"], r.G) and np.array_equal(g["rec_cand"], r.cand)
    assert g["dissipated"] == orc.dissipated
    return g


@pytest.mark.parametrize("P", [2, 3, 4])
def test_loopback_cfg0(P):
    g = check(ci.config(0), P, 200)
    assert g["rec_elem"].size > 0


def test_loopback_weak_block_predamage():
    p = ci.weak_scaling_block(P=2, cells_per_rank=(20, 16, 4), steps=0)
    g = check(p, 2, 160)
    assert g["rec_elem"].size > 10


def test_loopback_dirichlet():
    p = ci.edge_impact_plate(cells=(30, 16, 3), dims=(0.03, 0.016, 0.003), steps=0)
    check(p, 3, 120)


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_energy_ledger(P):
    """The ranks' ledger shares (owned nodes, owned edges, own records) sum to the whole
    mesh's ledger: equal to the oracle's to the rounding bound of the sums."""
    dist = _gpu()
    p = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6)
    grp = dist.LoopbackGroup(p, P)
    orc = oracle.Oracle(p)
    grp.step(150, 1)
    orc.run(150, 1)
    g, o = grp.energy(), orc.energy()
    tol = 4 * 6 * p.n_tets * np.finfo(np.float64).eps
    scale = max(abs(o[k]) for k in ("kinetic", "strain", "external", "reaction"))
    for k in ("kinetic", "strain", "external", "reaction"):
        assert abs(g[k] - o[k]) <= tol * scale, (k, g[k], o[k])
    assert g["dissipated"] == pytest.approx(o["dissipated"], rel=1e-12)
    assert o["reaction"] > 0.0 and o["dissipated"] > 0.0


@pytest.mark.parametrize("P", [2, 3, 4])
def test_loopback_p2p_halo(P):
    """The P2P halo (stage D and the split pass store into the peers' receive buffers, the
    receiver unpacks after the step) gives the same bits as the single-domain oracle."""
    dist = _gpu()
    import paper_2508_04076_b200 as cem
    for prob, steps in ((ci.config(0), 200),
                        (ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6), 150)):
        grp = dist.LoopbackGroup(prob, P, flags=cem.CEM_F_P2P)
        orc = oracle.Oracle(prob)
        for _ in range(2):
            grp.step(steps // 2, 1)
            orc.run(steps // 2, 1)
        g, o, r = grp.state(), orc.state(), orc.records()
        for k in ("u", "v", "a"):
            assert np.array_equal(g[k], o[k]), k
        assert np.array_equal(g["tet_state"], o["state"])
        assert np.array_equal(g["rec_elem"], r.elem) and np.array_equal(g["rec_G"], r.G)
        assert g["rec_elem"].size > 0


@pytest.mark.parametrize("seed", range(4))
def test_loopback_randomized(seed):
    """Seeded random problems on P = 2..4 ranks, copy and P2P halos alternately: bitwise."""
    dist = _gpu()
    import paper_2508_04076_b200 as cem
    rng = np.random.default_rng(2000 + seed)
    cells = tuple(int(c) for c in rng.integers([8, 4, 2], [16, 9, 4]))
    X, T, ijk = ci.kuhn_lattice(cells, tuple(float(x) for x in rng.uniform(0.01, 0.05, 3)),
                                int(rng.integers(1 << 30)), jitter=0.1)
    E = T.shape[0]
    gc = rng.uniform(0.5, 10.0, E)
    gc[rng.random(E) < 0.03] = 0.0
    faces, tr, _ = ci._loaded_faces(T, np.ones(E, np.uint8), ijk, 1, 0, tuple(rng.normal(0.0, 2e6, 3)))
    p = ci.make_problem(X, T, tet_gc=gc, tface=faces, tface_t=tr)
    P = int(rng.integers(2, 5))
    grp = dist.LoopbackGroup(p, P, flags=cem.CEM_F_P2P if seed % 2 else 0)
    orc = oracle.Oracle(p)
    grp.step(100, 1)
    orc.run(100, 1)
    g, o, r = grp.state(), orc.state(), orc.records()
    for k in ("u", "v", "a"):
        assert np.array_equal(g[k], o[k]), k
    assert np.array_equal(g["rec_elem"], r.elem) and np.array_equal(g["tet_state"], o["state"])
    assert r.elem.size > 0


@pytest.mark.parametrize("P,p2p", [(2, False), (3, True)])
def test_loopback_long_list_criterion_kernel(P, p2p, monkeypatch):
    """Every step through the long-list criterion kernels (k_filter + k_eval) on P ranks: owner-only
    records, ghost splits delivered by the halo (copy or P2P), bitwise equal to the oracle."""
    monkeypatch.setenv("CEM_CRITB_MIN", "0")
    dist = _gpu()
    import paper_2508_04076_b200 as cem
    p = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6)
    grp = dist.LoopbackGroup(p, P, flags=cem.CEM_F_P2P if p2p else 0)
    orc = oracle.Oracle(p)
    for _ in range(2):
        grp.step(100, 1)
        orc.run(100, 1)
    g, o, r = grp.state(), orc.state(), orc.records()
    for k in ("u", "v", "a"):
        assert np.array_equal(g[k], o[k]), k
    assert np.array_equal(g["mass"], o["m"])
    assert np.array_equal(g["tet_state"], o["state"])
    assert np.array_equal(g["rec_elem"], r.elem) and np.array_equal(g["rec_G"], r.G)
    assert r.elem.size > 0
