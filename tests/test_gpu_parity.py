"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

The bar: identical split sets and BITWISE identical u, v, a, masses,
active flags, records and U_d -- the kernels follow the oracle's association order with
FMA contraction off, so any difference is a bug.  The north-star tolerance (relative L2
of u <= 1e-11 per 1000 steps) is asserted as well, so a report of the gap is available
if bitwise equality is ever relaxed.
"""
import numpy as np
import pytest

import cem_inputs as ci
import oracle

pytestmark = pytest.mark.gpu


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_04076_b200 as cem
    return cem


def run_pair(prob, steps, crack_every=1, chunks=1, flags=0, profile=False):
    cem = _gpu()
    sim = cem.Simulation.from_problem(prob, flags=flags)
    if profile:
        sim.set_profiling(True)
    orc = oracle.Oracle(prob)
    per = steps // chunks
    for _ in range(chunks):
        sim.step(per, crack_every)
        orc.run(per, crack_every)
    return sim, orc


def assert_parity(sim, orc, prob):
    g = sim.state()
    o = orc.state()
    assert g.step == orc.step_count
    assert g.dt == orc.dt
    # north-star tolerance first (informative), then the bitwise contract
    du = np.linalg.norm(g.u - o["u"]) / max(np.linalg.norm(o["u"]), 1e-300)
    assert du <= 1e-11
    r = orc.records()
    assert np.array_equal(g.rec_elem, r.elem), "split sets differ"
    assert np.array_equal(g.rec_step, r.step)
    assert np.array_equal(g.rec_cand, r.cand)
    assert np.array_equal(g.rec_G, r.G)
    assert np.array_equal(g.rec_area, r.area)
    assert np.array_equal(g.tet_state, o["state"])
    assert np.array_equal(g.mass, o["m"])
    for k in ("u", "v", "a"):
        bad = np.nonzero(getattr(g, k) != o[k])
        assert bad[0].size == 0, f"{k} differs at nodes {bad[0][:10]}"
    assert g.dissipated == orc.dissipated
    assert g.n_active == int(o["state"].sum())
    return g


def test_cfg0_full_run_bitwise():
    """BASELINE configs[0] in full: 200 steps with crack splitting every step."""
    p = ci.config(0)
    sim, orc = run_pair(p, p.steps, 1)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0          # non-vacuous: config 0 cracks


def test_cfg0_elastodynamics_long():
    p = ci.config(0).with_gc(np.inf)
    sim, orc = run_pair(p, 1000, 0, chunks=4)
    assert_parity(sim, orc, p)


@pytest.mark.parametrize("cells,seed,steps", [((40, 16, 4), 11, 300), ((33, 13, 3), 12, 257)])
def test_notched_plate_multi_tile(cells, seed, steps):
    """cfg1-like plate at sizes that span many thread blocks with a ragged tail."""
    L = 0.1 / 20
    p = ci.notched_plate(cells=cells, dims=(cells[0] * L / 2, cells[1] * L / 2, cells[2] * L / 4), seed=seed,
                         steps=steps)
    sim, orc = run_pair(p, steps, 1, chunks=3)
    assert_parity(sim, orc, p)


def test_edge_impact_dirichlet():
    """cfg2-like: prescribed-velocity ramp and two notches."""
    p = ci.edge_impact_plate(cells=(40, 20, 3), dims=(0.04, 0.02, 0.003), steps=300)
    sim, orc = run_pair(p, 300, 1, chunks=2)
    assert_parity(sim, orc, p)


def test_weak_block_predamage():
    """cfg3-like block with 0.5 % pre-damaged tets (Gc_e = 0) -> many splits."""
    p = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=300)
    sim, orc = run_pair(p, 300, 1)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 50


@pytest.mark.parametrize("critb_min", ["0", "300"])
@pytest.mark.parametrize("case", ["cfg0", "plate", "ct", "predamage", "overflow"])
def test_long_list_criterion_kernel(case, critb_min, monkeypatch):
    """The long-list criterion kernels (k_filter: refined early-out per listed tet; k_eval: 5 tets per warp)
    gives the oracle's bits: forced for every step (CEM_CRITB_MIN=0) and switched in mid-run by
    the list length (300)."""
    monkeypatch.setenv("CEM_CRITB_MIN", critb_min)
    if case == "cfg0":
        p, steps = ci.config(0), 200
    elif case == "plate":
        p, steps = ci.notched_plate(cells=(40, 16, 4), dims=(0.1, 0.04, 0.005), seed=11, steps=300), 300
    elif case == "ct":
        p, steps = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6), 250
    elif case == "predamage":
        p, steps = ci.weak_scaling_block(P=1, cells_per_rank=(30, 30, 5), steps=300), 300
    else:
        p = ci.notched_plate(cells=(60, 4, 20), dims=(0.06, 0.004, 0.02), seed=21, notch=False, steps=0)
        p.tet_gc[:] = 0.0
        steps = 8
    sim, orc = run_pair(p, steps, 1, chunks=2)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


def test_early_out_is_conservative():
    p = ci.config(0)
    cem = _gpu()
    a = cem.Simulation.from_problem(p)
    b = cem.Simulation.from_problem(p, flags=cem.CEM_F_NO_EARLY_OUT)
    a.step(200, 1); b.step(200, 1)
    sa, sb = a.state(), b.state()
    assert np.array_equal(sa.rec_elem, sb.rec_elem) and np.array_equal(sa.u, sb.u)


@pytest.mark.parametrize("flags", ["PERSISTENT", "PERSISTENT|NO_DISCARD"])
def test_persistent_path_bitwise(flags):
    """The persistent wavefront kernel gives the same bits as the oracle (and the staged path)."""
    cem = _gpu()
    fl = 0
    for f in flags.split("|"):
        fl |= getattr(cem, "CEM_F_" + f)
    p = ci.weak_scaling_block(P=1, cells_per_rank=(24, 20, 4), steps=150)
    sim, orc = run_pair(p, 150, 1, chunks=3, flags=fl)
    assert_parity(sim, orc, p)
    q = ci.config(0)
    sim, orc = run_pair(q, 200, 1, chunks=2, flags=fl)
    assert_parity(sim, orc, q)


def test_mixed_staged_then_persistent():
    cem = _gpu()
    p = ci.config(0)
    sim = cem.Simulation.from_problem(p, flags=cem.CEM_F_PERSISTENT)
    orc = oracle.Oracle(p)
    sim.set_profiling(True); sim.step(37, 1); sim.set_profiling(False)
    sim.step(63, 1)
    orc.run(100, 1)
    assert_parity(sim, orc, p)


def test_profiled_paths_agree():
    p = ci.config(0)
    sim, orc = run_pair(p, 120, 1, profile=True)
    assert_parity(sim, orc, p)
    t = sim.kernel_times()
    assert set(t) == {"stage_AB_strain_edge_stress", "stage_C_force_earlyout", "criterion_split", "stage_D_node_update"}
    assert all(v > 0 for v in t.values())


def test_split_overflow_path():
    """Thousands of simultaneous splits per step (unordered device records, host-ordered readback)."""
    p = ci.notched_plate(cells=(100, 4, 30), dims=(0.1, 0.004, 0.03), seed=21, notch=False, steps=0)
    p.tet_gc[:] = 0.0
    sim, orc = run_pair(p, 12, 1)
    g = assert_parity(sim, orc, p)
    counts = np.bincount(g.rec_step)
    assert counts.max() > 8192


def test_crack_update_matches_oracle_criterion():
    p = ci.config(0)
    cem = _gpu()
    sim = cem.Simulation.from_problem(p)
    sim.step(40, 0)                      # no cracking during the run
    st = sim.state()
    orc = oracle.Oracle(p)
    orc.run(40, 0)
    G, k, A, fl = orc.criterion(orc.state()["u"])
    n = sim.crack_update()
    g2 = sim.state()
    assert n == int(fl.sum()) > 0
    assert np.array_equal(np.sort(g2.rec_elem), np.nonzero(fl)[0])
    assert np.array_equal(g2.rec_G, G[g2.rec_elem])
    assert np.array_equal(g2.rec_cand, k[g2.rec_elem])


def test_deterministic_rerun():
    p = ci.weak_scaling_block(P=1, cells_per_rank=(20, 20, 4), steps=100)
    cem = _gpu()
    a = cem.Simulation.from_problem(p); a.step(100, 1)
    b = cem.Simulation.from_problem(p); b.step(100, 1)
    sa, sb = a.state(), b.state()
    assert sa.u.tobytes() == sb.u.tobytes() and np.array_equal(sa.rec_elem, sb.rec_elem)


def test_nonfinite_detected():
    cem = _gpu()
    p = ci.config(0).with_gc(np.inf)
    p.dt = 1e-5                          # ~40x the stability limit -> blows up
    sim = cem.Simulation.from_problem(p)
    sim.step(400, 0)
    with pytest.raises(cem.CemError) as ei:
        sim.state()
    assert ei.value.status == cem.CEM_ENONFINITE
    s = sim.state(check=False)
    assert s.nonfinite == 1 and s.nonfinite_node >= 0


@pytest.mark.parametrize("k,steps", [(3, 8), (2, 6), (1, 200), (4, 3)])
def test_full_size_config_bitwise(k, steps):
    """BASELINE configs at full size in the bench's launch configuration (PDL-chained stage
    kernels): configs[3] (1.02M tets), [2] (1.08M), [1] (207k, 200 steps), [4] (7.68M tets on
    one B200, 3 steps) against the oracle."""
    p = ci.config(k)
    sim, orc = run_pair(p, steps, 1)
    assert_parity(sim, orc, p)


@pytest.mark.parametrize("v0", [1.375, 3.993])
def test_compact_tension_dirichlet_branching(v0):
    """N2 workload: slot faces driven / held in x, fracture every step."""
    p = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=40 * v0, t0=20e-6)
    sim, orc = run_pair(p, 300)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


def test_compact_tension_full_size():
    """cfg6 (259k tets, v0 = 3.318 m/s) in the launch configuration bench.py uses."""
    p = ci.config(6)
    sim, orc = run_pair(p, 8)
    assert_parity(sim, orc, p)


# ---------------------------------------------------------------- degenerate and edge cases
def test_single_tet():
    """E = 1 (one partial warp, one block per stage) under a traction on one face."""
    X, T = ci.single_tet(0.01)
    p = ci.make_problem(X, T, tface=np.array([[1, 2, 3]]), tface_t=np.array([[2e6, 1e6, 0.0]]))
    sim, orc = run_pair(p, 50)
    assert_parity(sim, orc, p)


@pytest.mark.parametrize("critb_min", [None, "0"])
def test_high_valence_fan(critb_min, monkeypatch):
    """40 tets around one edge: the edge's incidence row and its end nodes' force-slot rows are
    40 long (several ELL chunks in stages AB and D, several batches in the mass recomputation),
    ring nodes pulled radially with a velocity ramp, low Gc so tets split."""
    if critb_min is not None:
        monkeypatch.setenv("CEM_CRITB_MIN", critb_min)
    X, T = ci.fan_mesh(40)
    ring = np.arange(2, X.shape[0], dtype=np.int32)
    v0 = 0.02 * X[ring] / np.linalg.norm(X[ring], axis=1)[:, None]   # splits spread over steps ~110-260
    p = ci.make_problem(X, T, Gc=0.5, vbc=(ring, np.full(ring.size, 7, np.uint8), v0, 2e-6))
    sim, orc = run_pair(p, 300, 1, chunks=3)
    g = assert_parity(sim, orc, p)
    assert g.rec_elem.size > 0


def test_all_tets_inactive():
    """No active tet: no stiffness, every mass 0 -> every node frozen, u stays 0."""
    X, T, _ = ci.kuhn_lattice((3, 2, 2), (0.03, 0.02, 0.02), 1)
    p = ci.make_problem(X, T, tet_state=np.zeros(T.shape[0], np.uint8), dt=1e-7)  # no tet to derive dt from
    sim, orc = run_pair(p, 20)
    g = assert_parity(sim, orc, p)
    assert np.all(g.u == 0.0) and np.all(g.mass == 0.0)


def test_isolated_node_and_partial_notch():
    """A node referenced by no tet (mass 0, frozen) next to a loaded, partly inactive plate."""
    p = ci.notched_plate(cells=(6, 4, 2), dims=(0.03, 0.02, 0.005), seed=9, steps=0)
    X = np.vstack([p.X, [[0.5, 0.5, 0.5]]])
    q = ci.make_problem(X, p.tets, tet_state=p.tet_state, tet_gc=p.tet_gc, tface=p.tface, tface_t=p.tface_t)
    sim, orc = run_pair(q, 80)
    g = assert_parity(sim, orc, q)
    assert g.mass[-1] == 0.0 and np.all(g.u[-1] == 0.0)


@pytest.mark.parametrize("E_target", [31, 33, 257, 511, 513])
def test_ragged_sizes(E_target):
    """Tet counts around warp (32) and block (256) boundaries: the first E_target tets of a
    lattice (their nodes renumbered densely)."""
    X, T, _ = ci.kuhn_lattice((8, 6, 2), (0.04, 0.03, 0.01), 3)
    T = T[:E_target]
    used, inv = np.unique(T.ravel(), return_inverse=True)
    p = ci.make_problem(X[used], inv.reshape(-1, 4).astype(np.int32),
                        tface=np.zeros((0, 3), np.int32), tface_t=np.zeros((0, 3)))
    # an initial kick through a prescribed velocity on the first node keeps the run non-trivial
    p = ci.make_problem(p.X, p.tets, vbc=(np.array([0], np.int32), np.array([7], np.uint8),
                                          np.array([[1.0, -0.5, 0.25]]), 1e-6))
    sim, orc = run_pair(p, 60)
    g = assert_parity(sim, orc, p)
    assert np.abs(g.u).max() > 0


@pytest.mark.parametrize("critb_min", [None, "0"])
@pytest.mark.parametrize("seed", range(8))
def test_randomized_problems(seed, critb_min, monkeypatch):
    """Seeded random problems: lattice size, jitter, material, traction direction, a random
    inactive set, random per-element Gc (some pre-damaged), an optional prescribed-velocity
    patch -- 120 steps with the criterion every step, bitwise vs the oracle; with the default
    criterion-kernel choice and with the long-list kernels forced on every step."""
    if critb_min is not None:
        monkeypatch.setenv("CEM_CRITB_MIN", critb_min)
    rng = np.random.default_rng(1000 + seed)
    cells = tuple(int(c) for c in rng.integers([4, 3, 2], [14, 9, 5]))
    dims = tuple(float(x) for x in rng.uniform(0.01, 0.05, 3))
    X, T, ijk = ci.kuhn_lattice(cells, dims, int(rng.integers(1 << 30)), jitter=float(rng.uniform(0.0, 0.2)))
    E = T.shape[0]
    state = (rng.random(E) > 0.05).astype(np.uint8)
    gc = rng.uniform(0.5, 20.0, E)
    gc[rng.random(E) < 0.02] = 0.0
    trac = rng.normal(0.0, 2e6, 3)
    faces, tr, _ = ci._loaded_faces(T, state, ijk, int(rng.integers(3)), 0, tuple(trac))
    vbc = None
    if seed % 2:
        nodes = np.nonzero(ijk[:, 0] == cells[0])[0][:6].astype(np.int32)
        vbc = (nodes, rng.integers(1, 8, nodes.size).astype(np.uint8), rng.normal(0.0, 2.0, (nodes.size, 3)),
               float(rng.uniform(0.0, 2e-6)))
    p = ci.make_problem(X, T, E=float(rng.uniform(10e9, 200e9)), nu=float(rng.uniform(0.1, 0.35)),
                        rho=float(rng.uniform(1500, 8000)), tet_state=state, tet_gc=gc, tface=faces, tface_t=tr,
                        vbc=vbc)
    sim, orc = run_pair(p, 120, 1, chunks=2)
    assert_parity(sim, orc, p)


def test_full_size_cracking_phase_kernel_choice(monkeypatch):
    """BASELINE configs[1] at full size into its cracking phase (~60k listed tets per step by
    step 3000): the long-list kernels on every step and the one-warp-per-tet kernel on every
    step give the same bits (the oracle parity of both is tested at small sizes above)."""
    cem = _gpu()
    p = ci.config(1)
    out = []
    for m in ("0", "1000000000"):
        monkeypatch.setenv("CEM_CRITB_MIN", m)
        sim = cem.Simulation.from_problem(p)
        sim.step(3000, 1)
        out.append(sim.state())
        sim.close()
    a, b = out
    assert a.rec_elem.size > 10000
    for k in ("u", "v", "a", "mass", "tet_state", "rec_elem", "rec_step", "rec_cand", "rec_G", "rec_area"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
