"""Oracle pins for the explicit Newmark (beta = 0) integration.

P6 1-dof m = 2, F = 4, dt = 0.1, gamma = 1/2 from rest: u1 = 0.01, v1 = 0.2, a1 = 2 and
   u_n = (n dt)^2 exactly (hand integration; golden/newmark_1dof.txt).
P7 energy balance with Gc = inf: |KE + SE - W_ext| <= 1e-3 peak W_ext;
   1D wave speed of a laterally constrained bar = c_d = sqrt((lam+2mu)/rho).
Ramp: prescribed dofs follow v = (t/t0) v0 exactly.
"""
import os

import numpy as np
import pytest

import cem_inputs as ci
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_newmark_one_dof():
    vals = {}
    for line in open(os.path.join(GOLDEN, "newmark_1dof.txt")):
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            vals[k.strip()] = float(v)
    m, F, dt = np.array([vals["m"]]), np.array([vals["F"]]), vals["dt"]
    u = np.zeros(1); v = np.zeros(1); a = F / m              # a0 = F/m
    for n in range(1, 11):
        u = oracle.predict(u, v, a, dt)
        v, a = oracle.newmark_free(m, F, np.zeros(1), v, a, dt, 0.5)
        if n == 1:
            assert u[0] == pytest.approx(vals["u1"], rel=1e-14)
            assert v[0] == pytest.approx(vals["v1"], rel=1e-14)
            assert a[0] == pytest.approx(vals["a1"], rel=1e-14)
        assert u[0] == pytest.approx((n * dt) ** 2, rel=1e-13)


def _energies(o, p, f):
    s = o.state()
    KE = 0.5 * np.sum(s["m"][:, None] * s["v"] ** 2)
    SE = o.strain_energy(s["u"])
    W = np.vdot(f, s["u"])
    return KE, SE, W


def test_energy_balance_no_fracture():
    p = ci.notched_plate(cells=(10, 4, 2), dims=(0.05, 0.02, 0.005), seed=5, steps=0).with_gc(np.inf)
    o = oracle.Oracle(p)
    f = o.fext()
    hist = []
    for _ in range(40):
        o.run(50, 0)
        hist.append(_energies(o, p, f))
    hist = np.array(hist)
    Wpeak = np.abs(hist[:, 2]).max()
    bal = hist[:, 0] + hist[:, 1] - hist[:, 2]
    assert Wpeak > 0
    assert np.abs(bal).max() <= 1e-3 * Wpeak


def test_bar_wave_speed():
    """Laterally constrained bar (uniaxial strain) under a step traction at x = 0: the
    wave front (half-plateau particle velocity) travels at c_d (within 3 %)."""
    n = 120
    p = ci.notched_plate(cells=(n, 1, 1), dims=(0.12, 0.001, 0.001), seed=0, notch=False, steps=0, jitter=0.0)
    ijk = p.node_ijk
    # traction on x = 0 face pushing +x
    X, T = p.X, p.tets
    faces = []
    for e in range(T.shape[0]):
        for f in range(4):
            tri = [T[e, a] for a in range(4) if a != f]
            if all(ijk[t, 0] == 0 for t in tri):
                faces.append(tri)
    sig0 = 1e6
    tface_t = np.tile([sig0, 0.0, 0.0], (len(faces), 1))
    nodes = np.arange(p.n_nodes, dtype=np.int32)
    vbc = (nodes, np.full(p.n_nodes, 6, np.uint8), np.zeros((p.n_nodes, 3)), 0.0)   # v_y = v_z = 0
    q = ci.make_problem(X, T, E=p.E, nu=p.nu, rho=p.rho, tet_gc=np.full(T.shape[0], np.inf),
                        tface=faces, tface_t=tface_t, vbc=vbc)
    o = oracle.Oracle(q)
    lam, mu = o.lame()
    cd = np.sqrt((lam + 2 * mu) / q.rho)
    steps = int(0.6 * 0.12 / cd / o.dt)
    o.run(steps, 0)
    t = steps * o.dt
    vx = o.state()["v"][:, 0]
    xs = np.unique(X[:, 0])
    prof = np.array([vx[np.isclose(X[:, 0], x)].mean() for x in xs])
    plateau = sig0 / (q.rho * cd)               # particle velocity behind the front
    behind = prof[xs < 0.3 * cd * t]
    assert np.abs(behind.mean() - plateau) < 0.05 * plateau
    front = xs[np.nonzero(prof < 0.5 * plateau)[0][0]]
    assert front / t == pytest.approx(cd, rel=0.03)


def test_dirichlet_ramp_exact():
    p = ci.edge_impact_plate(cells=(8, 8, 1), dims=(0.008, 0.008, 0.001), steps=0, t0=1e-6)
    o = oracle.Oracle(p)
    dt = o.dt
    for n in range(1, 30):
        o.run(1, 1)
        t = n * dt
        v = o.state()["v"]
        want = (t / 1e-6) * 16.5 if t <= 1e-6 else 16.5
        assert np.all(v[p.vbc_node, 0] == want)


def test_thread_count_determinism(cfg0):
    import subprocess, sys, json
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import cem_inputs as ci, oracle;"
            "o = oracle.Oracle(ci.config(0)); o.run(60, 1); s = o.state();"
            "import hashlib; print(hashlib.sha1(s['u'].tobytes() + s['state'].tobytes()).hexdigest())"
            % os.path.dirname(GOLDEN)[:-len('/tests')])
    outs = set()
    for nt in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=nt)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env).decode().strip())
    assert len(outs) == 1
