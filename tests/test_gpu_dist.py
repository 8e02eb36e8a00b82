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
