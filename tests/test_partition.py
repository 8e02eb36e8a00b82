"""Multi-rank decomposition on CPU.

* plan invariants of `cem_partition` (the library's host-side logic): unique ownership,
  layer 1 = owned tets + tets of owned nodes, the ghost ring completes every edge of a
  layer-1 tet, send/recv lists of every pair of ranks line up;
* world_size-2 gloo run: each rank advances the CPU oracle on its local sub-mesh and
  exchanges (u, v, a) of non-owned nodes and the state of ghost tets after every step,
  exactly the data the GPU path exchanges; the owned results equal the single-domain
  oracle BIT FOR BIT, including the split set.
"""
import os
import sys

import numpy as np
import pytest

import cem_inputs as ci

LOCAL_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _plan(prob, P):
    from paper_2508_04076_b200.dist import partition
    return [partition(prob.X, prob.tets, P, r) for r in range(P)]


@pytest.mark.parametrize("P", [2, 3, 4])
def test_partition_invariants(P):
    p = ci.weak_scaling_block(P=1, cells_per_rank=(12, 8, 3), steps=0)
    plans = _plan(p, P)
    E, N = p.n_tets, p.n_nodes
    owner = plans[0]["tet_owner"]
    assert np.all([np.array_equal(pl["tet_owner"], owner) for pl in plans])   # same plan everywhere
    assert set(np.unique(owner)) == set(range(P))
    counts = np.bincount(owner, minlength=P)
    assert counts.max() - counts.min() <= 1                                     # RCB balance
    # node ownership: owner of the lowest-id incident tet
    first = np.full(N, E)
    for e in range(E):
        for k in p.tets[e]:
            first[k] = min(first[k], e)
    assert np.array_equal(plans[0]["node_owner"], owner[first])
    inc = {}
    for e, t in enumerate(p.tets):
        for a, b in LOCAL_EDGES:
            inc.setdefault((min(t[a], t[b]), max(t[a], t[b])), []).append(e)
    owned_nodes_total = 0
    for r, pl in enumerate(plans):
        tg, ng = pl["tet_global"], pl["node_global"]
        assert np.all(np.diff(tg) > 0) and np.all(np.diff(ng) > 0)
        l1 = set(tg[(pl["tet_flag"] & 1) != 0])
        owned = set(np.nonzero(owner == r)[0])
        assert set(tg[(pl["tet_flag"] & 2) != 0]) == owned and owned <= l1
        own_nodes = set(ng[pl["node_owned"] == 1])
        owned_nodes_total += len(own_nodes)
        for k in own_nodes:                           # f_int of an owned node is complete
            assert {e for e in range(E) if k in p.tets[e]} <= l1
        local = set(tg)
        for e in l1:                                  # sigma of every layer-1 edge is complete
            t = p.tets[e]
            for a, b in LOCAL_EDGES:
                assert set(inc[(min(t[a], t[b]), max(t[a], t[b]))]) <= local
        assert set(p.tets[list(local)].ravel()) == set(ng)
    assert owned_nodes_total == N
    # exchange lists pair up: r sends to q exactly what q receives from r, in the same order
    for r, pl in enumerate(plans):
        for j, q in enumerate(pl["peers"]):
            jq = list(plans[q]["peers"]).index(r)
            sent = pl["node_global"][pl["send_nodes"][j]]
            recv = plans[q]["node_global"][plans[q]["recv_nodes"][jq]]
            assert np.array_equal(sent, recv)
            sent = pl["tet_global"][pl["send_tets"][j]]
            recv = plans[q]["tet_global"][plans[q]["recv_tets"][jq]]
            assert np.array_equal(sent, recv)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle
        from paper_2508_04076_b200.dist import partition
        prob = ci.notched_plate(cells=(12, 6, 2), dims=(0.03, 0.015, 0.005), seed=3, steps=0)
        pl = partition(prob.X, prob.tets, world, rank)
        tg, ng = pl["tet_global"], pl["node_global"]
        g2l = {int(k): i for i, k in enumerate(ng)}
        lt = np.vectorize(lambda k: g2l[int(k)])(prob.tets[tg]).astype(np.int32)
        faces = [f for f in prob.tface if all(int(k) in g2l for k in f)]
        tt = [prob.tface_t[i] for i, f in enumerate(prob.tface) if all(int(k) in g2l for k in f)]
        lf = np.array([[g2l[int(k)] for k in f] for f in faces], np.int32).reshape(-1, 3)
        sub = ci.make_problem(prob.X[ng], lt, E=prob.E, nu=prob.nu, rho=prob.rho, tet_state=prob.tet_state[tg],
                              tet_gc=prob.tet_gc[tg], tface=lf, tface_t=np.array(tt).reshape(-1, 3))
        glob = oracle.Oracle(prob)
        orc = oracle.Oracle(sub, dt=glob.dt)          # every rank uses the global time step
        peers = list(pl["peers"])

        def exchange():
            s = orc.state()
            ops, bufs = [], []
            for j, qr in enumerate(peers):
                sn, st = pl["send_nodes"][j], pl["send_tets"][j]
                msg = np.concatenate([s["u"][sn].ravel(), s["v"][sn].ravel(), s["a"][sn].ravel(),
                                      s["state"][st].astype(np.float64)])
                ops.append(dist.isend(torch.from_numpy(msg), qr))
                rn, rt = pl["recv_nodes"][j], pl["recv_tets"][j]
                rb = torch.empty(9 * len(rn) + len(rt), dtype=torch.float64)
                ops.append(dist.irecv(rb, qr))
                bufs.append((rn, rt, rb))
            for o in ops:
                o.wait()
            u, v, a, stt = s["u"], s["v"], s["a"], s["state"]
            for rn, rt, rb in bufs:
                b = rb.numpy(); n = len(rn)
                u[rn] = b[:3 * n].reshape(-1, 3); v[rn] = b[3 * n:6 * n].reshape(-1, 3)
                a[rn] = b[6 * n:9 * n].reshape(-1, 3); stt[rt] = b[9 * n:].astype(np.uint8)
            orc.set_state(u, v, a)
            orc.set_active(stt)

        exchange()
        for _ in range(60):
            orc.run(1, 1)
            exchange()
        s = orc.state()
        own = pl["node_owned"] == 1
        ot = (pl["tet_flag"] & 2) != 0
        r = orc.records()
        keep = np.isin(r.elem, np.nonzero(ot)[0])
        mine = dict(nodes=ng[own], u=s["u"][own], v=s["v"][own], a=s["a"][own], tets=tg[ot], state=s["state"][ot],
                    rec=(r.step[keep], tg[r.elem[keep]]))
        allp = [None] * world if rank == 0 else None
        dist.gather_object(mine, allp, dst=0)
        if rank == 0:
            glob.run(60, 1)
            gs = glob.state()
            u = np.full((prob.n_nodes, 3), np.nan); st = np.zeros(prob.n_tets, np.uint8)
            steps, elems = [], []
            for m in allp:
                u[m["nodes"]] = m["u"]
                st[m["tets"]] = m["state"]
                steps.append(m["rec"][0]); elems.append(m["rec"][1])
            gr = glob.records()
            el = np.concatenate(elems); sp = np.concatenate(steps)
            order = np.lexsort((el, sp))
            ok = (np.array_equal(u, gs["u"]) and np.array_equal(st, gs["state"]) and
                  np.array_equal(el[order], gr.elem) and len(gr.elem) > 0)
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_single_domain():
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
