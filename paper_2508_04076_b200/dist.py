"""Multi-GPU driver of the CEM step -- argument marshalling only.

* `partition(prob, nranks, rank)` -- the library's deterministic decomposition plan
  (`cem_partition`): local tets/nodes (ascending global id), masks, exchange lists.
* `DistSimulation` -- one rank per GPU under torchrun: rank 0 asks the library for an NCCL
  unique id, torch.distributed broadcasts it (plumbing), every rank calls `cem_init_mesh`
  with nranks > 1; `cem_step` then runs the three stage kernels plus the NCCL halo exchange
  per step on the rank's stream.
* `LoopbackGroup` -- P ranks emulated in one process on one device (`CEM_F_LOOPBACK`,
  `cem_step_group`): the same kernels, masks and pack/unpack, with device copies as the
  transport.  Used to test the multi-rank path on a single B200.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import (CEM_F_LOOPBACK, CEM_OK, D, I32, I64, U8, CemError, Simulation, _arr, _lib, _ptr, cem_mesh_in,
               cem_part_out)


def partition(X, tets, nranks, rank):
    """Decomposition plan of `rank` (dict of numpy arrays; local ids index the local mesh)."""
    Xa = _arr(X, np.float64, (-1, 3)); Ta = _arr(tets, np.int32, (-1, 4))
    mesh = cem_mesh_in(Xa.shape[0], _ptr(Xa, D), Ta.shape[0], _ptr(Ta, I32), None, None)
    o = cem_part_out()
    rc = _lib.cem_partition(C.byref(mesh), int(nranks), int(rank), C.byref(o))
    if rc != CEM_OK:
        raise CemError(rc, _lib.cem_last_error(None).decode())
    try:
        def a(p, n, dt):
            return np.ctypeslib.as_array(p, shape=(int(n),)).astype(dt, copy=True) if n else np.zeros(0, dt)
        npeer = o.n_peers
        out = dict(tet_global=a(o.tet_global, o.n_tets, np.int32), tet_flag=a(o.tet_flag, o.n_tets, np.uint8),
                   node_global=a(o.node_global, o.n_nodes, np.int32), node_owned=a(o.node_owned, o.n_nodes, np.uint8),
                   peers=a(o.peers, npeer, np.int32), tet_owner=a(o.tet_owner, Ta.shape[0], np.int32),
                   node_owner=a(o.node_owner, Xa.shape[0], np.int32))
        for name in ("send_node", "recv_node", "send_tet", "recv_tet"):
            off = a(getattr(o, name + "_off"), npeer + 1, np.int64)
            flat = a(getattr(o, name + "s"), off[-1] if npeer else 0, np.int32)
            out[name + "s"] = [flat[off[j]:off[j + 1]] for j in range(npeer)]
        return out
    finally:
        _lib.cem_partition_free(C.byref(o))


def merge_records(steps, elems, areas, gc):
    """Order records by (step, element) and sum U_d in that order (cem_merge_records)."""
    n = len(steps)
    st = _arr(steps, np.int64); el = _arr(elems, np.int32); ar = _arr(areas, np.float64); g = _arr(gc, np.float64)
    order = np.empty(n, np.int64); ud = C.c_double()
    rc = _lib.cem_merge_records(n, _ptr(st, I64), _ptr(el, I32), _ptr(ar, D), _ptr(g, D), _ptr(order, I64),
                                C.byref(ud))
    if rc != CEM_OK:
        raise CemError(rc, "cem_merge_records")
    return order, ud.value


def _assemble(prob, parts, states):
    """Global state from the ranks' local states: owned nodes and owned tets."""
    N, E = prob.n_nodes, prob.n_tets
    u = np.zeros((N, 3)); v = np.zeros((N, 3)); a = np.zeros((N, 3)); m = np.zeros(N)
    st = np.zeros(E, np.uint8)
    rs, re, rk, rg, ra = [], [], [], [], []
    for pl, s in zip(parts, states):
        own = pl["node_owned"] == 1
        g = pl["node_global"][own]
        u[g] = s.u[own]; v[g] = s.v[own]; a[g] = s.a[own]; m[g] = s.mass[own]
        ot = (pl["tet_flag"] & 2) != 0
        st[pl["tet_global"][ot]] = s.tet_state[ot]
        rs.append(s.rec_step); re.append(s.rec_elem); rk.append(s.rec_cand); rg.append(s.rec_G); ra.append(s.rec_area)
    rs, re, rk, rg, ra = (np.concatenate(x) for x in (rs, re, rk, rg, ra))
    order, ud = merge_records(rs, re, ra, prob.tet_gc)
    return dict(u=u, v=v, a=a, mass=m, tet_state=st, rec_step=rs[order], rec_elem=re[order], rec_cand=rk[order],
                rec_G=rg[order], rec_area=ra[order], dissipated=ud)


class LoopbackGroup:
    """nranks sub-domain contexts on one device, stepped together (cem_step_group)."""

    def __init__(self, prob, nranks, flags=0, device=0, **kw):
        import torch
        self.prob, self.nranks = prob, nranks
        self.parts = [partition(prob.X, prob.tets, nranks, r) for r in range(nranks)]
        stream = torch.cuda.Stream(torch.device("cuda", device))
        self.sims = [Simulation.from_problem(prob, flags=flags | CEM_F_LOOPBACK, device=device, stream=stream,
                                             rank=r, nranks=nranks, **kw) for r in range(nranks)]
        self._arr = (C.c_void_p * nranks)(*[s._h.value for s in self.sims])
        self.torch_stream = stream

    def step(self, nsteps, crack_every=1):
        rc = _lib.cem_step_group(self._arr, self.nranks, int(nsteps), int(crack_every))
        if rc != CEM_OK:
            raise CemError(rc, _lib.cem_last_error(self.sims[0]._h).decode())
        return self

    def state(self):
        return _assemble(self.prob, self.parts, [s.state() for s in self.sims])

    @property
    def launch_count(self):
        return sum(s.launch_count for s in self.sims)

    def energy(self):
        """Energy ledger of the whole mesh: the sum of the ranks' shares (cem_energy)."""
        parts = [s.energy() for s in self.sims]
        out = dict(parts[0])
        for k in ("kinetic", "strain", "external", "reaction", "dissipated"):
            out[k] = sum(p[k] for p in parts)
        return out


class DistSimulation:
    """One rank of a torchrun job (one GPU per rank, NCCL halo exchange inside cem_step)."""

    def __init__(self, prob, device=0, transport="nccl", **kw):
        """transport "nccl": NCCL communicator (+ the NVLink P2P halo when every rank can map its
        peers); "host_ipc": no NCCL -- CUDA-IPC receive buffers whose handles, and a per-step host
        rendezvous, go through torch.distributed on the CPU (gloo works; ranks may share a GPU)."""
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()
        self.prob = prob
        if transport == "host_ipc":
            import torch

            def allgather(blob):
                t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
                out = [torch.empty_like(t) for _ in range(self.nranks)]
                dist.all_gather(out, t)
                return [bytes(x.numpy().tobytes()) for x in out]
            self.part = partition(prob.X, prob.tets, self.nranks, self.rank)
            self.sim = Simulation.from_problem(prob, device=device, rank=self.rank, nranks=self.nranks,
                                               host_allgather=allgather, **kw)
            self.torch_stream = self.sim.torch_stream
            self.n_tets_owned = int(((self.part["tet_flag"] & 2) != 0).sum())
            return
        buf = [None]
        if self.rank == 0:
            idb = C.create_string_buffer(128)
            rc = _lib.cem_nccl_unique_id(C.cast(idb, C.c_void_p))
            if rc != CEM_OK:
                raise CemError(rc, _lib.cem_last_error(None).decode())
            buf[0] = idb.raw
        dist.broadcast_object_list(buf, src=0)
        self.part = partition(prob.X, prob.tets, self.nranks, self.rank)
        self.sim = Simulation.from_problem(prob, device=device, rank=self.rank, nranks=self.nranks,
                                           nccl_id=buf[0], **kw)
        self.torch_stream = self.sim.torch_stream
        self.n_tets_owned = int(((self.part["tet_flag"] & 2) != 0).sum())

    def step(self, nsteps, crack_every=1):
        self.sim.step(nsteps, crack_every)
        return self

    @property
    def launch_count(self):
        return self.sim.launch_count

    def energy(self):
        """Energy ledger of the whole mesh (the ranks' shares summed with all_reduce); every rank
        gets the same dict."""
        import torch
        e = self.sim.energy()
        keys = ("kinetic", "strain", "external", "reaction", "dissipated")
        t = torch.tensor([e[k] for k in keys], dtype=torch.float64, device=f"cuda:{self.sim.device}")
        self.dist.all_reduce(t)
        out = dict(e)
        out.update({k: float(v) for k, v in zip(keys, t.tolist())})
        return out

    def state(self, gather=True):
        """Local state; with gather=True rank 0 returns the assembled global state (others None)."""
        s = self.sim.state()
        if not gather:
            return s
        allp = [None] * self.nranks if self.rank == 0 else None
        self.dist.gather_object((self.part, s), allp, dst=0)
        if self.rank != 0:
            return None
        return _assemble(self.prob, [p for p, _ in allp], [x for _, x in allp])
