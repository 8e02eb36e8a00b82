"""paper_2508_04076_b200 -- B200-native explicit step of the 3D Crack Element Method.

Thin ctypes binding over `libcem.so` (include/cem.h).  Argument marshalling only: every
step of the method runs in the CUDA kernels of `csrc/`.  PyTorch supplies device
memory (the workspace is a torch uint8 tensor) and the CUDA stream.  There is no CPU
fallback: if the extension is missing this module raises at import time.

Names follow the paper (arXiv 2508.04076): ES-FEM edge smoothing domains, energy release
rate G (eq:G-I / eq:G-II), Gc, explicit Newmark (beta = 0, gamma = 1/2).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CEM_LIB") or os.path.join(_HERE, "libcem.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

CEM_OK, CEM_EINVAL, CEM_EDEGENERATE, CEM_ENEGVOL, CEM_ETOPOLOGY, CEM_ENONFINITE, CEM_ECUDA, \
    CEM_ENCCL, CEM_ESTATE, CEM_ENOMEM = range(10)
STATUS_NAMES = ["CEM_OK", "CEM_EINVAL", "CEM_EDEGENERATE", "CEM_ENEGVOL", "CEM_ETOPOLOGY",
                "CEM_ENONFINITE", "CEM_ECUDA", "CEM_ENCCL", "CEM_ESTATE", "CEM_ENOMEM"]
CEM_F_NO_EARLY_OUT = 0x1
CEM_F_STAGED = 0x2
CEM_F_NO_DISCARD = 0x4
CEM_F_PERSISTENT = 0x8
CEM_F_LOOPBACK = 0x10
CEM_F_P2P = 0x20
CEM_F_FRONT_BOTH_STRETCHED = 0x40
CEM_HOST, CEM_DEVICE = 0, 1

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
U8 = C.POINTER(C.c_uint8)


class cem_material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double), ("Gc", C.c_double)]


class cem_mesh_in(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("X", D), ("n_tets", C.c_int64), ("tets", I32),
                ("tet_state", U8), ("tet_gc", D), ("nodes_per_elem", C.c_int32)]


class cem_load_in(C.Structure):
    _fields_ = [("n_tfaces", C.c_int64), ("tface", I32), ("tface_t", D), ("n_vbc", C.c_int64),
                ("vbc_node", I32), ("vbc_mask", U8), ("vbc_v0", D), ("vbc_t0", C.c_double),
                ("f_nodal", D), ("body", C.c_double * 3)]


ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_size_t, C.c_void_p, C.POINTER(C.c_void_p))
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class cem_opts(C.Structure):
    _fields_ = [("dt", C.c_double), ("cfl", C.c_double), ("gamma", C.c_double), ("flags", C.c_uint32),
                ("device", C.c_int), ("stream", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("dev_alloc", ALLOC_FN), ("alloc_user", C.c_void_p),
                ("rank", C.c_int), ("nranks", C.c_int), ("nccl_id", C.c_void_p),
                ("host_allgather", ALLGATHER_FN), ("host_user", C.c_void_p)]


class cem_state_out(C.Structure):
    _fields_ = [("u", D), ("v", D), ("a", D), ("tet_state", U8), ("mass", D),
                ("rec_step", I64), ("rec_elem", I32), ("rec_cand", I32), ("rec_G", D), ("rec_area", D),
                ("rec_capacity", C.c_int64), ("step", C.c_int64), ("time", C.c_double), ("dt", C.c_double),
                ("n_active", C.c_int64), ("n_records", C.c_int64), ("dissipated", C.c_double),
                ("nonfinite", C.c_int32), ("nonfinite_node", C.c_int32)]


class cem_energy_out(C.Structure):
    _fields_ = [("step", C.c_int64), ("time", C.c_double), ("kinetic", C.c_double), ("strain", C.c_double),
                ("external_work", C.c_double), ("reaction_work", C.c_double), ("dissipated", C.c_double)]


_P = C.POINTER
_lib.cem_workspace_size.argtypes = [_P(cem_mesh_in), _P(cem_opts), _P(C.c_size_t)]
_lib.cem_init_mesh.argtypes = [_P(cem_mesh_in), _P(cem_material), _P(cem_load_in), _P(cem_opts),
                               _P(C.c_void_p)]
_lib.cem_step.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
_lib.cem_crack_update.argtypes = [C.c_void_p, I64]
_lib.cem_get_state.argtypes = [C.c_void_p, _P(cem_state_out), C.c_int]
_lib.cem_energy.argtypes = [C.c_void_p, _P(cem_energy_out)]
_lib.cem_set_state.argtypes = [C.c_void_p, _P(cem_state_out)]
_lib.cem_sizes.argtypes = [C.c_void_p, I64, I64, I64]
_lib.cem_launch_count.argtypes = [C.c_void_p]
_lib.cem_launch_count.restype = C.c_int64
_lib.cem_set_profiling.argtypes = [C.c_void_p, C.c_int]
_lib.cem_kernel_times.argtypes = [C.c_void_p, I32, C.POINTER(C.c_char_p), D, C.c_int32]
_lib.cem_last_error.argtypes = [C.c_void_p]
_lib.cem_last_error.restype = C.c_char_p
_lib.cem_destroy.argtypes = [C.c_void_p]
_lib.cem_abi_version.restype = C.c_int32
for _f in ("cem_workspace_size", "cem_init_mesh", "cem_step", "cem_crack_update", "cem_get_state",
           "cem_sizes", "cem_set_profiling", "cem_kernel_times", "cem_energy", "cem_set_state"):
    getattr(_lib, _f).restype = C.c_int

class cem_part_out(C.Structure):
    _fields_ = [("n_tets", C.c_int64), ("n_nodes", C.c_int64), ("tet_global", I32), ("tet_flag", U8),
                ("node_global", I32), ("node_owned", U8), ("n_peers", C.c_int32), ("peers", I32),
                ("send_node_off", I64), ("recv_node_off", I64), ("send_tet_off", I64), ("recv_tet_off", I64),
                ("send_nodes", I32), ("recv_nodes", I32), ("send_tets", I32), ("recv_tets", I32),
                ("tet_owner", I32), ("node_owner", I32)]


_lib.cem_partition.argtypes = [_P(cem_mesh_in), C.c_int, C.c_int, _P(cem_part_out)]
_lib.cem_partition.restype = C.c_int
_lib.cem_partition_free.argtypes = [_P(cem_part_out)]
_lib.cem_nccl_unique_id.argtypes = [C.c_void_p]
_lib.cem_nccl_unique_id.restype = C.c_int
_lib.cem_step_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_int64, C.c_int32]
_lib.cem_step_group.restype = C.c_int
_lib.cem_merge_records.argtypes = [C.c_int64, I64, I32, D, D, I64, D]
_lib.cem_merge_records.restype = C.c_int

EXPORTED = ["cem_workspace_size", "cem_init_mesh", "cem_step", "cem_crack_update", "cem_get_state", "cem_set_state",
            "cem_energy",
            "cem_sizes", "cem_launch_count", "cem_set_profiling", "cem_kernel_times",
            "cem_last_error", "cem_destroy", "cem_abi_version", "cem_partition", "cem_partition_free",
            "cem_nccl_unique_id", "cem_step_group", "cem_merge_records"]


class CemError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _arr(a, dt, shape=None):
    a = np.ascontiguousarray(a, dtype=dt)
    if shape is not None:
        a = a.reshape(shape)
    return a


@dataclass
class State:
    u: np.ndarray
    v: np.ndarray
    a: np.ndarray
    tet_state: np.ndarray
    mass: np.ndarray
    step: int
    time: float
    dt: float
    n_active: int
    dissipated: float
    nonfinite: int
    nonfinite_node: int
    rec_step: np.ndarray
    rec_elem: np.ndarray
    rec_cand: np.ndarray
    rec_G: np.ndarray
    rec_area: np.ndarray


class Simulation:
    """One CEM simulation on one GPU (cem_init_mesh ... cem_destroy)."""

    def __init__(self, X, tets, E, nu, rho, Gc=np.inf, tet_state=None, tet_gc=None,
                 tface=None, tface_t=None, vbc_node=None, vbc_mask=None, vbc_v0=None, vbc_t0=0.0,
                 dt=0.0, cfl=0.5, gamma=0.5, flags=0, device=0, stream=None, use_torch=True,
                 rank=0, nranks=1, nccl_id=None, f_nodal=None, body=(0.0, 0.0, 0.0), host_allgather=None):
        self._h = C.c_void_p()
        keep = []
        # elements: [E,4] linear tets (ES-T-FEM) or [E,8] trilinear hexahedra (ES-H-FEM)
        npe = 8 if np.ndim(tets) == 2 and np.shape(tets)[1] == 8 else 4
        Xa = _arr(X, np.float64, (-1, 3)); Ta = _arr(tets, np.int32, (-1, npe))
        st = None if tet_state is None else _arr(tet_state, np.uint8)
        gc = None if tet_gc is None else _arr(tet_gc, np.float64)
        keep += [Xa, Ta, st, gc]
        mesh = cem_mesh_in(Xa.shape[0], _ptr(Xa, D), Ta.shape[0], _ptr(Ta, I32), _ptr(st, U8), _ptr(gc, D), npe)
        mat = cem_material(E, nu, rho, Gc)
        tf = _arr(np.zeros((0, 3)) if tface is None else tface, np.int32, (-1, 3))
        tt = _arr(np.zeros((0, 3)) if tface_t is None else tface_t, np.float64, (-1, 3))
        vn = _arr(np.zeros(0) if vbc_node is None else vbc_node, np.int32)
        vm = _arr(np.zeros(0) if vbc_mask is None else vbc_mask, np.uint8)
        vv = _arr(np.zeros((0, 3)) if vbc_v0 is None else vbc_v0, np.float64, (-1, 3))
        fn = None if f_nodal is None else _arr(f_nodal, np.float64, (-1, 3))
        keep += [tf, tt, vn, vm, vv, fn]
        load = cem_load_in(tf.shape[0], _ptr(tf, I32), _ptr(tt, D), vn.shape[0], _ptr(vn, I32),
                           _ptr(vm, U8), _ptr(vv, D), vbc_t0, _ptr(fn, D), (C.c_double * 3)(*[float(b) for b in body]))
        self._tensors = []
        self._alloc_cb = None
        self.device = device
        stream_ptr = None
        if use_torch:
            import torch
            dev = torch.device("cuda", device)
            if stream is None:
                # a dedicated non-default stream: CUDA graphs cannot be captured on the
                # legacy default stream
                stream = torch.cuda.Stream(dev)
            self.torch_stream = stream
            stream_ptr = stream.cuda_stream

            def _alloc(nbytes, user, out):
                try:
                    t = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
                    self._tensors.append(t)
                    out[0] = C.c_void_p(t.data_ptr())
                    return 0
                except Exception:  # pragma: no cover - reported through the status code
                    return 1
            self._alloc_cb = ALLOC_FN(_alloc)
        else:
            self.torch_stream = None
            stream_ptr = stream
        self._nccl_id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        self._gather_cb = ALLGATHER_FN()
        if host_allgather is not None:
            # host_allgather(bytes) -> list of nranks bytes objects (rank order), e.g. over gloo
            def _gather(send, recv, nbytes, user):
                try:
                    parts = host_allgather(C.string_at(send, nbytes))
                    blob = b"".join(parts)
                    if len(blob) != nbytes * nranks:
                        return 1
                    C.memmove(recv, blob, len(blob))
                    return 0
                except Exception:  # pragma: no cover - reported through the status code
                    return 1
            self._gather_cb = ALLGATHER_FN(_gather)
        opts = cem_opts(dt, cfl, gamma, flags, device, stream_ptr, None, 0,
                        self._alloc_cb if self._alloc_cb is not None else ALLOC_FN(), None, rank, nranks,
                        None if self._nccl_id is None else C.cast(self._nccl_id, C.c_void_p),
                        self._gather_cb, None)
        self.rank, self.nranks = rank, nranks
        rc = _lib.cem_init_mesh(C.byref(mesh), C.byref(mat), C.byref(load), C.byref(opts), C.byref(self._h))
        if rc != CEM_OK:
            raise CemError(rc, _lib.cem_last_error(None).decode())
        n, e, s = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.cem_sizes(self._h, C.byref(n), C.byref(e), C.byref(s))
        self.n_nodes, self.n_tets, self.n_edges = n.value, e.value, s.value
        # split records: one per element; a hexahedral context also records its remainder tets E + 3e + i
        self.rec_capacity = (4 if npe == 8 else 1) * e.value

    @classmethod
    def from_problem(cls, prob, **kw):
        """Build from a `cem_inputs.Problem`-like object (duck-typed attributes)."""
        return cls(prob.X, prob.tets, prob.E, prob.nu, prob.rho, Gc=prob.Gc, tet_state=prob.tet_state,
                   tet_gc=prob.tet_gc, tface=prob.tface, tface_t=prob.tface_t, vbc_node=prob.vbc_node,
                   vbc_mask=prob.vbc_mask, vbc_v0=prob.vbc_v0, vbc_t0=prob.vbc_t0, dt=prob.dt,
                   cfl=prob.cfl, gamma=prob.gamma, f_nodal=getattr(prob, "f_nodal", None),
                   body=getattr(prob, "body", (0.0, 0.0, 0.0)), **kw)

    def _check(self, rc):
        if rc != CEM_OK:
            raise CemError(rc, _lib.cem_last_error(self._h).decode())

    def step(self, nsteps, crack_every=1):
        self._check(_lib.cem_step(self._h, int(nsteps), int(crack_every)))
        return self

    def crack_update(self):
        n = C.c_int64()
        self._check(_lib.cem_crack_update(self._h, C.byref(n)))
        return n.value

    def set_profiling(self, on=True):
        self._check(_lib.cem_set_profiling(self._h, 1 if on else 0))

    def kernel_times(self):
        n = C.c_int32()
        names = (C.c_char_p * 16)()
        ms = (C.c_double * 16)()
        self._check(_lib.cem_kernel_times(self._h, C.byref(n), names, ms, 16))
        return {names[i].decode(): ms[i] for i in range(n.value)}

    @property
    def launch_count(self):
        """Kernels launched by this simulation so far (cem_launch_count)."""
        return _lib.cem_launch_count(self._h)

    def state(self, records=True, check=True) -> State:
        N, E = self.n_nodes, self.n_tets
        u = np.empty((N, 3)); v = np.empty((N, 3)); a = np.empty((N, 3))
        st = np.empty(E, np.uint8); m = np.empty(N)
        out = cem_state_out()
        out.u, out.v, out.a = _ptr(u, D), _ptr(v, D), _ptr(a, D)
        out.tet_state, out.mass = _ptr(st, U8), _ptr(m, D)
        cap = self.rec_capacity if records else 0
        rs = np.empty(cap, np.int64); re = np.empty(cap, np.int32); rk = np.empty(cap, np.int32)
        rg = np.empty(cap); ra = np.empty(cap)
        out.rec_step, out.rec_elem, out.rec_cand = _ptr(rs, I64), _ptr(re, I32), _ptr(rk, I32)
        out.rec_G, out.rec_area, out.rec_capacity = _ptr(rg, D), _ptr(ra, D), cap
        rc = _lib.cem_get_state(self._h, C.byref(out), CEM_HOST)
        if rc not in (CEM_OK, CEM_ENONFINITE) or (check and rc == CEM_ENONFINITE):
            self._check(rc)
        nr = min(out.n_records, cap)
        return State(u, v, a, st, m, out.step, out.time, out.dt, out.n_active, out.dissipated,
                     out.nonfinite, out.nonfinite_node, rs[:nr], re[:nr], rk[:nr], rg[:nr], ra[:nr])

    def set_state(self, s: State) -> None:
        """cem_set_state: resume from a snapshot of state() (this or another simulation of the same
        mesh, material and loads); the records must be complete (state(records=True))."""
        keep = [_arr(s.u, np.float64, (-1, 3)), _arr(s.v, np.float64, (-1, 3)), _arr(s.a, np.float64, (-1, 3)),
                _arr(s.tet_state, np.uint8), _arr(s.mass, np.float64), _arr(s.rec_step, np.int64),
                _arr(s.rec_elem, np.int32), _arr(s.rec_cand, np.int32), _arr(s.rec_G, np.float64),
                _arr(s.rec_area, np.float64)]
        inp = cem_state_out()
        inp.u, inp.v, inp.a = _ptr(keep[0], D), _ptr(keep[1], D), _ptr(keep[2], D)
        inp.tet_state, inp.mass = _ptr(keep[3], U8), _ptr(keep[4], D)
        inp.rec_step, inp.rec_elem, inp.rec_cand = _ptr(keep[5], I64), _ptr(keep[6], I32), _ptr(keep[7], I32)
        inp.rec_G, inp.rec_area = _ptr(keep[8], D), _ptr(keep[9], D)
        inp.n_records, inp.rec_capacity, inp.step = keep[5].size, keep[5].size, int(s.step)
        self._check(_lib.cem_set_state(self._h, C.byref(inp)))

    def device_state(self, records=True) -> dict:
        """cem_get_state(CEM_DEVICE): torch tensors on the simulation's device, filled by the
        library in the caller's numbering (u, v, a [N,3]; tet_state [E]; mass [N]; records
        sorted by (step, element))."""
        import torch
        dev = torch.device("cuda", self.device)
        N, E = self.n_nodes, self.n_tets
        t = dict(u=torch.empty((N, 3), dtype=torch.float64, device=dev),
                 v=torch.empty((N, 3), dtype=torch.float64, device=dev),
                 a=torch.empty((N, 3), dtype=torch.float64, device=dev),
                 tet_state=torch.empty(E, dtype=torch.uint8, device=dev),
                 mass=torch.empty(N, dtype=torch.float64, device=dev))
        cap = self.rec_capacity if records else 0
        r = dict(rec_step=torch.empty(cap, dtype=torch.int64, device=dev),
                 rec_elem=torch.empty(cap, dtype=torch.int32, device=dev),
                 rec_cand=torch.empty(cap, dtype=torch.int32, device=dev),
                 rec_G=torch.empty(cap, dtype=torch.float64, device=dev),
                 rec_area=torch.empty(cap, dtype=torch.float64, device=dev))
        torch.cuda.synchronize(dev)  # the tensors' allocation is ordered before the library's stream
        out = cem_state_out()
        vp = lambda x, ty: C.cast(C.c_void_p(x.data_ptr()), ty)
        out.u, out.v, out.a = vp(t["u"], D), vp(t["v"], D), vp(t["a"], D)
        out.tet_state, out.mass = vp(t["tet_state"], U8), vp(t["mass"], D)
        if cap:
            out.rec_step, out.rec_elem = vp(r["rec_step"], I64), vp(r["rec_elem"], I32)
            out.rec_cand, out.rec_G, out.rec_area = vp(r["rec_cand"], I32), vp(r["rec_G"], D), vp(r["rec_area"], D)
        out.rec_capacity = cap
        rc = _lib.cem_get_state(self._h, C.byref(out), CEM_DEVICE)
        if rc not in (CEM_OK, CEM_ENONFINITE):
            self._check(rc)
        nr = min(out.n_records, cap)
        t.update({k: v[:nr] for k, v in r.items()})
        t.update(step=out.step, time=out.time, n_active=out.n_active, dissipated=out.dissipated,
                 nonfinite=out.nonfinite)
        return t

    def energy(self) -> dict:
        """Energy ledger at the current step (cem_energy): kinetic, strain, external, reaction,
        dissipated (J)."""
        out = cem_energy_out()
        self._check(_lib.cem_energy(self._h, C.byref(out)))
        return dict(step=out.step, time=out.time, kinetic=out.kinetic, strain=out.strain,
                    external=out.external_work, reaction=out.reaction_work, dissipated=out.dissipated)

    def close(self):
        if self._h:
            _lib.cem_destroy(self._h)
            self._h = C.c_void_p()
        self._tensors = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def workspace_size(X, tets):
    npe = 8 if np.ndim(tets) == 2 and np.shape(tets)[1] == 8 else 4
    Xa = _arr(X, np.float64, (-1, 3)); Ta = _arr(tets, np.int32, (-1, npe))
    mesh = cem_mesh_in(Xa.shape[0], _ptr(Xa, D), Ta.shape[0], _ptr(Ta, I32), None, None, npe)
    b = C.c_size_t()
    rc = _lib.cem_workspace_size(C.byref(mesh), None, C.byref(b))
    if rc:
        raise CemError(rc, _lib.cem_last_error(None).decode())
    return b.value


def abi_version():
    return _lib.cem_abi_version()
