"""CPU oracle for the CEM explicit step -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and bench.py's `cpu_baseline` / `--impl
reference` legs may import this package.  The product package
`paper_2508_04076_b200` never imports it and shares no code with it.

`liboracle.so` is built from `cem_oracle.c` (plain C99 + OpenMP, -ffp-contract=off).
`l0_literal.py` is the literal assembled-B̃ form of PAPER.md eq:strain_discretization /
eq:fint_discretization used to pin the factored C form.

Parity status per function: every function here is pinned by a
`-m "not gpu"` test; none is "parity unpinned" except the whole-run crack pattern vs the
paper's figures (no paper data exists).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "cem_oracle.c")
_SRC_HEX = os.path.join(_HERE, "cem_oracle_hex.c")
_HDR_XS = os.path.join(_HERE, "exact_sum.h")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(_SRC),
                                                                           os.path.getmtime(_SRC_HEX),
                                                                           os.path.getmtime(_HDR_XS)):
        tmp = _SO + ".tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SRC_HEX, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
U8 = C.POINTER(C.c_uint8)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_int64, D, C.c_int64, I32, U8, D, C.c_double, C.c_double, C.c_double,
                                 C.c_int64, I32, D, C.c_int64, I32, U8, D, C.c_double, C.c_double,
                                 C.c_double, C.c_double, D, D, C.c_uint32, C.c_char_p, C.c_int]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_run.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.orc_run.restype = C.c_int
        for f in ("orc_n_edges", "orc_step_count", "orc_n_records"):
            getattr(L, f).argtypes = [C.c_void_p]; getattr(L, f).restype = C.c_int64
        for f in ("orc_dt", "orc_dissipated"):
            getattr(L, f).argtypes = [C.c_void_p]; getattr(L, f).restype = C.c_double
        L.orc_get_state.argtypes = [C.c_void_p, D, D, D, U8, D]
        L.orc_get_records.argtypes = [C.c_void_p, I64, I32, I32, D, D]
        L.orc_get_fext.argtypes = [C.c_void_p, D]
        L.orc_get_geometry.argtypes = [C.c_void_p, D, D]
        L.orc_get_edges.argtypes = [C.c_void_p, I32, I64]
        L.orc_set_state.argtypes = [C.c_void_p, D, D, D]
        L.orc_set_active.argtypes = [C.c_void_p, U8]
        L.orc_edge_stress.argtypes = [C.c_void_p, D, D, D]
        L.orc_internal_force.argtypes = [C.c_void_p, D, D]
        L.orc_strain_energy.argtypes = [C.c_void_p, D]; L.orc_strain_energy.restype = C.c_double
        L.orc_criterion.argtypes = [C.c_void_p, D, D, I32, D, U8]
        L.orc_candidates.argtypes = [C.c_void_p, D, C.c_int64, D, D]
        L.orc_principal.argtypes = [D, D, D, I32, I32]
        L.orc_tet_geometry.argtypes = [D, D, D]
        L.orc_sig_proj.argtypes = [D, D]; L.orc_sig_proj.restype = C.c_double
        L.orc_exact_sum.argtypes = [C.c_int64, D]; L.orc_exact_sum.restype = C.c_double
        L.orc_element_forces.argtypes = [C.c_void_p, D]
        L.orc_lame.argtypes = [C.c_double, C.c_double, D, D]
        L.orc_lame_of.argtypes = [C.c_void_p, D, D]
        L.orc_newmark_free.argtypes = [C.c_int64, D, D, D, D, D, C.c_double, C.c_double]
        L.orc_predict.argtypes = [C.c_int64, D, D, D, C.c_double]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_energy.argtypes = [C.c_void_p, D]
        # ES-H-FEM hexahedra (cem_oracle_hex.c)
        L.hx_create.restype = C.c_void_p
        L.hx_create.argtypes = [C.c_int64, D, C.c_int64, I32, U8, C.c_double, C.c_double, C.c_double,
                                C.c_int64, I32, D, C.c_int64, I32, U8, D, C.c_double, C.c_double, C.c_double,
                                C.c_double, D, D, D, C.c_uint32, C.c_char_p, C.c_int]
        L.hx_destroy.argtypes = [C.c_void_p]
        L.hx_run.argtypes = [C.c_void_p, C.c_int64, C.c_int32]; L.hx_run.restype = C.c_int
        for f in ("hx_n_edges", "hx_n_edges_all", "hx_n_records"):
            getattr(L, f).argtypes = [C.c_void_p]; getattr(L, f).restype = C.c_int64
        L.hx_dissipated.argtypes = [C.c_void_p]; L.hx_dissipated.restype = C.c_double
        L.hx_get_records.argtypes = [C.c_void_p, I64, I32, I32, D, D]
        L.hx_get_elements.argtypes = [C.c_void_p, U8, U8, I32, D]
        L.hx_candidates.argtypes = [C.c_void_p, D, C.c_int64, D, D, I32]
        L.hx_force_split.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.hx_edge_stress_all.argtypes = [C.c_void_p, D, D, D, I32]
        L.orc_tet_cand_x.argtypes = [D, D, D, C.c_uint32, D, D]
        L.hx_dt.argtypes = [C.c_void_p]; L.hx_dt.restype = C.c_double
        L.hx_get_state.argtypes = [C.c_void_p, D, D, D, D]
        L.hx_get_fext.argtypes = [C.c_void_p, D]
        L.hx_get_geometry.argtypes = [C.c_void_p, D, D]
        L.hx_edge_stress.argtypes = [C.c_void_p, D, D, D, I32]
        L.hx_internal_force.argtypes = [C.c_void_p, D, D]
        L.hx_strain_energy.argtypes = [C.c_void_p, D]; L.hx_strain_energy.restype = C.c_double
        L.hx_set_state.argtypes = [C.c_void_p, D, D, D]
        L.hx_geometry.argtypes = [D, D, D]; L.hx_geometry.restype = C.c_int
        _lib = L
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


@dataclass
class Records:
    step: np.ndarray
    elem: np.ndarray
    cand: np.ndarray
    G: np.ndarray
    area: np.ndarray


class Oracle:
    """One oracle simulation (mirrors the product's cem_init_mesh / cem_step semantics)."""

    # criterion variant flag (R11; the product's CEM_F_FRONT_BOTH_STRETCHED has the same value)
    FRONT_BOTH_STRETCHED = 0x40

    def __init__(self, prob, dt=None, flags=0):
        L = lib()
        self.prob = prob
        self._keep = [
            _c(prob.X, np.float64), _c(prob.tets, np.int32), _c(prob.tet_state, np.uint8),
            _c(prob.tet_gc, np.float64), _c(prob.tface, np.int32), _c(prob.tface_t, np.float64),
            _c(prob.vbc_node, np.int32), _c(prob.vbc_mask, np.uint8), _c(prob.vbc_v0, np.float64),
        ]
        X, T, st, gc, tf, tt, vn, vm, vv = self._keep
        fn = getattr(prob, "f_nodal", None)
        fn = None if fn is None else _c(fn, np.float64).reshape(-1, 3)
        body = _c(getattr(prob, "body", (0.0, 0.0, 0.0)), np.float64)
        self._keep += [fn, body]
        err = C.create_string_buffer(256)
        self.N, self.E = prob.n_nodes, prob.n_tets
        self.h = L.orc_create(self.N, _p(X, D), self.E, _p(T, I32), _p(st, U8), _p(gc, D),
                              prob.E, prob.nu, prob.rho, tf.shape[0], _p(tf, I32), _p(tt, D),
                              vn.shape[0], _p(vn, I32), _p(vm, U8), _p(vv, D), prob.vbc_t0,
                              prob.dt if dt is None else dt, prob.cfl, prob.gamma, _p(fn, D), _p(body, D),
                              int(flags), err, 256)
        if not self.h:
            raise ValueError("oracle rejected the mesh: " + err.value.decode())
        self.S = L.orc_n_edges(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    @property
    def dt(self):
        return lib().orc_dt(self.h)

    @property
    def step_count(self):
        return lib().orc_step_count(self.h)

    @property
    def dissipated(self):
        return lib().orc_dissipated(self.h)

    def lame(self):
        lam, mu = C.c_double(), C.c_double()
        lib().orc_lame_of(self.h, C.byref(lam), C.byref(mu))
        return lam.value, mu.value

    def run(self, nsteps, crack_every=1):
        rc = lib().orc_run(self.h, int(nsteps), int(crack_every))
        if rc:
            raise FloatingPointError("oracle: non-finite state")
        return self

    def state(self):
        u = np.empty((self.N, 3)); v = np.empty((self.N, 3)); a = np.empty((self.N, 3))
        st = np.empty(self.E, np.uint8); m = np.empty(self.N)
        lib().orc_get_state(self.h, _p(u, D), _p(v, D), _p(a, D), _p(st, U8), _p(m, D))
        return dict(u=u, v=v, a=a, state=st, m=m)

    def set_state(self, u=None, v=None, a=None):
        u = None if u is None else _c(u, np.float64)
        v = None if v is None else _c(v, np.float64)
        a = None if a is None else _c(a, np.float64)
        lib().orc_set_state(self.h, _p(u, D), _p(v, D), _p(a, D))

    def set_active(self, state):
        st = _c(state, np.uint8)
        lib().orc_set_active(self.h, _p(st, U8))

    def records(self):
        n = lib().orc_n_records(self.h)
        r = Records(np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n), np.empty(n))
        lib().orc_get_records(self.h, _p(r.step, I64), _p(r.elem, I32), _p(r.cand, I32), _p(r.G, D), _p(r.area, D))
        return r

    def fext(self):
        f = np.empty((self.N, 3)); lib().orc_get_fext(self.h, _p(f, D)); return f

    def geometry(self):
        V = np.empty(self.E); g = np.empty((self.E, 4, 3))
        lib().orc_get_geometry(self.h, _p(V, D), _p(g, D)); return V, g

    def edges(self):
        en = np.empty((self.S, 2), np.int32); cnt = np.empty(self.S, np.int64)
        lib().orc_get_edges(self.h, _p(en, I32), _p(cnt, I64)); return en, cnt

    def edge_stress(self, u):
        u = _c(u, np.float64); s = np.empty((self.S, 6)); vh = np.empty(self.S)
        lib().orc_edge_stress(self.h, _p(u, D), _p(s, D), _p(vh, D)); return s, vh

    def internal_force(self, u):
        u = _c(u, np.float64); f = np.empty((self.N, 3))
        lib().orc_internal_force(self.h, _p(u, D), _p(f, D)); return f

    def element_forces(self):
        """f_{e,a} [E][4][3] of the last internal_force call"""
        fe = np.empty((self.E, 4, 3)); lib().orc_element_forces(self.h, _p(fe, D)); return fe

    def strain_energy(self, u):
        u = _c(u, np.float64); return lib().orc_strain_energy(self.h, _p(u, D))

    def criterion(self, u):
        u = _c(u, np.float64)
        G = np.empty(self.E); k = np.empty(self.E, np.int32); A = np.empty(self.E); fl = np.empty(self.E, np.uint8)
        lib().orc_criterion(self.h, _p(u, D), _p(G, D), _p(k, I32), _p(A, D), _p(fl, U8))
        return G, k, A, fl

    def energy(self):
        """Energy ledger at the current step: kinetic, strain, external, reaction, dissipated."""
        out = np.empty(5)
        lib().orc_energy(self.h, _p(out, D))
        return dict(kinetic=out[0], strain=out[1], external=out[2], reaction=out[3], dissipated=out[4])

    def candidates(self, u, e):
        u = _c(u, np.float64); G = np.empty(24); A = np.empty(24)
        lib().orc_candidates(self.h, _p(u, D), int(e), _p(G, D), _p(A, D)); return G, A


class HexOracle:
    """ES-H-FEM oracle on trilinear hexahedra (cem_oracle_hex.c): elastodynamics and crack patterns
    III-VI with triangular-prism remainders (readings R23-R29)."""

    def __init__(self, prob, dt=None, flags=0):
        L = lib()
        self.prob = prob
        fn = getattr(prob, "f_nodal", None)
        fn = None if fn is None else _c(fn, np.float64).reshape(-1, 3)
        self._keep = [_c(prob.X, np.float64), _c(prob.tets, np.int32), _c(prob.tet_state, np.uint8),
                      _c(prob.tface, np.int32), _c(prob.tface_t, np.float64), _c(prob.vbc_node, np.int32),
                      _c(prob.vbc_mask, np.uint8), _c(prob.vbc_v0, np.float64), fn,
                      _c(getattr(prob, "body", (0.0, 0.0, 0.0)), np.float64),
                      _c(getattr(prob, "tet_gc", np.full(prob.tets.shape[0], np.inf)), np.float64)]
        X, H, st, tf, tt, vn, vm, vv, fn, body, gc = self._keep
        err = C.create_string_buffer(256)
        self.N, self.E = X.shape[0], H.shape[0]
        self.h = L.hx_create(self.N, _p(X, D), self.E, _p(H, I32), _p(st, U8), prob.E, prob.nu, prob.rho,
                             tf.shape[0], _p(tf, I32), _p(tt, D), vn.shape[0], _p(vn, I32), _p(vm, U8), _p(vv, D),
                             prob.vbc_t0, prob.dt if dt is None else dt, prob.cfl, prob.gamma, _p(fn, D),
                             _p(body, D), _p(gc, D), int(flags), err, 256)
        if not self.h:
            raise ValueError("hex oracle rejected the mesh: " + err.value.decode())
        self.S = L.hx_n_edges(self.h)
        self.S_all = L.hx_n_edges_all(self.h)
        self.step_count = 0

    def __del__(self):
        if getattr(self, "h", None):
            lib().hx_destroy(self.h)
            self.h = None

    @property
    def dt(self):
        return lib().hx_dt(self.h)

    def run(self, nsteps, crack_every=0):
        rc = lib().hx_run(self.h, int(nsteps), int(crack_every))
        self.step_count += int(nsteps)
        if rc:
            raise FloatingPointError("hex oracle: non-finite state")
        return self

    @property
    def dissipated(self):
        return lib().hx_dissipated(self.h)

    def records(self):
        n = lib().hx_n_records(self.h)
        r = Records(np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n), np.empty(n))
        lib().hx_get_records(self.h, _p(r.step, I64), _p(r.elem, I32), _p(r.cand, I32), _p(r.G, D), _p(r.area, D))
        return r

    def elements(self):
        """hex_active [E], tet_active [E,3], tet_nodes [E,3,4] (global; -1 without remainder), tet V [E,3]"""
        ha = np.empty(self.E, np.uint8); ta = np.empty((self.E, 3), np.uint8)
        tn = np.empty((self.E, 3, 4), np.int32); tv = np.empty((self.E, 3))
        lib().hx_get_elements(self.h, _p(ha, U8), _p(ta, U8), _p(tn, I32), _p(tv, D))
        return dict(hex_active=ha, tet_active=ta, tet_nodes=tn, tet_V=tv)

    def candidates(self, u, e):
        """G [84], area [84], remainder prism local nodes [84, 6] (-1: none) of hex e for u"""
        u = _c(u, np.float64); G = np.empty(84); A = np.empty(84); P = np.empty((84, 6), np.int32)
        lib().hx_candidates(self.h, _p(u, D), int(e), _p(G, D), _p(A, D), _p(P, I32)); return G, A, P

    def force_split(self, e, k):
        lib().hx_force_split(self.h, int(e), int(k))

    def edge_stress_all(self, u):
        u = _c(u, np.float64); S = self.S_all
        s = np.empty((S, 6)); vh = np.empty(S); en = np.empty((S, 2), np.int32)
        lib().hx_edge_stress_all(self.h, _p(u, D), _p(s, D), _p(vh, D), _p(en, I32)); return s, vh, en

    def state(self):
        u = np.empty((self.N, 3)); v = np.empty((self.N, 3)); a = np.empty((self.N, 3)); m = np.empty(self.N)
        lib().hx_get_state(self.h, _p(u, D), _p(v, D), _p(a, D), _p(m, D))
        return dict(u=u, v=v, a=a, m=m)

    def set_state(self, u=None, v=None, a=None):
        u = None if u is None else _c(u, np.float64)
        v = None if v is None else _c(v, np.float64)
        a = None if a is None else _c(a, np.float64)
        lib().hx_set_state(self.h, _p(u, D), _p(v, D), _p(a, D))

    def fext(self):
        f = np.empty((self.N, 3)); lib().hx_get_fext(self.h, _p(f, D)); return f

    def geometry(self):
        V = np.empty(self.E); g = np.empty((self.E, 8, 3))
        lib().hx_get_geometry(self.h, _p(V, D), _p(g, D)); return V, g

    def edge_stress(self, u):
        u = _c(u, np.float64); s = np.empty((self.S, 6)); vh = np.empty(self.S); en = np.empty((self.S, 2), np.int32)
        lib().hx_edge_stress(self.h, _p(u, D), _p(s, D), _p(vh, D), _p(en, I32)); return s, vh, en

    def internal_force(self, u):
        u = _c(u, np.float64); f = np.empty((self.N, 3))
        lib().hx_internal_force(self.h, _p(u, D), _p(f, D)); return f

    def strain_energy(self, u):
        u = _c(u, np.float64); return lib().hx_strain_energy(self.h, _p(u, D))


def hex_geometry(X8):
    """(V, grad [8,3]) of one hexahedron, or None if its Jacobian is not positive."""
    X8 = _c(X8, np.float64); V = C.c_double(); g = np.empty((8, 3))
    ok = lib().hx_geometry(_p(X8, D), C.byref(V), _p(g, D))
    return (V.value, g) if ok else None


def principal(s6):
    s6 = _c(s6, np.float64); lam = np.empty(3); vec = np.empty((3, 3))
    k1 = C.c_int32(); deg = C.c_int32()
    lib().orc_principal(_p(s6, D), _p(lam, D), _p(vec, D), C.byref(k1), C.byref(deg))
    return lam, vec, k1.value, deg.value


def exact_sum(x):
    """The oracle's nodal-assembly sum (R27): exact sum of the doubles, rounded once."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().orc_exact_sum(x.size, _p(x, D))


def sig_proj(s6, m):
    """sigma_G . m (unnormalised m) of the stress s6, R8."""
    s6 = _c(s6, np.float64); m = _c(m, np.float64)
    return lib().orc_sig_proj(_p(s6, D), _p(m, D))


def tet_geometry(X4):
    X4 = _c(X4, np.float64); V = C.c_double(); g = np.empty((4, 3))
    lib().orc_tet_geometry(_p(X4, D), C.byref(V), _p(g, D)); return V.value, g


def lame(E, nu):
    lam, mu = C.c_double(), C.c_double()
    lib().orc_lame(E, nu, C.byref(lam), C.byref(mu)); return lam.value, mu.value


def newmark_free(m, fext, fint, v, a, dt, gamma=0.5):
    m, fext, fint = _c(m, np.float64), _c(fext, np.float64), _c(fint, np.float64)
    v = _c(v, np.float64).copy(); a = _c(a, np.float64).copy()
    lib().orc_newmark_free(m.size, _p(m, D), _p(fext, D), _p(fint, D), _p(v, D), _p(a, D), dt, gamma)
    return v, a


def predict(u, v, a, dt):
    u = _c(u, np.float64).copy(); v = _c(v, np.float64); a = _c(a, np.float64)
    lib().orc_predict(u.size, _p(u, D), _p(v, D), _p(a, D), dt); return u


def num_threads():
    return lib().orc_num_threads()


def set_threads(n):
    """OpenMP threads of subsequent oracle calls (bench.py's single-thread baseline)."""
    lib().orc_set_threads(int(n))
