"""C-ABI boundary checks that need no GPU: libcem.so loads, exports every symbol that
include/cem.h declares, and host-side validation returns the documented status codes
(cem_init_mesh validates before touching the device)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import cem_inputs as ci

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cem.h")).read()
    return sorted(set(re.findall(r"CEM_API\s+[\w\s\*]+?\b(cem_\w+)\s*\(", src)))


def test_header_declares_abi():
    syms = declared_symbols()
    for s in ["cem_init_mesh", "cem_step", "cem_crack_update", "cem_get_state", "cem_workspace_size",
              "cem_last_error", "cem_destroy"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_2508_04076_b200 as cem
    out = subprocess.check_output(["nm", "-D", "--defined-only", cem.LIB_PATH]).decode()
    exported = set(re.findall(r" T (cem_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(cem.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert set(cem.EXPORTED) == set(declared_symbols())
    assert cem.abi_version() == 2


def test_library_is_sm100a():
    import paper_2508_04076_b200 as cem
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cem.LIB_PATH]).decode()
    assert "sm_100a" in out


def _sim(prob, **kw):
    import paper_2508_04076_b200 as cem
    return cem.Simulation(prob.X, prob.tets, prob.E, prob.nu, prob.rho, tet_state=prob.tet_state,
                          tet_gc=prob.tet_gc, use_torch=False, **kw)


def _status(fn):
    import paper_2508_04076_b200 as cem
    with pytest.raises(cem.CemError) as ei:
        fn()
    return ei.value.status


def test_validation_errors():
    import paper_2508_04076_b200 as cem
    p = ci.notched_plate(cells=(3, 2, 1), dims=(0.03, 0.02, 0.01), seed=1, steps=0)
    bad = ci.make_problem(p.X, p.tets[:, [0, 1, 3, 2]])                # flipped orientation
    assert _status(lambda: _sim(bad)) == cem.CEM_ENEGVOL
    dup = ci.make_problem(p.X, np.concatenate([p.tets, p.tets[:1, [1, 0, 3, 2]]]))
    assert _status(lambda: _sim(dup)) == cem.CEM_ETOPOLOGY
    oob = ci.make_problem(p.X, np.where(p.tets == 0, p.n_nodes + 5, p.tets))
    assert _status(lambda: _sim(oob)) == cem.CEM_ETOPOLOGY
    rep = ci.make_problem(p.X, np.concatenate([p.tets, [[0, 0, 1, 2]]]))
    assert _status(lambda: _sim(rep)) == cem.CEM_ETOPOLOGY
    X = p.X.copy(); X[:, 2] = 0.0                                         # flat mesh
    assert _status(lambda: _sim(ci.make_problem(X, p.tets))) in (cem.CEM_EDEGENERATE, cem.CEM_ENEGVOL)
    assert _status(lambda: _sim(ci.make_problem(p.X, p.tets, nu=0.5))) == cem.CEM_EINVAL
    assert _status(lambda: _sim(ci.make_problem(p.X, p.tets, E=-1.0))) == cem.CEM_EINVAL
    none_active = ci.make_problem(p.X, p.tets, tet_state=np.zeros(p.n_tets, np.uint8))
    assert _status(lambda: _sim(none_active)) == cem.CEM_EINVAL      # no active tet to derive dt from


def test_workspace_size_counts_edges():
    import paper_2508_04076_b200 as cem
    p = ci.config(0)
    b = cem.workspace_size(p.X, p.tets)
    # at least the edge stress field (6 doubles per edge) and the element tables
    assert b > 2918 * 48 + 1920 * (16 * 8 + 24 + 48 + 96)


def test_maximum_size_rejected_before_reading():
    """Meshes beyond one context's 32-bit index ranges (E >= 2^32/12 - 64 tets or N >= 2^31
    nodes) are rejected with CEM_EINVAL before any array is read (include/cem.h)."""
    import ctypes as C
    import paper_2508_04076_b200 as cem
    X = np.zeros((4, 3)); T = np.array([[0, 1, 2, 3]], np.int32)
    for n_nodes, n_tets in ((4, (1 << 32) // 12), (1 << 31, 1)):
        mesh = cem.cem_mesh_in(n_nodes, X.ctypes.data_as(C.POINTER(C.c_double)), n_tets,
                               T.ctypes.data_as(C.POINTER(C.c_int32)), None, None)
        b = C.c_size_t()
        assert cem._lib.cem_workspace_size(C.byref(mesh), None, C.byref(b)) == cem.CEM_EINVAL


def test_set_state_null_arguments():
    """cem_set_state validates its arguments before touching a context (no GPU needed)."""
    import paper_2508_04076_b200 as cem
    assert cem._lib.cem_set_state(None, None) == cem.CEM_EINVAL
