"""The bounds-checked debug build (libcem_dbg.so, -DCEM_DEBUG_BOUNDS: every gathered index of the
stage kernels and the criterion lists checked against its table or shared-memory extent) runs the
representative paths with no violation and the same bits as the oracle.  compute-sanitizer is closed
on this GPU pool; this stands in for its memcheck."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_bounds_build_runs_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2508_04076_b200", "libcem_dbg.so")
    if not os.path.exists(lib):
        pytest.skip("libcem_dbg.so not built")
    env = dict(os.environ, CEM_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    for tag in ("staged", "long-list", "wave", "loopback P=3 flags=0", "loopback P=3 flags=32", "crack update",
                "hex"):
        assert tag in r.stdout, (tag, r.stdout)
