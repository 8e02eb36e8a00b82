"""The "fast build" (device FMA contraction, libcem_fast.so built by __graft_entry__.build()) meets
the north star's gate against the oracle instead of bit equality: relative L2 of u <= 1e-11 per
1000 steps and an identical split set (SURVEY.md §8(c) "Parity protocol", BASELINE.json north_star).
Configs 0 (200 steps), 1 (1000 steps) and 3 (300 steps; 1000 with CEM_LONG_TESTS=1), crack check
every step (the oracle's run time sets the test's)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fast_build_north_star_gate():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2508_04076_b200", "libcem_fast.so")
    if not os.path.exists(lib):
        pytest.skip("libcem_fast.so not built")
    cases = ["0:200", "1:1000", "3:1000" if os.environ.get("CEM_LONG_TESTS") == "1" else "3:300"]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fast_build_check.py")] + cases,
                       env=dict(os.environ, CEM_LIB=lib), cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(rows) == 3
    for row in rows:
        assert row["lib"] == "libcem_fast.so"
        assert row["rel_l2_u"] <= 1e-11, row
        assert row["same_split_set"] and row["same_split_steps"], row
        assert row["splits"] > 0, row
