import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long CPU test")
    # a fresh checkout has no built artefacts (*.so are git-ignored): build them once (nvcc
    # cross-compiles for sm_100a without a GPU)
    if not os.path.exists(os.path.join(ROOT, "paper_2508_04076_b200", "libcem.so")) and not os.environ.get("CEM_LIB"):
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def cfg0():
    import cem_inputs
    return cem_inputs.config(0)
