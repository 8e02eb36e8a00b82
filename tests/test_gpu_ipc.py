"""The real multi-process halo path on one GPU (round-1 review item): two OS processes, each a
rank with its own CUDA context on cuda:0, map each other's receive buffers with
cudaIpcOpenMemHandle, store into them from stage D and the split pass, signal with
st.release.sys and consume with ld.acquire.sys + unpack -- bitwise equal to the single-domain
oracle on config 0 and on a compact-tension case.

The per-step rendezvous is on the host (opts.host_allgather over gloo), after each rank's stores
have completed, so the device flag wait finds its flags already set and never spins: two
processes' kernels that spin on each other on ONE GPU are not guaranteed to be co-scheduled
(/opt/skills/guides/B200_PROFILING.md: such runs raised Xid 109).  The NCCL / spinning NVLink
path needs one GPU per rank."""
import json
import os
import signal
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case,steps", [("cfg0", 200), ("ct", 250)])
def test_two_processes_cuda_ipc_halo_bitwise(case, steps, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "verdict.json"
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_ipc_worker.py"), case,
                                       str(steps), str(out)], env=env, cwd=ROOT, start_new_session=True,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    try:
        for p in procs:
            o, _ = p.communicate(timeout=420)
            logs.append(o)
    finally:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, signal.SIGKILL)
    assert all(p.returncode == 0 for p in procs), "\n".join(x[-3000:] for x in logs)
    res = json.loads(out.read_text())
    assert res["opened_peers"] == 1
    assert res["ok"], res["why"]
    assert res["splits"] > 0
