"""Worker of tests/test_gpu_ipc.py: one rank of a 2-process run on ONE GPU with the host-ordered
CUDA-IPC halo (no NCCL).  Rank 0 compares the assembled state with the oracle and writes a verdict."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import cem_inputs as ci  # noqa: E402


def main():
    case, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    import paper_2508_04076_b200.dist as cdist
    if case == "cfg0":
        p = ci.config(0)
    else:
        p = ci.compact_tension(cells=(24, 24, 3), dims=(0.2, 0.2, 0.025), v0=60.0, t0=20e-6)
    ds = cdist.DistSimulation(p, device=0, transport="host_ipc")
    ds.step(steps // 2, 1)
    ds.step(steps - steps // 2, 1)
    g = ds.state()
    if rank == 0:
        import oracle
        o = oracle.Oracle(p).run(steps, 1)
        s = o.state()
        r = o.records()
        res = {"splits": int(r.elem.size), "ok": True, "why": []}
        for k in ("u", "v", "a"):
            if not np.array_equal(g[k], s[k]):
                res["ok"] = False
                res["why"].append(k)
        for k, ref in (("tet_state", s["state"]), ("mass", s["m"]), ("rec_elem", r.elem), ("rec_step", r.step),
                       ("rec_cand", r.cand), ("rec_G", r.G), ("rec_area", r.area)):
            if not np.array_equal(g[k], ref):
                res["ok"] = False
                res["why"].append(k)
        if g["dissipated"] != o.dissipated:
            res["ok"] = False
            res["why"].append("dissipated")
        res["opened_peers"] = len(ds.part["peers"])
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
