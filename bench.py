#!/usr/bin/env python3
"""bench.py -- tet·steps/s of the fp64 explicit CEM step (ES-FEM strain, stress, crack
criterion, force assembly, Newmark update, split pass) on B200, and its HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cem|reference] [--config 3]

Workload (BASELINE.json configs[3], the weak-scaling block the metric is quoted on at
1/2/4/8 GPUs): 100x100x17 Kuhn cells x 6 = 1.02M tets per GPU, E = 32 GPa, nu = 0.2,
rho = 2450, Gc = 3 J/m^2, 0.5 % pre-damaged tets, 1 MPa traction, crack check every step.
Inputs are synthetic and seeded (cem_inputs); the per-step working set (~0.4 GB) is
larger than the 126 MB L2, so no L2 flush is needed between timed steps.

One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tet·steps/sec (fp64 explicit ES-FEM step) at 1/2/4/8 B200; % HBM roofline"
UNIT = "tet·steps/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def b_alg_per_step(N, E, S):
    """177 B/node + 17 B/tet + 96 B/edge."""
    return 177 * N + 17 * E + 96 * S


# the same bytes charged to the stage kernel that moves them (DESIGN.md "Algorithmic bytes",
# per-stage table): AB reads u (24 B/node), conn + state (17 B/tet) and writes sigma (48 B/edge);
# C reads sigma (48 B/edge); D moves the rest of the node terms (153 B/node)
STAGE_KERNELS = {"stage_AB_strain_edge_stress": ("k_AB", lambda N, E, S: 24 * N + 17 * E + 48 * S),
                 "stage_C_force_earlyout": ("k_C", lambda N, E, S: 48 * S),
                 "stage_D_node_update": ("k_D", lambda N, E, S: 153 * N)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.samples = []
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [l for t, l in self.samples if t0 <= t <= t1] or [l for t, l in self.samples]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except Exception:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_problem(cfg, P=1):
    import cem_inputs as ci
    return ci.config(cfg, P=1) if cfg == 3 else ci.config(cfg)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(prob, budget_s=12.0):
    """The oracle as it stands, timed on this host's cores on a bounded sample, plus the same
    oracle on ONE thread (OMP_NUM_THREADS = nproc and = 1; results do not depend
    on the thread count)."""
    import oracle
    t0 = time.time()
    o = oracle.Oracle(prob)
    init_s = time.time() - t0
    o.run(1, 1)  # first step (page-in)
    steps, t0 = 0, time.time()
    while True:
        o.run(1, 1)
        steps += 1
        if time.time() - t0 > budget_s or steps >= 50:
            break
    el = time.time() - t0
    cores = oracle.num_threads()
    oracle.set_threads(1)
    t1 = time.time()
    o.run(2, 1)
    el1 = time.time() - t1
    oracle.set_threads(cores)
    return {"value": prob.n_tets * steps / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "value_1_thread": prob.n_tets * 2 / el1,
            "sample": f"{prob.name}: {steps} oracle steps (criterion every step) after 1 warm step on {cores} "
                      f"threads, then 2 steps on 1 thread; init {init_s:.1f}s excluded"}


def fp64_peak():
    """Measured fp64 FMA throughput (tools/dfma_peak, built by __graft_entry__.build())."""
    tool = os.path.join(ROOT, "tools", "dfma_peak")
    if not os.path.exists(tool):
        return None
    try:
        out = subprocess.run([tool], capture_output=True, text=True, timeout=60).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the CPU oracle on the same workload (bounded sample per step)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import cem_inputs as ci
    import oracle
    # the cem arm's workload itself (config 3, 1.02M tets): one oracle step is ~0.06 s on 16 cores,
    # so W + K steps stay within a few minutes up to K ~ 2000
    prob = ci.config(3)
    o = oracle.Oracle(prob)
    o.run(args.warmup, 1)
    t0 = time.time()
    o.run(args.steps, 1)
    el = time.time() - t0
    val = prob.n_tets * args.steps / el
    full = prob
    T = full.tets.astype(np.int64)
    pairs = np.concatenate([np.sort(T[:, [a, b]], axis=1) for a, b in ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))])
    S_full = int(np.unique(pairs[:, 0] * full.n_nodes + pairs[:, 1]).size)
    ws_n = max(1, args.gpus)
    config = {"workload": f"cfg3: {full.name} {full.n_tets} tets/{full.n_nodes} nodes/{S_full} edges per GPU, "
                          f"crack check + split pass every step",
              "tets_per_gpu": full.n_tets,
              "parallelism": f"{ws_n} GPUs: RCB slabs + 2-ring ghost layer, NCCL halo exchange per step"
              if ws_n > 1 else "1 GPU",
              "l2": "per-step working set > 126 MB L2 (no flush needed)"}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Kuhn lattice, cem_inputs)",
            "config": config,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"the full config-3 block ({prob.n_tets} tets) x {args.steps} steps after "
                                       f"{args.warmup} warm-up steps on the host cores (OpenMP), crack check every step"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="cem", choices=["cem", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_2508_04076_b200 as cem

    if ws > 1:
        # weak scaling (BASELINE.json configs[3]): global grid (100 P) x 100 x 17, RCB slabs,
        # one rank per GPU, NCCL halo exchange inside every step
        import cem_inputs as ci
        import paper_2508_04076_b200.dist as cdist
        prob = ci.config(3, P=ws) if args.config == 3 else make_problem(args.config)
        sim = cdist.DistSimulation(prob, device=local)
        E = sim.n_tets_owned
        N, S = sim.sim.n_nodes, sim.sim.n_edges
    else:
        prob = make_problem(args.config)
        sim = cem.Simulation.from_problem(prob, device=local)
        N, E, S = sim.n_nodes, sim.n_tets, sim.n_edges
    stream = sim.torch_stream
    crack_every = 1

    # clock sampler first (nvidia-smi needs a moment to start), then the warm-up steps (untimed)
    # directly followed by the timed ones: no idle gap between them
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    sim.step(args.warmup, crack_every)
    l0 = sim.launch_count
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th0 = time.time()
    ev0.record(stream)
    sim.step(args.steps, crack_every)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    th1 = time.time()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = sim.launch_count - l0
    st = sim.state(records=False) if ws == 1 else sim.sim.state(records=False)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tot = torch.tensor([float(E)], device=dev)
        dist.all_reduce(tot)
        E_all = float(tot.item())
    else:
        E_all = float(E)
    # per-kernel durations on the launching stream (eager launches bracketed by CUDA events)
    kt = {}
    kp0 = kp1 = time.time()
    if ws == 1:
        sim.set_profiling(True)
        sim.step(args.steps, crack_every)
        kt = sim.kernel_times()
        kp1 = time.time()
        sim.set_profiling(False)
    sampler.stop()
    clocks = sampler.summary(th0 - 0.05, max(th1, kp1) + 0.05)

    ms_step = ms / args.steps
    value = E_all * args.steps / (ms / 1e3)
    hbm, peak_kind = peaks()
    balg = b_alg_per_step(N, E, S)
    achieved = balg / (ms_step / 1e3) / 1e9
    kernels = {k: {"ms_per_launch": v / args.steps} for k, v in kt.items()}
    tot_k = sum(v for v in kt.values())
    for k in kernels:
        kernels[k]["share"] = kt[k] / tot_k if tot_k > 0 else None
    traffic = traffic_live = None
    tj = {}
    tpath = os.path.join(ROOT, "profiles", "traffic_per_step.json")
    if os.path.exists(tpath) and args.config == 3 and ws == 1:  # the committed capture is config 3, 1 GPU
        try:
            tj = json.load(open(tpath))
            traffic, traffic_live = tj.get("dram_bytes_per_step"), tj.get("dram_bytes_per_step_live")
        except Exception:
            traffic = traffic_live = None
    # roofline of the dominant stage kernel: its algorithmic bytes per launch over its average
    # launch duration (CUDA events on the launching stream, measured above); traffic = its ncu
    # DRAM bytes per launch (one --set full capture, profiles/traffic_per_step.json)
    roof = {"bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None, "traffic": None,
            "peak_kind": peak_kind}
    if kernels:
        dom = max((k for k in kernels if k in STAGE_KERNELS), key=lambda k: kernels[k]["ms_per_launch"], default=None)
        if dom:
            kname, fb = STAGE_KERNELS[dom]
            b_launch = fb(N, E, S)
            ach = b_launch / (kernels[dom]["ms_per_launch"] / 1e3) / 1e9
            cold = tj.get("per_kernel_cold", {}).get(kname)
            roof.update({"kernel": kname, "achieved": ach, "frac": ach / hbm, "b_alg_bytes_per_launch": b_launch,
                         "ms_per_launch": kernels[dom]["ms_per_launch"],
                         "traffic": (cold["dram_read"] + cold["dram_write"]) if cold else None,
                         "traffic_source": ("stored ncu --set full capture of this build, config 3: "
                                            f"profiles/traffic_per_step.json ({tj.get('round', '?')})") if cold else None})
    # the whole step as one unit (SURVEY.md §8(d)'s "% of HBM roofline" of the metric)
    roof["step"] = {"achieved": achieved, "frac": achieved / hbm, "b_alg_bytes_per_step": balg,
                    "traffic": traffic,
                    # DRAM bytes the step really moves (ncu, no flush between kernels; profiles/)
                    # over this run's step time: the share of HBM bandwidth the kernels sustain
                    "traffic_live": traffic_live,
                    "dram_frac_live": (traffic_live / (ms_step / 1e3) / 1e9 / hbm) if traffic_live else None}
    # on-chip floors of the step from the stored ncu capture of this build (per-launch counters of
    # k_AB, k_C, k_D: L1 data-pipe wavefronts per SM, warp instructions, fp64 thread operations;
    # DESIGN.md section 6): the time each unit alone would need at its peak, next to the HBM floor
    pipes = tj.get("per_kernel_pipes")
    if pipes:
        clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        roof["on_chip_floors"] = {
            "l1_data_pipe_us": sum(q["l1_wavefronts_per_sm"] for q in pipes.values()) / clk * 1e6,
            "issue_us": sum(q["warp_inst"] for q in pipes.values()) / (sms * 4 * clk) * 1e6,
            "fp64_us": sum(q["fp64_thread_ops"] for q in pipes.values()) / 18.1e12 * 1e6,
            "hbm_b_alg_us": balg / hbm / 1e3,
            "measured_us": ms_step * 1e3,
            "binding": "l1_data_pipe (shared-memory + global-load wavefronts, one per SM and clock)",
            "source": f"stored ncu --set full capture, profiles/traffic_per_step.json ({tj.get('round', '?')}); "
                      "fp64 at the measured 18.1 T instructions/s (tools/dfma_peak)"}
    if roof["achieved"] is None:  # (no per-kernel times, N > 1): the step view
        roof.update({"kernel": "cem_step (unit = one step)", "achieved": achieved, "frac": achieved / hbm,
                     "traffic": traffic})

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Kuhn lattice, cem_inputs)",
        "config": {"workload": f"cfg{args.config}: {prob.name} {E} tets/{N} nodes/{S} edges per GPU, "
                               f"crack check + split pass every step",
                   "tets_per_gpu": E,
                   "parallelism": f"{ws} GPUs: RCB slabs + 2-ring ghost layer, NCCL halo exchange per step"
                   if ws > 1 else "1 GPU",
                   "l2": "per-step working set > 126 MB L2 (no flush needed)"},
        "roofline": roof,
        "kernels": kernels,
        "timed_steps": [args.warmup, args.warmup + args.steps],
        "phase": ("cracking (config 3 splits its 5143 pre-damaged tets by step ~45; the criterion kernels "
                  "evaluate them every step until then)" if args.config == 3 and args.warmup < 45 else
                  "steady state" if args.config == 3 else None),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "fp64_peak_measured": fp64_peak() if rank == 0 else None,
        "n_active_end": int(st.n_active),
    }
    if ws == 1:
        line["splits_total"] = int(sim.state().rec_elem.size)

    if not args.no_e2e and rank == 0 and ws == 1:
        # end to end through the public API: host mesh -> cem_init_mesh (H2D) -> K steps -> state (D2H)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        sim2 = cem.Simulation.from_problem(prob, device=local)
        ta = time.perf_counter()
        sim2.step(args.steps, crack_every)
        s2 = sim2.state(records=True)
        t1 = time.perf_counter()
        h2d = prob.X.nbytes + prob.tets.nbytes + prob.tet_state.nbytes + prob.tet_gc.nbytes + \
            prob.tface.nbytes + prob.tface_t.nbytes
        d2h = 3 * s2.u.nbytes + s2.tet_state.nbytes + s2.mass.nbytes
        line["e2e"] = {"value": E * args.steps / (t1 - t0), "unit": UNIT,
                       "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                       "init_s": ta - t0, "steps_and_readback_s": t1 - ta,
                       "what": "cem_init_mesh from host arrays (host preprocessing + H2D) + K steps + "
                               "cem_get_state(CEM_HOST)"}
        sim2.close()
    if not args.no_cpu_baseline and rank == 0 and ws == 1:
        line["cpu_baseline"] = cpu_baseline(prob)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
