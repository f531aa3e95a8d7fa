#!/usr/bin/env python
"""Benchmark of the B200 ORCA step (arXiv 1908.10107) -- prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config uniform_1m] [--impl ours|reference]

Metric (BASELINE.json): agent-updates/s (and ms/frame) of the full per-timestep ORCA
update (binning -> 3x3 k-nearest -> half-planes -> LP2/LP3 -> integrate), i.e. one
"step" = one pass of every hot-path stage over all agents.

Timing: W untimed warm-up steps; then K timed steps, each bracketed by CUDA
events on the library's own stream, with an L2 flush (a 512 MiB write) between timed
steps because the 1M-agent working set (~56 MB) would otherwise stay L2-resident; barrier
+ synchronize around the timed region; max over ranks.  `e2e` repeats the metric through
the public C-ABI with pinned HOST buffers (orca_set_agents H2D -> orca_step ->
orca_get_state D2H every step).  `cpu_baseline` / `--impl reference` time the fp64 oracle
(test infrastructure) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SMS = 148
FP32_LANES_PER_SM = 128  # B200: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / DESIGN.md §7)

# algorithmic fp32 lane-ops per counted unit
# Algorithmic work per launch: 5 c_cand + 50 k + 15 I_LP fp32 lane-ops per
# agent-step, with c_cand = agents in the 3x3 bins (the paper's candidate set),
# k = half-planes built, I_LP = LP inner iterations (constraint checks + LP1 iterations +
# LP3 projections); every unit counted exactly per launch by orca_debug_work.
OPS = dict(stencil=5, lines=50, checks=15, lp1=15, proj=15)
# What the kernel executed (its fine-column runs within the search radius read ~1/15 of
# the 3x3 candidates): reported beside the contract figure.
OPS_EXEC = dict(cand=5, lines=40, checks=4, lp1=8, proj=10)


def source_sha() -> str:
    """sha256 of the CUDA sources + C header: ties an ncu capture (profiles/traffic.json) to
    the revision it measured (scripts/ncu_extract.py writes the same hash)."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1908_10107_b200", "csrc")
    for f in sorted(os.listdir(csrc)) + ["../../include/orca.h"]:
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(csrc, f), "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="uniform_1m")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=6.0, help="single-thread oracle sample (cpu_baseline)")
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="--impl reference: time budget of the timed full oracle steps")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--no-suite", action="store_true", help="skip the other BASELINE workloads (N=1 only)")
    ap.add_argument("--only-timed", action="store_true",
                    help="profiling: stop after the timed steps (no A/B sweeps, e2e, baselines); prints a short line")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="test only: all ranks on GPU 0 (gloo for torch, ORCA_NCCL_LIB=tests/fake_nccl for liborca)")
    ap.add_argument("--lp3-lanes", type=int, default=-1, help="lanes per infeasible agent in the LP3 kernel (-1: auto)")
    ap.add_argument("--variant", type=int, default=-1, help="-1: auto (default), 0: thread per agent, 1: 8-lane group per agent, 2: register top-k, "
                         "3: work-unit LP2")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(config):
    from paper_1908_10107_b200 import workloads as W
    w = W.make(config)
    rho = {"uniform": 0.25, "uniform_1m": 0.25, "dense": 0.5, "uniform_4m": 0.25}.get(config)
    return w, rho


def oracle_rate(w, seconds, rng_seed=0):
    """fp64 oracle (single thread) on a bounded random sample of agents of the same
    workload state; returns (agents/s, sample size, elapsed)."""
    from oracle import oracle as O
    p = O.make_params(**w["params"])
    n = len(w["pos"])
    rng = np.random.default_rng(rng_seed)
    probe = np.sort(rng.choice(n, min(n, 2000), replace=False))
    t0 = time.perf_counter()
    O.step(p, w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"), pref_speed=w.get("pref_speed", 1.0),
           agents=probe)
    t1 = time.perf_counter() - t0
    m = int(min(n, max(2000, len(probe) * seconds / max(t1, 1e-6))))
    sample = np.sort(rng.choice(n, m, replace=False))
    t0 = time.perf_counter()
    O.step(p, w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"), pref_speed=w.get("pref_speed", 1.0),
           agents=sample)
    el = time.perf_counter() - t0
    return m / el, m, el


def run_reference(args):
    """This tier's reference arm: the fp64 oracle (oracle/, unchanged) stepping the WHOLE
    crowd of the bench workload, every step a full synchronous step of all agents, on all host
    cores (forked workers on disjoint agent slices of the same pre-step state; oracle/par.py).
    W warm-up and K timed steps as asked, unless K would not fit the time budget: then as many
    full timed steps as fit (at least one), and `steps` reports what ran."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O, par
    w, rho = workload(args.config)
    n = len(w["pos"])
    p = O.make_params(**w["params"])
    po = par.ParallelOracle(p, w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"),
                            pref_speed=w.get("pref_speed", 1.0))
    warm = min(args.warmup, 1)
    t_warm = po.step(warm) if warm else 0.0
    per = t_warm / warm if warm else None
    budget = args.ref_seconds
    steps = args.steps if per is None else max(1, min(args.steps, int(budget / max(per, 1e-9))))
    el = po.step(steps)
    po.close()
    value = n * steps / el
    line = {
        "impl": "reference", "metric": "agent-updates/s", "value": value, "unit": "agent-updates/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "steps_requested": args.steps,
        "warmup_requested": args.warmup,
        "ms_per_step": 1000.0 * el / steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["name"], "n_agents": n, "rho": rho, **w["params"]},
        "cpu_baseline": {"value": value, "unit": "agent-updates/s", "cores": po.procs, "kind": "oracle",
                         "cpu_model": par.cpu_model(),
                         "sample": f"{steps} full synchronous steps of all {n} agents (after {warm} warm-up step), "
                                   f"agents split over {po.procs} forked processes per step, {el:.1f} s"},
        "e2e": {"value": value, "unit": "agent-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def oracle_baselines(w, seconds):
    """cpu_baseline of the bench line (rank 0, N = 1): the oracle as it stands on the host
    cores -- one full step of the whole workload on all cores, and a single-thread sample of
    the same state for the per-core rate -- plus the BASELINE's small configs run in full
    (C0 circle 1000 steps, C1 corridor 600 steps)."""
    from oracle import oracle as O, par
    from paper_1908_10107_b200 import workloads as W
    n = len(w["pos"])
    p = O.make_params(**w["params"])
    po = par.ParallelOracle(p, w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"),
                            pref_speed=w.get("pref_speed", 1.0))
    el = po.step(1)
    po.close()
    r1, m1, el1 = oracle_rate(w, seconds)
    out = {"value": n / el, "unit": "agent-updates/s", "cores": po.procs, "kind": "oracle",
           "cpu_model": par.cpu_model(),
           "sample": f"one full synchronous step of all {n} agents of the initial state, agents split over "
                     f"{po.procs} forked processes, {el:.1f} s",
           "single_thread": {"value": r1, "cores": 1,
                             "sample": f"{m1} random agents of the same state, one thread, {el1:.1f} s"}}
    configs = {}
    for name, steps in (("circle", 1000), ("corridor", 600)):
        wc = W.make(name)
        pc = O.make_params(**wc["params"])
        poc = par.ParallelOracle(pc, wc["pos"], wc["vel"], pref=wc["pref"], goals=wc.get("goals"),
                                 pref_speed=wc.get("pref_speed", 1.0), procs=1 if name == "circle" else None)
        elc = poc.step(steps)
        configs[wc["name"]] = {"n_agents": len(wc["pos"]), "steps": steps, "seconds": elc,
                               "ms_per_frame": 1000.0 * elc / steps,
                               "agent_updates_per_s": len(wc["pos"]) * steps / elc, "cores": poc.procs}
        poc.close()
    out["configs_full_runs"] = configs
    return out


def suite(orca, torch, peak_tops):
    """BASELINE.json's other workloads at N=1 (north star: "throughput on synthetic circle,
    bidirectional-corridor and random-uniform crowds"): device time per frame of K graph-
    replayed steps after W warm-up steps and one untimed call of K steps (W > 0; C0 and C1 are
    timed from their first step, graph instantiation included; small working sets: L2-resident),
    agent-updates/s,
    and the step's ALU fraction (counted lane-ops of k_step+k_lp3 / whole-step time / peak).
    Plus the launch-chain latency floor (a 1-agent context)."""
    from paper_1908_10107_b200 import workloads as W
    cases = [("circle_C0", W.make("circle"), 0, 1000), ("corridor_C1", W.make("corridor"), 0, 600)]
    for rho in (0.01, 0.05, 0.1, 0.25, 0.5):
        cases.append((f"uniform100k_rho{rho}", W.make("uniform", rho=rho), 10, 100))
    cases.append(("dense_C3", W.make("dense"), 5, 40))
    out = {}
    for name, w, warm, steps in cases:
        ctx = orca.Orca(w["params"])
        ctx.set_agents(w["pos"], w["vel"], w["pref"])
        if w.get("goals") is not None:
            ctx.set_goals(w["goals"], w["pref_speed"])
        if warm:  # warm-up, then one untimed call of the timed length (instantiates its graph)
            ctx.step(warm)
            ctx.step(steps)
        work = ctx.work()
        rg0 = ctx.stats()["regrids"]
        stream = torch.cuda.ExternalStream(ctx.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            ctx.step(steps)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        n = len(w["pos"])
        ops = sum(OPS[k] * work[k] for k in OPS)
        st = ctx.stats()
        out[name] = {"n_agents": n, "steps": steps, "warmup": warm, "ms_per_frame": ms,
                     "agent_updates_per_s": n / (ms / 1000.0),
                     "alu_frac_of_step": ops / (ms / 1000.0) / (peak_tops * 1e12),
                     "infeasible_per_step": st["infeasible"] / max(1, st["steps"]),
                     "regrids_in_timed_region": st["regrids"] - rg0,
                     "remaining": ctx.count() if w.get("goals") is not None else n}
        ctx.close()
    # the paper's crossing experiments: agents walk to their goals and
    # leave there; steps until everyone has left (or a cap) and the device time per step
    rng = np.random.default_rng(7)
    for name, w, het in (("two_way_2500", W.make("two_way"), False),
                         ("two_way_2500_heterogeneous", W.make("two_way"), True),
                         ("eight_way_10k", W.make("eight_way"), False)):
        n = len(w["pos"])
        ctx = orca.Orca(w["params"])
        ctx.set_agents(w["pos"], w["vel"], w["pref"])
        ctx.set_goals(w["goals"], w["pref_speed"])
        ctx.set_goal_removal(w["params"]["radius"])
        if het:  # radius and desired speed each uniform over 3 values, max = 1.25 x desired
            desired = rng.choice([1.0, 1.33, 2.0], n).astype(np.float32)
            ctx.set_agent_props(rng.choice([0.5, 0.75, 1.0], n).astype(np.float32), 1.25 * desired, desired)
        stream = torch.cuda.ExternalStream(ctx.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps, cap = 0, 4000
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
        while ctx.count() > 0 and steps < cap:
            ctx.step(100)
            steps += 100
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        st = ctx.stats()
        out[name] = {"n_agents": n, "steps_run": steps, "remaining": ctx.count(), "removed": st["removed"],
                     "ms_per_step": e0.elapsed_time(e1) / steps, "infeasible_per_step": st["infeasible"] / steps}
        ctx.close()
    # per-step trace dump (f4): 100 steps of 100k agents with every frame copied to
    # pinned host memory on the copy stream, against the same 100 steps without frames
    w = W.make("uniform")
    n = len(w["pos"])
    ctx = orca.Orca(w["params"])
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    ctx.step(10)
    frames = torch.empty((100, n, 2), dtype=torch.float32).pin_memory()
    ctx.step_trace(5, frames[:5])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.step(100)
    ctx.count()  # synchronises
    plain = (time.perf_counter() - t0) * 10.0
    t0 = time.perf_counter()
    ctx.step_trace(100, frames)
    traced = (time.perf_counter() - t0) * 10.0
    out["trace_uniform100k"] = {"ms_per_step_plain_wall": plain, "ms_per_step_with_frames_wall": traced,
                                "frame_bytes": n * 8}
    ctx.close()
    # latency floor: the same launch chain on one agent
    ctx = orca.Orca(W.DEFAULT_PARAMS)
    one = np.zeros((1, 2), np.float32)
    ctx.set_agents(one, one, one)
    ctx.step(10)
    stream = torch.cuda.ExternalStream(ctx.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        ctx.step(200)
        e1.record(stream)
    torch.cuda.synchronize()
    out["latency_floor_ms_per_step"] = e0.elapsed_time(e1) / 200
    ctx.close()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        # NCCL's own init lines (communicator size per rank) on stderr, for the driver's checks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.shared_gpu:  # test mode: every rank on GPU 0, liborca's NCCL from ORCA_NCCL_LIB
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1908_10107_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    from paper_1908_10107_b200 import orca

    w, rho = workload(args.config)
    n_total = len(w["pos"])
    if world > 1:
        nid = orca.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(nid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        ctx = orca.Orca(w["params"], device=local, rank=rank, world=world, nccl_id=bytes(t.cpu().tolist()))
    else:
        ctx = orca.Orca(w["params"], device=local)
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    if w.get("goals") is not None:
        ctx.set_goals(w["goals"], w["pref_speed"])
    ctx.set_variant(args.variant)
    ctx.set_lp3_lanes(args.lp3_lanes)
    stream = torch.cuda.ExternalStream(ctx.stream())
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # ---- warm-up (also instantiates the 1-step and K-step graphs outside the timed region)
    for _ in range(args.warmup):
        ctx.step(1)
    ctx.step(min(args.steps, 64))
    barrier()
    work0 = ctx.work()  # (synchronises: a pending grid re-derivation is seen by the next step)
    ctx.step(1)  # ... and applied here, before the timed region
    barrier()
    ctx.reset_stats()
    maint0 = ctx.stats()

    # ---- timed region: K steps, L2 flushed between steps, events on the library stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with Clocks(local) as clk:
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                flush.zero_()
                evs[s][0].record(stream)
                ctx.step(1)
                evs[s][1].record(stream)
        barrier()
    per = [a.elapsed_time(b) for a, b in evs]
    ms = float(sum(per))
    per_step_stats = [float(np.median(per)), float(np.min(per)), float(np.max(per))]
    if world > 1:
        t = torch.tensor([ms] + per_step_stats, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        per_step_stats = [float(x) for x in t[1:].tolist()]
    if args.only_timed:  # (ncu launch lists: the step's own kernels only)
        if rank == 0:
            print(json.dumps({"metric": "agent-updates/s", "ms_per_step": ms / args.steps, "only_timed": True,
                              "launch_info": ctx.launch_info(), "config": {"workload": w["name"]}}), flush=True)
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return
    st = ctx.stats()
    st["maintenance_in_timed_region"] = {k: st[k] - maint0[k] for k in ("rebalances", "regrids")}
    launch_info = ctx.launch_info()  # kernels per step as launched in the timed region
    kernel_config = ctx.kernel_config()  # the step-kernel instantiation of the timed region
    ms_per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1000.0)

    # ---- L2-resident variant (context): K steps in one graph, no flush
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        ctx.step(args.steps)
        e1.record(stream)
    barrier()
    ms_res = e0.elapsed_time(e1) / args.steps

    # ---- per-kernel times (un-graphed, events around every launch, L2 flushed between)
    stage = np.zeros(4)
    for s in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        stage += np.array(ctx.step_timed(1))
    stage /= args.steps
    comm = None
    if world > 1:  # liborca's communicator size and the exchange time, per rank
        parts = [None] * world
        dist.all_gather_object(parts, (ctx.comm_info()["comm_ranks"], float(stage[3])))
        comm = {"comm_ranks": [q[0] for q in parts], "exchange_ms_per_rank": [q[1] for q in parts]}
    work1 = ctx.work()
    work = {k: 0.5 * (work0[k] + work1[k]) for k in work0}
    # kernel variant A/B (same results bit for bit): fused-step ms per step
    variant_ms = {}
    for v in (0, 1, 2, 3):
        ctx.set_variant(v)
        ctx.step(2)
        acc = 0.0
        for s in range(max(3, args.steps // 4)):
            with torch.cuda.stream(stream):
                flush.zero_()
            acc += ctx.step_timed(1)[0]
        variant_ms[str(v)] = acc / max(3, args.steps // 4)
    ctx.set_variant(args.variant)
    # LP constraint order A/B (reading Q8; same optimum, different work), variant 0; and the
    # work-unit variant 3 in the sequential order, where its work units run
    order_ms = {}
    for name, mode, v in (("greedy", 0, 0), ("sequential", 2, 0), ("randomized", 1, 0),
                          ("sequential_work_units", 2, 3)):
        ctx.set_variant(v)
        ctx.set_lp_order(mode, 1, 0)
        ctx.step(2)
        acc = 0.0
        for s in range(max(3, args.steps // 4)):
            with torch.cuda.stream(stream):
                flush.zero_()
            acc += ctx.step_timed(1)[0]
        order_ms[name] = acc / max(3, args.steps // 4)
    ctx.set_lp_order(0)
    ctx.set_variant(args.variant)
    # LP3 kernel lanes per infeasible agent A/B (same results bit for bit), on the queued path
    # (orca_set_lp3_inline(0)); "inline" = LP3 inside k_step, the automatic choice below one
    # wave of k_step blocks
    lp3_ms = {}
    for lanes in (1, 4, 8, 16, "inline"):
        ctx.set_lp3_inline(1 if lanes == "inline" else 0)
        ctx.set_lp3_lanes(1 if lanes == "inline" else lanes)
        ctx.step(2)
        acc = 0.0
        for s in range(max(3, args.steps // 4)):
            with torch.cuda.stream(stream):
                flush.zero_()
            acc += ctx.step_timed(1)[0]
        lp3_ms[str(lanes)] = acc / max(3, args.steps // 4)
    ctx.set_lp3_lanes(args.lp3_lanes)
    ctx.set_lp3_inline(-1)

    # ---- e2e through the public API with pinned host buffers: every step uploads the
    # kinematic state (orca_set_state: H2D of pos + vel, re-binning), steps once and reads
    # the result back (orca_get_state, or this rank's strip via orca_get_local_state).  The
    # uploaded state is the simulation as it stands after the device-timed runs (a
    # checkpoint reload of the same crowd), so e2e and value time the same phase of the
    # workload rather than the collision-rich first step from the random initial velocities.
    hp = torch.empty((n_total, 2), dtype=torch.float32).pin_memory()
    hv = torch.empty((n_total, 2), dtype=torch.float32).pin_memory()
    hq = torch.from_numpy(w["pref"]).pin_memory()
    if world == 1:
        ctx.get_state(hp, hv)
    else:
        parts = [None] * world
        dist.all_gather_object(parts, ctx.get_local_state())
        gp = np.full((n_total, 2), np.nan, np.float32)
        gv = np.full((n_total, 2), np.nan, np.float32)
        for ids_, p_, v_ in parts:
            gp[ids_] = p_
            gv[ids_] = v_
        hp.copy_(torch.from_numpy(gp))
        hv.copy_(torch.from_numpy(gv))
    e2e_state = "state after the timed steps, re-uploaded every step (pos + vel)"
    if not (torch.isfinite(hp).all() and torch.isfinite(hv).all()):  # removed agents: initial state
        hp.copy_(torch.from_numpy(w["pos"]))
        hv.copy_(torch.from_numpy(w["vel"]))
        e2e_state = "initial state"
    ctx.set_agents(hp, hv, hq)
    ctx.step(1)
    n_loc = ctx.count()
    cap = n_loc + n_loc // 2 + 4096
    oi = torch.empty(cap, dtype=torch.int32).pin_memory()
    op = torch.empty((cap, 2), dtype=torch.float32).pin_memory()
    ov = torch.empty((cap, 2), dtype=torch.float32).pin_memory()

    def readback():
        if world == 1:
            ctx.get_state(op[:n_total], ov[:n_total])
            return n_total
        m = ctx.count()
        if m > cap:
            raise RuntimeError("e2e readback buffer too small")
        orca.lib().orca_get_local_state(ctx._ctx, orca._ptr(oi), orca._ptr(op), orca._ptr(ov))
        return m

    readback()
    ne = max(1, args.e2e_steps)

    def e2e_sync():
        for _ in range(5):  # warm: a re-grid the reloaded state triggers happens here, not timed
            ctx.set_state(hp, hv)
            ctx.step(1)
            readback()
        barrier()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(ne):
            ctx.set_state(hp, hv)
            ctx.step(1)
            m = readback()
            d2h += m * (16 if world == 1 else 20)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el, d2h

    el, d2h = e2e_sync()
    e2e = {"value": n_total * ne / el, "unit": "agent-updates/s",
           "h2d_bytes_per_step": int(hp.numel() * 4 * 2), "d2h_bytes_per_step": int(d2h // ne),
           "ms_per_step": 1000.0 * el / ne, "wall_clock": True, "input": e2e_state,
           "api": "orca_set_state -> orca_step(1) -> orca_get_state (synchronous)"}
    if world == 1:
        # pipelined public API: the upload of step s+1 (copy stream) and the read-back of step
        # s-1 (second copy stream) overlap step s; one wait at the end of the timed region
        outs = [(op[:n_total], ov[:n_total]),
                (torch.empty((n_total, 2), dtype=torch.float32).pin_memory(),
                 torch.empty((n_total, 2), dtype=torch.float32).pin_memory())]
        for s in range(10):  # warm (slot buffers, streams, a pending re-grid)
            ctx.set_state_async(hp, hv)
            ctx.step(1)
            ctx.get_state_async(*outs[s % 2])
        ctx.io_wait()
        barrier()
        t0 = time.perf_counter()
        for s in range(ne):
            ctx.set_state_async(hp, hv)
            ctx.step(1)
            ctx.get_state_async(*outs[s % 2])
        ctx.io_wait()
        ela = time.perf_counter() - t0
        e2e_sync_line = {k: e2e[k] for k in ("value", "ms_per_step", "api")}
        three_calls = {"value": n_total * ne / ela, "ms_per_step": 1000.0 * ela / ne,
                       "api": "orca_set_state_async -> orca_step(1) -> orca_get_state_async per step, "
                              "orca_io_wait once"}
        # the one-call frame (orca_step_io_async): the step's own binning is deferred to the next
        # frame's in-place reload (same results bit for bit, tests/test_gpu_io_async.py)
        for s in range(10):
            ctx.step_io_async(hp, hv, *outs[s % 2])
        ctx.io_wait()
        rg0 = ctx.stats()["regrids"]
        # three timed windows of ne frames each (the PCIe-bound frame varies ~20 % between windows on
        # one host, profiles/r02/repeat_r02b3): the line reports the median window, all three listed
        windows = []
        for rep in range(3):
            barrier()
            t0 = time.perf_counter()
            for s in range(ne):
                ctx.step_io_async(hp, hv, *outs[s % 2])
            ctx.io_wait()
            windows.append(time.perf_counter() - t0)
        elf = sorted(windows)[1]
        regrids_e2e = ctx.stats()["regrids"] - rg0
        e2e = {"value": n_total * ne / elf, "unit": "agent-updates/s",
               "h2d_bytes_per_step": int(hp.numel() * 4 * 2), "d2h_bytes_per_step": int(n_total * 16),
               "ms_per_step": 1000.0 * elf / ne, "wall_clock": True, "input": e2e_state,
               "api": "orca_step_io_async per frame (H2D of pos+vel, one step, D2H of pos+vel), orca_io_wait "
                      "once (pipelined: the upload of frame s+1 and the read-back of frame s-1 overlap step s)",
               "windows_ms_per_step": [round(1000.0 * x / ne, 4) for x in windows], "window": "median of 3",
               "three_calls": three_calls, "synchronous": e2e_sync_line, "regrids_in_timed_region": regrids_e2e}

    # ---- roofline of the dominant kernel (k_step): ALU bound.  peak = the FP32
    # FFMA lane-op rate measured in this run by orca_probe_alu (at the clock it ran at)
    pk, pk_kind = peaks()
    probe = orca.probe_alu(local)
    ops = sum(OPS[k] * work[k] for k in OPS)
    t_step = stage[0] / 1000.0
    achieved = ops / t_step / 1e12
    peak = probe["fp32_lane_ops_per_s"] / 1e12
    nominal = SMS * FP32_LANES_PER_SM * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    traffic, ncu, traffic_note = None, None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            ent = json.load(open(tpath)).get(args.config, {})
            kn = ent.get("k_step_ncu", {})
            if kn.get("source_sha") == source_sha():
                traffic = ent.get("k_step_dram_bytes")
                keep = ("issue_slots_busy_pct", "avg_active_threads_per_warp", "achieved_occupancy_pct",
                        "fma_pipe_active_pct", "alu_pipe_active_pct", "fp64_pipe_active_pct", "warp_instructions",
                        "duration_ns", "report", "source_sha")
                ncu = {k: v for k, v in kn.items() if k in keep} or None
            else:
                traffic_note = "profiles/traffic.json was captured from another source revision: not used"
        except Exception as e:  # noqa: BLE001
            traffic_note = f"profiles/traffic.json unreadable: {e}"
    ops_exec = sum(OPS_EXEC[k] * work[k] for k in OPS_EXEC)
    roofline = {"bound": "alu", "kernel": "k_step(+k_lp3)", "achieved": achieved, "peak": peak, "unit": "Tlane-op/s",
                "frac": achieved / peak, "frac_executed": ops_exec / t_step / 1e12 / peak,
                "traffic": traffic, "traffic_note": traffic_note, "ncu": ncu,
                "work_model": "SURVEY §8(d): 5 c_cand(3x3 bins) + 50 half-planes + 15 LP inner iterations per agent-step",
                "executed": {"achieved": ops_exec / t_step / 1e12, "frac": ops_exec / t_step / 1e12 / peak,
                             "ops_per_launch": ops_exec,
                             "model": "5 candidates read + 40 half-planes + 4 checks + 8 LP1 it + 10 LP3 proj"},
                "peak_source": "measured in this run: orca_probe_alu FP32 FFMA lane-ops/s "
                               f"(probe SM clock {probe['sm_mhz']:.0f} MHz, {probe['fp32_lanes_per_sm_clk']:.1f} "
                               "FMA lanes/SM/clk)",
                "peak_nominal": nominal, "probe": probe,
                "ops_per_launch": ops, "work_per_launch": work,
                "stage_ms": {"k_step+k_lp3": stage[0], "k_scan": stage[1], "k_scatter": stage[2],
                             "exchange": stage[3]}}
    # HBM view of the binning kernels (context)
    hbm_bytes_scatter = n_total / world * (4 + 4 + 4 + 3 * 8 + 4 + 3 * 8 + 4)
    hbm = {"kernel": "k_scatter", "achieved_gbs": hbm_bytes_scatter / (stage[2] / 1000.0) / 1e9 if stage[2] > 0 else None,
           "peak_gbs": pk.get("hbm_gbs"), "bytes_per_launch": hbm_bytes_scatter}

    line = {
        "metric": "agent-updates/s", "value": value, "unit": "agent-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w["name"], "n_agents": n_total, "rho": rho, **w["params"],
                   "l2": "flushed between timed steps (512 MiB write); per-step CUDA events on the library stream",
                   "parallelism": f"strips{world}" if world > 1 else "single",
                   "exchange": ("peer-memory" if ctx.transport() == 0 else "nccl") if world > 1 else None},
        "ms_per_step_l2_resident": ms_res,
        "ms_per_step_median_min_max": per_step_stats,
        # per step: k_step, k_lp3, k_scan, k_scatter (+ strips: k_receive and one k_push per
        # neighbour with the peer-memory exchange)
        "gpu_launches": launch_info["kernels_per_step"] * args.steps, "launch_info": launch_info,
        "kernel_config": kernel_config,
        "kernel_variant": args.variant, "k_step_ms_by_variant": variant_ms, "k_step_ms_by_lp_order": order_ms,
        "lp3_lanes": args.lp3_lanes, "k_step_ms_by_lp3_lanes": lp3_ms,
        "roofline": roofline, "hbm_context": hbm, "comm": comm,
        "stats": st,
    }
    line["e2e"] = e2e
    if rank == 0:
        c = clk.summary()
        line["clocks"] = c
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_baselines(w, args.cpu_seconds)
    ctx.close()
    if rank == 0:
        if world == 1 and not args.no_suite:
            line["suite"] = suite(orca, torch, peak)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start the N ranks itself (one
    process per GPU, torch.distributed.run on 127.0.0.1) with the same arguments."""
    import secrets
    port = os.environ.get("MASTER_PORT") or str(29500 + secrets.randbelow(2000))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", port, os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
