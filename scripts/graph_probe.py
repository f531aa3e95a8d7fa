"""Probe: host and device time of orca_step(1) right after orca_set_agents (graph path)
versus orca_step_timed (direct launches), same state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

w = W.make(sys.argv[1] if len(sys.argv) > 1 else "uniform_1m")
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = O.Orca(w["params"])
hp = torch.from_numpy(w["pos"]).pin_memory()
hv = torch.from_numpy(w["vel"]).pin_memory()
hq = torch.from_numpy(w["pref"]).pin_memory()
ctx.set_agents(hp, hv, hq)
if warm:
    ctx.step(warm)
    ctx.get_state(hp, hv)
stream = torch.cuda.ExternalStream(ctx.stream())
for rep in range(4):
    ctx.set_agents(hp, hv, hq)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        e0.record(stream)
        ctx.step(1)
        e1.record(stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"graph step after set_agents: host launch {1000*(t1-t0):.3f} ms, host total {1000*(t2-t0):.3f} ms, "
          f"device {e0.elapsed_time(e1):.3f} ms")
for rep in range(2):
    ctx.set_agents(hp, hv, hq)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ms = ctx.step_timed(1)
    t2 = time.perf_counter()
    print(f"direct step after set_agents: host total {1000*(t2-t0):.3f} ms, device stages {[round(x, 3) for x in ms]}")
# the e2e loop pattern: set_agents -> step(1) -> get_state, device-timed step
op = torch.empty((len(w["pos"]), 2), dtype=torch.float32).pin_memory()
ov = torch.empty((len(w["pos"]), 2), dtype=torch.float32).pin_memory()
for rep in range(5):
    ctx.set_agents(hp, hv, hq)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        e0.record(stream)
        ctx.step(1)
        e1.record(stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx.get_state(op, ov)
    t2 = time.perf_counter()
    print(f"e2e pattern: step host {1000*(t1-t0):.3f} ms (device {e0.elapsed_time(e1):.3f}), get_state {1000*(t2-t1):.3f} ms")
