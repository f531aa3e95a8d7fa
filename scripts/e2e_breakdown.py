"""Host-timed breakdown of the e2e loop (set_agents from pinned host -> step(1) -> get_state
into pinned host) at one workload; prints per-call means (ms)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "uniform_1m"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # reload the state after `warm` steps
w = W.make(cfg)
n = len(w["pos"])
ctx = O.Orca(w["params"])
hp = torch.from_numpy(w["pos"]).pin_memory()
hv = torch.from_numpy(w["vel"]).pin_memory()
hq = torch.from_numpy(w["pref"]).pin_memory()
op = torch.empty((n, 2), dtype=torch.float32).pin_memory()
ov = torch.empty((n, 2), dtype=torch.float32).pin_memory()
if warm:
    ctx.set_agents(hp, hv, hq)
    ctx.step(warm)
    ctx.get_state(hp, hv)
for _ in range(3):
    ctx.set_agents(hp, hv, hq)
    ctx.step(1)
    ctx.get_state(op, ov)
T = {"set_agents": 0.0, "step": 0.0, "get_state": 0.0}
R = 20
for _ in range(R):
    t0 = time.perf_counter()
    ctx.set_agents(hp, hv, hq)
    t1 = time.perf_counter()
    ctx.step(1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.get_state(op, ov)
    t3 = time.perf_counter()
    T["set_agents"] += t1 - t0
    T["step"] += t2 - t1
    T["get_state"] += t3 - t2
# raw copy speeds for context
x = torch.empty(n * 6, dtype=torch.float32, device="cuda")
h = torch.empty(n * 6, dtype=torch.float32).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(R):
    x.copy_(h, non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t0) / R
t0 = time.perf_counter()
for _ in range(R):
    h[: n * 4].copy_(x[: n * 4], non_blocking=True)
torch.cuda.synchronize()
d2h = (time.perf_counter() - t0) / R
print(cfg, "warm", warm, {k: round(1000 * v / R, 4) for k, v in T.items()},
      f"raw H2D {n*24/1e6:.0f} MB {1000*h2d:.3f} ms ({n*24/h2d/1e9:.1f} GB/s), "
      f"raw D2H {n*16/1e6:.0f} MB {1000*d2h:.3f} ms ({n*16/d2h/1e9:.1f} GB/s)")
# step(1) + sync without reloading (history radius valid, graph cached)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(R):
    ctx.step(1)
    torch.cuda.synchronize()
print("  step(1)+sync, no reload:", round(1000 * (time.perf_counter() - t0) / R, 4), "ms")
# first step after a reload, timed on the device
ctx.set_agents(hp, hv, hq)
ms = ctx.step_timed(1)
print("  device ms of the first step after set_agents:", [round(x, 4) for x in ms])
ms = ctx.step_timed(1)
print("  device ms of the second step:", [round(x, 4) for x in ms])
