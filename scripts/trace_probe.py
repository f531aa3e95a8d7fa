"""Probe of orca_step_trace cost: plain steps vs traced steps, pinned torch vs numpy frames."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

w = W.make("uniform")
n = len(w["pos"])
ctx = O.Orca(w["params"])
ctx.set_agents(w["pos"], w["vel"], w["pref"])
ctx.step(10)
pinned = torch.empty((50, n, 2), dtype=torch.float32).pin_memory()
npf = np.empty((50, n, 2), np.float32)
for name, fr in (("pinned", pinned), ("numpy", npf), ("pinned", pinned)):
    ctx.step_trace(2, fr[:2])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.step_trace(50, fr)
    print(name, "ms/step with frames", (time.perf_counter() - t0) * 20.0, flush=True)
t0 = time.perf_counter()
for _ in range(50):
    ctx.step(1)
ctx.count()
print("step(1) x50 ms/step", (time.perf_counter() - t0) * 20.0)
t0 = time.perf_counter()
ctx.step(50)
ctx.count()
print("step(50) ms/step", (time.perf_counter() - t0) * 20.0)
