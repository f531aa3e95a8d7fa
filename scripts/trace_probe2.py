import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

w = W.make("uniform")
n = len(w["pos"])
ctx = O.Orca(w["params"])
ctx.set_agents(w["pos"], w["vel"], w["pref"])


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    ctx.count()
    return round((time.perf_counter() - t0) * 1000, 3)


print("before trace: step(1)", [t(lambda: ctx.step(1)) for _ in range(5)])
print("before trace: step(50)", [t(lambda: ctx.step(50)) for _ in range(3)])
pinned = torch.empty((20, n, 2), dtype=torch.float32).pin_memory()
print("trace(20)", t(lambda: ctx.step_trace(20, pinned)))
print("after trace: step(1)", [t(lambda: ctx.step(1)) for _ in range(5)])
print("after trace: step(50)", [t(lambda: ctx.step(50)) for _ in range(3)])
