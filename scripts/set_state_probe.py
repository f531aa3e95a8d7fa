"""Host time of orca_set_agents vs orca_set_state (pinned host inputs), 1M agents."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

w = W.make("uniform_1m")
ctx = O.Orca(w["params"])
hp = torch.from_numpy(w["pos"]).pin_memory()
hv = torch.from_numpy(w["vel"]).pin_memory()
hq = torch.from_numpy(w["pref"]).pin_memory()
ctx.set_agents(hp, hv, hq)
ctx.step(30)
ctx.get_state(hp, hv)


def t(f, r=10):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(r):
        f()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / r * 1000, 4)


print("set_agents ms", t(lambda: ctx.set_agents(hp, hv, hq)))
print("set_state  ms", t(lambda: ctx.set_state(hp, hv)))
print("step(1)    ms", t(lambda: (ctx.step(1), ctx.count())))
print("get_state  ms", t(lambda: ctx.get_state(hp, hv)))
