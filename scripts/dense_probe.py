"""Suite's dense case (500k, rho 0.5): warm-up, one untimed 40-step call, then a timed 40-step
call; prints device ms per frame and re-grids inside (regression hunt)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

w = W.make("dense")
for rep in range(2):
    ctx = O.Orca(w["params"])
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    ctx.step(5)
    ctx.step(40)
    stream = torch.cuda.ExternalStream(ctx.stream())
    for call in range(3):
        rg0 = ctx.stats()["regrids"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            ctx.step(40)
            e1.record(stream)
        torch.cuda.synchronize()
        print(rep, call, "ms/frame", round(e0.elapsed_time(e1) / 40, 4), "wall ms", round((time.perf_counter() - t0) * 1e3, 2),
              "regrids", ctx.stats()["regrids"] - rg0, ctx.launch_info(), flush=True)
    ctx.close()
