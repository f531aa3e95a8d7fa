"""Per-chunk device time of the corridor workload (C1) for each kernel variant, with the
maintenance counters (regressions hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "corridor"
w = W.make(cfg)
for variant in (0, 1):
    ctx = O.Orca(w["params"])
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    ctx.set_variant(variant)
    stream = torch.cuda.ExternalStream(ctx.stream())
    row = []
    for chunk in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            ctx.step(60)
            e1.record(stream)
        torch.cuda.synchronize()
        row.append(round(e0.elapsed_time(e1) / 60, 4))
    st = ctx.stats()
    g = ctx.grid() if hasattr(ctx, "grid") else None
    wk = ctx.work()
    print(cfg, "variant", variant, "ms/step per 60-step chunk", row, "regrids", st["regrids"], "grid", g,
          "work/agent", {k: round(v / len(w["pos"]), 1) for k, v in wk.items()}, flush=True)
    ctx.close()
