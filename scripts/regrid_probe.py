"""Host cost of re-grids on spreading crowds: wall time of orca_step chunks with and without a
re-grid inside, plus ORCA_DEBUG_TIMING's per-re-grid and per-graph-rebuild lines (stderr).
python scripts/regrid_probe.py [config] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "corridor"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 600
w = W.make(cfg)
ctx = O.Orca(w["params"])
ctx.set_agents(w["pos"], w["vel"], w["pref"])
ctx.step(5)
torch.cuda.synchronize()
rows = []
for s in range(steps):
    rg0 = ctx.stats()["regrids"]
    t0 = time.perf_counter()
    ctx.step(1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rows.append((dt, ctx.stats()["regrids"] - rg0))
plain = sorted(d for d, r in rows if r == 0)
rg = [d for d, r in rows if r > 0]
print(f"{cfg}: {len(rg)} re-grids in {steps} steps; step wall ms median {1e3 * plain[len(plain) // 2]:.4f}; "
      f"steps with a re-grid: {[round(1e3 * d, 3) for d in rg]}")
