"""Per-frame I/O loop timing: orca_step_io_async vs the three async calls vs the synchronous
calls, with re-grid counts (python scripts/e2e_probe.py [config] [frames])."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "uniform"
ne = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
w = W.make(cfg)
n = len(w["pos"])
c = O.Orca(w["params"])
c.set_agents(w["pos"], w["vel"], w["pref"])
c.step(int(os.environ.get("PRE_STEPS", "30")))
p, v = c.get_state()
hp, hv = torch.from_numpy(p).pin_memory(), torch.from_numpy(v).pin_memory()
hq = torch.from_numpy(w["pref"]).pin_memory()
outs = [(torch.empty((n, 2)).pin_memory(), torch.empty((n, 2)).pin_memory()) for _ in range(2)]
if "--churn" in sys.argv:  # the bench's A/B section before its e2e part
    for v in (0, 1, 2, 3):
        c.set_variant(v)
        c.step(2)
        for _ in range(5):
            c.step_timed(1)
    c.set_variant(-1)
    for mode, v in ((0, 0), (2, 0), (1, 0), (2, 3)):
        c.set_variant(v)
        c.set_lp_order(mode, 1, 0)
        c.step(2)
        for _ in range(5):
            c.step_timed(1)
    c.set_lp_order(0)
    c.set_variant(-1)
    for lanes in (1, 4, 8, 16, "inline"):
        c.set_lp3_inline(1 if lanes == "inline" else 0)
        c.set_lp3_lanes(1 if lanes == "inline" else lanes)
        c.step(2)
        for _ in range(5):
            c.step_timed(1)
    c.set_lp3_lanes(-1)
    c.set_lp3_inline(-1)
    print("churned", c.launch_info(), flush=True)
c.set_agents(hp, hv, hq)
c.step(1)
if "--sync" in sys.argv:
    for _ in range(20):
        c.set_state(hp, hv)
        c.step(1)
        c.get_state()
for name in ("step_io", "three", "step_io", "three"):
    for s in range(3):
        if name == "step_io":
            c.step_io_async(hp, hv, *outs[s % 2])
        else:
            c.set_state_async(hp, hv)
            c.step(1)
            c.get_state_async(*outs[s % 2])
    c.io_wait()
    r0 = c.stats()["regrids"]
    t0 = time.perf_counter()
    for s in range(ne):
        if name == "step_io":
            c.step_io_async(hp, hv, *outs[s % 2])
        else:
            c.set_state_async(hp, hv)
            c.step(1)
            c.get_state_async(*outs[s % 2])
    c.io_wait()
    el = time.perf_counter() - t0
    print(f"{cfg} {name:8s} {1000 * el / ne:.4f} ms/frame  regrids +{c.stats()['regrids'] - r0}", flush=True)
