"""Whole-step device time (graphed orca_step(1), L2 flushed between steps, median of 30) of
kernel variants across crowd sizes -- the measurement behind the automatic variant choice
(DESIGN.md §12).  python scripts/variant_sizes_probe.py [variants] [sizes] [config]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O, workloads as W  # noqa: E402

variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,4").split(",")]
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10000,20000,50000,100000,150000,250000,500000,1000000").split(",")]
cfg = sys.argv[3] if len(sys.argv) > 3 else "uniform"
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for n in sizes:
    w = W.make(cfg, n=n)
    row = {"config": cfg, "n": n}
    ref = None
    for v in variants:
        c = O.Orca(w["params"])
        c.set_agents(w["pos"], w["vel"], w["pref"])
        c.set_variant(v)
        c.step(12)
        st = c.get_state()
        ref = st if ref is None else ref
        s = torch.cuda.ExternalStream(c.stream())
        ts = []
        for it in range(30):
            with torch.cuda.stream(s):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                c.step(1)
                e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row[f"v{v}_ms"] = round(float(np.median(ts)), 4)
        row[f"v{v}_same"] = bool(np.array_equal(ref[0], st[0]) and np.array_equal(ref[1], st[1]))
        row[f"v{v}_launch"] = c.launch_info()
        c.close()
    print(json.dumps(row), flush=True)
