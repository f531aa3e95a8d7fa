"""Whole-step device time of P loopback strips on one GPU (the multi-GPU decomposition's
overhead without the NVLink part): 1M uniform, P = 1, 2, 4, 8, overlap off/on, both transports.
python scripts/strips_probe.py [config]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "uniform_1m"
w = W.make(cfg)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
runs = [(1, 0, 0, -1), (2, 0, 0, -1), (2, 1, 0, -1), (4, 0, 0, -1), (4, 1, 0, -1), (8, 0, 0, -1), (8, 1, 0, -1),
        (8, 1, 1, -1)]
if len(sys.argv) > 2:  # e.g. "8:0:0:0,8:0:0:2": strips:overlap:transport:lp3_inline
    runs = [tuple(int(x) for x in r.split(":")) for r in sys.argv[2].split(",")]
for P, ov, tr, l3 in runs:
    c = O.Orca(w["params"], strips=P) if P > 1 else O.Orca(w["params"])
    c.set_agents(w["pos"], w["vel"], w["pref"])
    if P > 1:
        c.set_transport(tr)
        c.set_overlap(ov)
    c.set_lp3_inline(l3)
    c.step(10)
    s = torch.cuda.ExternalStream(c.stream())
    ts = []
    for it in range(20):
        with torch.cuda.stream(s):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            c.step(1)
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"config": cfg, "strips": P, "overlap": ov, "transport": tr, "lp3_inline": l3,
                      "ms_per_step": round(float(np.median(ts)), 4), "launch": c.launch_info()}), flush=True)
    c.close()
