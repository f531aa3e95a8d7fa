"""A/B of where LP3 runs (orca_set_lp3_inline 0 = k_lp3 kernel, 1 = per thread inside k_step,
2 = k_step's block-local queue): bit-identity after 12 steps and per-step device times
(L2 flushed between steps; whole graphed step, and k_step(+k_lp3) from orca_step_timed)."""
import json
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_10107_b200 import orca as O, workloads as W  # noqa: E402

flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["uniform_1m", "uniform", "dense"]
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2]
out = {}
for cfg in cfgs:
    name, _, n = cfg.partition(":")  # e.g. uniform:150000
    w = W.make(name, n=int(n)) if n else W.make(name)
    res = {}
    ref = None
    for mode in modes:
        c = O.Orca(w["params"])
        c.set_agents(w["pos"], w["vel"], w["pref"])
        c.set_lp3_inline(mode)
        c.step(12)
        st = c.get_state()
        if ref is None:
            ref = st
        same = bool(np.array_equal(ref[0], st[0]) and np.array_equal(ref[1], st[1]))
        s = torch.cuda.ExternalStream(c.stream())
        ts, ks = [], []
        for it in range(30):
            with torch.cuda.stream(s):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                c.step(1)
                e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        for it in range(10):
            with torch.cuda.stream(s):
                flush.zero_()
            ks.append(c.step_timed(1)[0])
        res[mode] = dict(same_as_first=same, step_ms=float(np.median(ts)), kstep_lp3_ms=float(np.median(ks)),
                         launch=c.launch_info())
        c.close()
    out[cfg] = res
    print(cfg, json.dumps(res), flush=True)
