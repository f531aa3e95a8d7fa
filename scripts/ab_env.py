"""A/B of an environment switch or of library builds (ORCA_LIB=vlibs/...): per config, a hash of the
state after 12 steps (bit-identity across runs) and the median whole-step device time (L2
flushed between steps).  python scripts/ab_env.py <configs> ; run once per setting."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1908_10107_b200 import orca as O, workloads as W
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cfg in sys.argv[1].split(","):
    name, _, n = cfg.partition(":")
    w = W.make(name, n=int(n)) if n else W.make(name)
    c = O.Orca(w["params"])
    c.set_agents(w["pos"], w["vel"], w["pref"])
    c.step(12)
    st = c.get_state()
    h = hashlib.sha1(np.ascontiguousarray(st[0]).tobytes() + np.ascontiguousarray(st[1]).tobytes()).hexdigest()[:12]
    s = torch.cuda.ExternalStream(c.stream())
    ts = []
    for it in range(40):
        with torch.cuda.stream(s):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            c.step(1)
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    stg = []
    for it in range(15):
        with torch.cuda.stream(s):
            flush.zero_()
        stg.append(c.step_timed(1))
    stage = [round(float(x), 4) for x in np.median(np.array(stg), axis=0)]  # step+lp3, exchange, scan, scatter
    print(cfg, json.dumps(dict(hash=h, step_ms=round(float(np.median(ts)), 4), stages=stage, launch=c.launch_info(),
                                stats_inf=c.stats()["infeasible"])), flush=True)
    c.close()
