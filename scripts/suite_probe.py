import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1908_10107_b200 import orca as O, workloads as W
w = W.make("corridor")
for mode in ("suite", "suite_nowork", "chunks64"):
    ctx = O.Orca(w["params"])
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    if mode == "suite":
        ctx.work()
    stream = torch.cuda.ExternalStream(ctx.stream())
    if mode.startswith("suite"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream); ctx.step(600); e1.record(stream)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(mode, "ms/frame", e0.elapsed_time(e1) / 600, "wall ms", (t1 - t0) * 1e3, ctx.stats()["regrids"], flush=True)
    else:
        row = []
        for c in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                e0.record(stream); ctx.step(64); e1.record(stream)
            torch.cuda.synchronize(); t1 = time.perf_counter()
            row.append((round(e0.elapsed_time(e1), 2), round((t1 - t0) * 1e3, 2), ctx.stats()["regrids"]))
        print(mode, row, flush=True)
    ctx.close()
