"""Scenarios shared by the fake-NCCL multi-process test and its single-GPU reference:
each returns (workload, run(ctx, w)) and run() drives the context identically everywhere."""
import numpy as np

from paper_1908_10107_b200 import workloads as W


def _uniform():
    w = W.make("uniform", n=20000, rho=0.3)

    def run(ctx, w):
        ctx.set_agents(w["pos"], w["vel"], w["pref"])
        ctx.step(7)
        ctx.rebalance()
        ctx.step(70)  # crosses a 64-step chunk: automatic capacity check between chunks

    return w, run


def _convergent():
    w = W.make("uniform", n=16000, rho=0.25)
    centre = w["pos"].mean(axis=0)
    goals = np.repeat(centre[None].astype(np.float32), len(w["pos"]), axis=0)

    def run(ctx, w):
        ctx.set_agents(w["pos"], w["vel"], w["pref"])
        ctx.set_goals(goals, 1.0)
        ctx.set_lp_order(True, 3, 0)
        for _ in range(10):
            ctx.step(64)

    return w, run


SCENARIOS = {"uniform": _uniform, "convergent": _convergent}
