"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck),
each driving the product path through the C-ABI: python scripts/sanitize_cases.py <case>.
Cases cover every kernel family: the step chain (k_step thread/group/register/work-unit
variants, inline and queued LP3 with 1 and 8 lanes, k_scan's decoupled look-back, k_scatter),
the strips exchange in loopback (k_push + arrival flags, k_receive, rebalance), the async
I/O path (k_reload), the trace dump and goals/removal/heterogeneous agents."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1908_10107_b200 import orca as O, workloads as W  # noqa: E402


def run_case(name):
    if name == "circle":
        w = W.make("circle")
        c = O.Orca(w["params"])
        c.set_agents(w["pos"], w["vel"], w["pref"])
        c.set_goals(w["goals"], w["pref_speed"])
        c.set_goal_removal(w["params"]["radius"])
        c.step(40)
        c.debug_step()
        for v in (0, 1, 2, 3):
            c.set_variant(v)
            c.step(2)
    elif name == "corridor":
        w = W.make("corridor")
        c = O.Orca(w["params"])
        c.set_agents(w["pos"], w["vel"], w["pref"])
        c.step(5)
        c.debug_step()
        c.set_lp3_inline(0)  # queued LP3 (k_lp3), thread and 8-lane group
        c.step(2)
        c.set_lp3_lanes(8)
        c.step(2)
        c.set_lp_order(1, 7, 0)
        c.step(2)
        c.set_variant(3)
        c.set_lp_order(2)
        c.step(2)
        c.work()
        hp = np.ascontiguousarray(w["pos"])
        hv = np.ascontiguousarray(w["vel"])
        c.set_state_async(hp, hv)
        c.step(1)
        op, ov = np.empty_like(hp), np.empty_like(hv)
        c.get_state_async(op, ov)
        c.io_wait()
    elif name == "strips4":
        w = W.make("uniform", n=8000, rho=0.3)
        for transport in (0, 1):
            c = O.Orca(w["params"], strips=4)
            c.set_agents(w["pos"], w["vel"], w["pref"])
            c.set_transport(transport)
            rng = np.random.default_rng(3)
            n = len(w["pos"])
            c.set_agent_props(rng.choice([0.4, 0.5], n).astype(np.float32),
                              np.full(n, 1.3, np.float32), np.full(n, 1.0, np.float32))
            c.step(6)
            c.rebalance()
            c.step(3)
            c.get_local_state()
            c.close()
    elif name == "trace":
        w = W.make("uniform", n=4000, rho=0.25)
        c = O.Orca(w["params"])
        c.set_agents(w["pos"], w["vel"], w["pref"])
        fr = np.zeros((4, len(w["pos"]), 2), np.float32)
        c.step_trace(4, fr)
    else:
        raise SystemExit(f"unknown case {name}")
    print("case", name, "ok")


if __name__ == "__main__":
    run_case(sys.argv[1])
