"""Run a few steps of one workload with a chosen LP3 placement (orca_set_lp3_inline), for ncu
captures: python scripts/mode_step.py <config> <mode> <steps>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_10107_b200 import orca as O, workloads as W
cfg, mode, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = W.make(cfg)
c = O.Orca(w["params"])
c.set_agents(w["pos"], w["vel"], w["pref"])
c.set_lp3_inline(mode)
c.step(steps)
print(c.stats())
c.close()
