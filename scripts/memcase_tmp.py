import sys
sys.path.insert(0, '/root/repo')
from paper_1908_10107_b200 import orca as O, workloads as W
w = W.make("uniform", n=20000, rho=0.25)
for mode in (0, 1, 2):
    c = O.Orca(w["params"])
    c.set_agents(w["pos"], w["vel"], w["pref"])
    c.set_variant(0)
    c.set_lp3_inline(mode)
    c.step(2)
    c.get_state()
    print("mode", mode, "ok", flush=True)
    c.close()
