import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1908_10107_b200 import orca as O, workloads as W
n = int(sys.argv[1]); what = sys.argv[2]
w = W.make("uniform", n=n, rho=0.25)
c = O.Orca(w["params"])
c.set_agents(w["pos"], w["vel"], w["pref"])
c.set_lp3_inline(0)
if what == "warm_then_dry":
    c.set_variant(0); c.step(3); c.set_variant(4)
    v4, f4, nb4, cnt4 = c.debug_step(); print("dry4 ok", flush=True)
    c.set_variant(0); v0, f0, nb0, cnt0 = c.debug_step()
    print("same nb", np.array_equal(nb0, nb4), "cnt", np.array_equal(cnt0, cnt4), "v", np.array_equal(v0, v4), "nan", np.isnan(v4).sum(), flush=True)
    bad = np.nonzero(np.any(nb0 != nb4, axis=1))[0][:5]
    print("bad", bad, nb0[bad], nb4[bad], cnt0[bad], cnt4[bad], flush=True)
elif what == "step0_state":
    c.set_variant(4); c.step(1); p, v = c.get_state()
    print("nan", np.isnan(p).sum(), np.isnan(v).sum(), "maxspeed", np.hypot(*v.T).max(), flush=True)
    c2 = O.Orca(w["params"]); c2.set_agents(w["pos"], w["vel"], w["pref"]); c2.set_lp3_inline(0); c2.step(1); p2, v2 = c2.get_state()
    print("same as v0", np.array_equal(p, p2), np.array_equal(v, v2), flush=True)
