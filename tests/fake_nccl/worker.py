"""One rank of a multi-process strips run on a single GPU through the fake NCCL
(tests/test_gpu_nccl_fake.py).  argv: rank world uid_hex out.npz scenario"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
import nccl_scenarios as S  # noqa: E402

rank, world, uid, out, scenario = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
nid = uid.encode().ljust(128, b"\0")
w, run = S.SCENARIOS[scenario]()
ctx = O.Orca(w["params"], device=0, rank=rank, world=world, nccl_id=nid)
ctx.set_transport(int(os.environ.get("ORCA_TEST_TRANSPORT", "0")))
run(ctx, w)
ids, pos, vel = ctx.get_local_state()
st = ctx.stats()
np.savez(out, ids=ids, pos=pos, vel=vel, rebalances=st["rebalances"], infeasible=st["infeasible"],
         collision_pairs=st["collision_pairs"], removed=st["removed"])
ctx.close()
