"""Probe: can two NCCL ranks share one GPU here (to exercise the strips' NCCL transport on a
one-GPU box)?  Run: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/nccl_same_gpu_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
nid = O.nccl_unique_id() if rank == 0 else bytes(128)
obj = [nid]
dist.broadcast_object_list(obj, 0)
w = W.make("uniform", n=20000, rho=0.3)
try:
    ctx = O.Orca(w["params"], device=0, rank=rank, world=world, nccl_id=obj[0])
    ctx.set_agents(w["pos"], w["vel"], w["pref"])
    ctx.step(10)
    ids, p, v = ctx.get_local_state()
    parts = [None] * world
    dist.all_gather_object(parts, (ids, p, v))
    if rank == 0:
        ref = O.Orca(w["params"])
        ref.set_agents(w["pos"], w["vel"], w["pref"])
        ref.step(10)
        rp, rv = ref.get_state()
        gp = np.full_like(rp, np.nan)
        gv = np.full_like(rv, np.nan)
        for i_, p_, v_ in parts:
            gp[i_] = p_
            gv[i_] = v_
        print("NCCL strips vs 1 GPU bit-identical:", np.array_equal(gp, rp) and np.array_equal(gv, rv), flush=True)
    ctx.rebalance()
    ctx.step(10)
    print(f"rank {rank}: rebalance + 10 steps ok, local {ctx.count()}", flush=True)
except Exception as e:
    print(f"rank {rank}: {type(e).__name__}: {e}", flush=True)
dist.barrier()
