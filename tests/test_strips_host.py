"""Host-side logic of the strip decomposition, CPU only.

* the C-ABI partition function (no GPU needed);
* a world_size-2 gloo run of the exchange protocol the CUDA runtime implements: each rank
  owns a strip of grid columns, and every step sends one buffer per neighbour holding
  (a) its emigrants and (b) its stayers in the edge column; the receiver appends (a) as
  owned agents and (b) as ghosts, and adds its own emigrants as ghosts.  After every step
  each rank's owned and ghost sets must equal the global truth.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest


@pytest.fixture(scope="module")
def orca():
    from paper_1908_10107_b200 import build
    build.build()
    from paper_1908_10107_b200 import orca as O
    return O


def test_partition_balanced_and_contiguous(orca):
    rng = np.random.default_rng(0)
    for nx in (1, 5, 40, 137):
        counts = rng.integers(0, 1000, nx)
        for world in range(1, min(nx, 9) + 1):
            b = orca.partition_columns(counts, world)
            assert b[0] == 0 and b[-1] == nx
            assert np.all(np.diff(b) >= 1)
            if world > 1 and counts.sum() > 0:
                loads = [counts[b[s]:b[s + 1]].sum() for s in range(world)]
                assert max(loads) <= counts.sum() / world + counts.max() + 1


def test_partition_errors(orca):
    with pytest.raises(orca.OrcaError):
        orca.partition_columns(np.ones(3, np.int64), 4)
    with pytest.raises(orca.OrcaError):
        orca.partition_columns(np.array([1, -1, 2], np.int64), 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _protocol_worker(rank, world, port, steps, result):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(42)  # same global truth on every rank
    n, nx, cs = 3000, 12, 15.0
    pos = rng.uniform(0, nx * cs, n)
    ids = np.arange(n)
    col = lambda x: np.clip(np.floor(x / cs).astype(int), 0, nx - 1)
    counts = np.bincount(col(pos), minlength=nx)
    from paper_1908_10107_b200 import orca as O
    b = O.partition_columns(counts, world)
    c0, c1 = int(b[rank]), int(b[rank + 1])
    own = ids[(col(pos) >= c0) & (col(pos) < c1)]
    ghost = ids[(col(pos) == c0 - 1) | (col(pos) == c1)]
    ok = True
    for step in range(steps):
        disp = np.random.default_rng(1000 + step).uniform(-0.9, 0.9, n) * cs  # |move| < one column
        pos = np.clip(pos + disp, -20.0, nx * cs + 20.0)
        cnew = col(pos[own])
        stay = own[(cnew >= c0) & (cnew < c1)]
        emL = own[cnew < c0]
        emR = own[cnew >= c1]
        send = {}
        if rank > 0:
            send[rank - 1] = (emL, stay[col(pos[stay]) == c0])
        if rank < world - 1:
            send[rank + 1] = (emR, stay[col(pos[stay]) == c1 - 1])
        recv = {}
        pending = []
        for peer, (em, halo) in send.items():
            msg = torch.tensor(np.concatenate([[len(em), len(halo)], em, halo]), dtype=torch.int64)
            ln = torch.tensor([len(msg)], dtype=torch.int64)
            pending.append(dist.isend(ln, peer))
            pending.append(dist.isend(msg, peer))
            pending.append((ln, msg))
        for peer in send:
            ln = torch.zeros(1, dtype=torch.int64)
            dist.recv(ln, peer)
            msg = torch.zeros(int(ln.item()), dtype=torch.int64)
            dist.recv(msg, peer)
            m = msg.numpy()
            recv[peer] = (m[2:2 + m[0]], m[2 + m[0]:2 + m[0] + m[1]])
        for h in pending:
            if hasattr(h, "wait"):
                h.wait()
        imm = np.concatenate([recv[p][0] for p in recv] + [np.zeros(0, int)])
        own = np.concatenate([stay, imm])
        ghost = np.concatenate([recv[p][1] for p in recv] + [emL, emR])
        # global truth
        call = col(pos)
        true_own = ids[(call >= c0) & (call < c1)]
        true_ghost = ids[(call == c0 - 1) | (call == c1)]
        ok &= np.array_equal(np.sort(own), true_own) and np.array_equal(np.sort(ghost), true_ghost)
    result[rank] = bool(ok)
    dist.destroy_process_group()


def test_exchange_protocol_gloo_world2():
    import torch.multiprocessing as mp
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_protocol_worker, args=(2, port, 25, result), nprocs=2, join=True)
    assert result[0] and result[1]


def test_exchange_protocol_gloo_world3():
    import torch.multiprocessing as mp
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_protocol_worker, args=(3, port, 15, result), nprocs=3, join=True)
    assert all(result[r] for r in range(3))
