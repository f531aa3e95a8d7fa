"""The strips' multi-rank (NCCL) code path, end to end, with several processes on ONE GPU.

Real NCCL refuses two ranks on one device, so the processes load the host-staged stand-in
tests/fake_nccl (ORCA_NCCL_LIB): the same ncclSend/ncclRecv groups inside the captured step
graphs, the same ncclAllReduce / ncclAllGather of the rebalance, with message sizes checked.
Every rank's strip, assembled by id, must equal the single-GPU run bit for bit
(DESIGN.md §8)."""
import os
import secrets
import subprocess
import sys

import numpy as np
import pytest

import nccl_scenarios as S

HERE = os.path.dirname(os.path.abspath(__file__))
FAKE_DIR = os.path.join(HERE, "fake_nccl")
FAKE_LIB = os.path.join(FAKE_DIR, "libfakenccl.so")


def _test_lib():
    """liborca_test.so: the product sources built with -DORCA_TEST_HOOKS, the only build that
    honours ORCA_NCCL_LIB (the product liborca.so never loads another NCCL)."""
    from paper_1908_10107_b200 import build
    return build.build(test_hooks=True)


def _build_fake():
    src = os.path.join(FAKE_DIR, "fake_nccl.cu")
    if os.path.exists(FAKE_LIB) and os.path.getmtime(FAKE_LIB) >= os.path.getmtime(src):
        return FAKE_LIB
    subprocess.run(["nvcc", "-shared", "-Xcompiler", "-fPIC", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", FAKE_LIB, src, "-lrt"], check=True)
    return FAKE_LIB


@pytest.fixture(scope="module")
def orca():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1908_10107_b200 import build
    build.build()
    from paper_1908_10107_b200 import orca as O
    return O


@pytest.mark.gpu
@pytest.mark.parametrize("world,scenario,transport", [(2, "uniform", 0), (3, "uniform", 0), (4, "convergent", 0),
                                                      (3, "uniform", 1), (4, "convergent", 1)])
def test_multirank_strips_bit_identical(orca, tmp_path, world, scenario, transport):
    """transport 0: peer memory (k_push into cudaIpc-mapped receive buffers + arrival flags);
    1: ncclSend/ncclRecv of the whole buffers (through the stand-in)."""
    lib = _build_fake()
    uid = "/orca_fake_" + secrets.token_hex(8)
    env = dict(os.environ, ORCA_NCCL_LIB=lib, ORCA_LIB=_test_lib(), ORCA_TEST_TRANSPORT=str(transport))
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"rank{r}.npz")
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, os.path.join(FAKE_DIR, "worker.py"), str(r), str(world), uid,
                                       out, scenario], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o.decode(errors="replace")[-2000:])
    assert all(p.returncode == 0 for p in procs), logs
    # single-GPU reference
    w, run = S.SCENARIOS[scenario]()
    ref = orca.Orca(w["params"])
    run(ref, w)
    rp, rv = ref.get_state()
    rs = ref.stats()
    n = len(w["pos"])
    gp = np.full((n, 2), np.nan, np.float32)
    gv = np.full((n, 2), np.nan, np.float32)
    seen = np.zeros(n, np.int64)
    tot = {"infeasible": 0, "collision_pairs": 0, "removed": 0}
    rebal = []
    for out in outs:
        d = np.load(out)
        gp[d["ids"]] = d["pos"]
        gv[d["ids"]] = d["vel"]
        seen[d["ids"]] += 1
        for k in tot:
            tot[k] += int(d[k])
        rebal.append(int(d["rebalances"]))
    assert np.all(seen == 1)  # every agent owned by exactly one rank
    assert np.array_equal(gp, rp) and np.array_equal(gv, rv)
    for k in ("infeasible", "collision_pairs", "removed"):
        assert tot[k] == rs[k], k
    assert len(set(rebal)) == 1 and rebal[0] >= 1  # every rank rebalanced together
    ref.close()


@pytest.mark.gpu
def test_bench_multirank_shared_gpu(orca, tmp_path):
    """bench.py's N>1 path (torchrun, per-rank strips, max-over-ranks timing, e2e gather) on
    one GPU through the fake NCCL: one valid JSON line from rank 0."""
    import json
    lib = _build_fake()
    env = dict(os.environ, ORCA_NCCL_LIB=lib, ORCA_LIB=_test_lib())
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(29600 + secrets.randbelow(300)), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--config", "uniform", "--e2e-steps", "2",
           "--shared-gpu"]
    r = subprocess.run(cmd, env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "strips2"
    assert d["config"]["exchange"] == "nccl"  # the multi-rank default
    assert d["comm"]["comm_ranks"] == [2, 2]  # every rank's liborca communicator holds 2 ranks
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["roofline"]["frac"] > 0


@pytest.mark.gpu
def test_bench_self_launch_shared_gpu(orca):
    """`python bench.py --gpus 2` WITHOUT torchrun starts its two ranks itself and reports
    n_gpus 2; a rank count that disagrees with --gpus exits non-zero."""
    import json
    lib = _build_fake()
    env = dict(os.environ, ORCA_NCCL_LIB=lib, ORCA_LIB=_test_lib())
    env.pop("WORLD_SIZE", None)
    root = os.path.dirname(HERE)
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "uniform", "--e2e-steps", "1", "--shared-gpu"]
    r = subprocess.run(cmd, env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "strips2"
    bad = subprocess.run(cmd, env=dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"), cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert bad.returncode != 0
