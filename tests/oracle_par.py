"""The fp64 oracle (test infrastructure) on all host cores: forked processes each run
``oracle.step`` on a disjoint slice of the agents of ONE pre-step state (every process bins
the full state, as the oracle does).  The per-agent results are independent of the split
(each agent's step reads only the pre-step state), so this equals one ``oracle.step`` call
-- ``tests/test_oracle_pins.py::test_step_subset_equals_full`` pins that -- and makes the
exhaustive full-size parity cases (100k - 4M agents) take seconds instead of minutes."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_JOB = {}


def _work(chunk):
    from oracle import oracle as O
    j = _JOB
    vt = None if j["vtest"] is None else j["vtest"][chunk]
    return O.step(j["params"], j["pos"], j["vel"], agents=chunk, vtest=vt, **j["kw"])


def procs() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def step(params, pos, vel, agents=None, vtest=None, nproc=None, **kw):
    """oracle.step over `agents` (default: all, by id) split across `nproc` forked workers;
    returns the same dict, indexed like `agents`."""
    from oracle import oracle as O
    O.lib()  # build / load before forking
    n = len(pos)
    ids = np.arange(n, dtype=np.int64) if agents is None else np.asarray(agents, np.int64)
    vt = None if vtest is None else np.asarray(vtest, np.float64).reshape(-1, 2)
    if vt is not None and agents is None:
        vt = vt[:n]
    nproc = nproc or procs()
    if nproc == 1 or len(ids) < 20000:
        return O.step(params, pos, vel, agents=ids, vtest=vt, **kw)
    # vtest is looked up by position in `ids`, so hand the workers index slices
    _JOB.clear()
    _JOB.update(params=params, pos=np.ascontiguousarray(pos, np.float32), vel=np.ascontiguousarray(vel, np.float32),
                vtest=None, kw=kw)
    parts = np.array_split(np.arange(len(ids)), nproc)
    if vt is not None:
        _JOB["vtest"] = np.zeros((n, 2), np.float64)  # by agent id (ids are distinct)
        _JOB["vtest"][ids] = vt
    with mp.get_context("fork").Pool(nproc) as pool:
        outs = pool.map(_work, [ids[pp] for pp in parts])
    res = {}
    for key in outs[0]:
        if key in ("origin", "dims"):
            res[key] = outs[0][key]
        else:
            res[key] = np.concatenate([o[key] for o in outs], axis=0)
    return res
