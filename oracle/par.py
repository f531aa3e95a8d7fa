"""The fp64 oracle stepping a WHOLE crowd on all host cores -- TEST / BASELINE INFRASTRUCTURE
ONLY (bench.py's cpu_baseline and --impl reference legs; see oracle.py's header).

Each step every worker process runs ``or_step`` (oracle/orca_oracle.c, unchanged) on a
disjoint contiguous slice of the agent ids of the same pre-step state; the state lives in
shared memory, so nothing but slice bounds crosses process boundaries.  Per agent the result
is exactly the single-process one (an agent's step reads only the pre-step state; pinned by
tests/test_oracle_pins.py::test_step_subset_equals_full), and the state update between steps
is or_run's: vel <- fl32(v'), pos <- fl32(p + dt v') on the grid frozen at the start."""
from __future__ import annotations

import ctypes
import multiprocessing as mp
import os
import time

import numpy as np

from oracle import oracle as O

_S = {}


def host_cores() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mp.RawArray(ctypes.c_char, max(n, 1))
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _work(job):
    lo, hi = job
    s = _S
    ids = np.arange(lo, hi, dtype=np.int64)
    r = O.step(s["params"], s["pos"], s["vel"], pref=s["pref"], goals=s["goals"], pref_speed=s["pref_speed"],
               origin=s["origin"], dims=s["dims"], agents=ids)
    s["vout"][lo:hi] = r["vel"]
    s["pout"][lo:hi] = r["pos"]
    s["flags"][lo:hi] = r["flags"]
    return hi - lo


class ParallelOracle:
    """oracle steps of one crowd on `procs` forked workers (default: every host core)."""

    def __init__(self, params, pos, vel, pref=None, goals=None, pref_speed=1.0, procs=None):
        O.lib()  # build / load before forking
        n = len(pos)
        self.n = n
        self.procs = procs or host_cores()
        self.params = params
        _S.clear()
        _S.update(params=params, pref_speed=pref_speed,
                  pos=_shared((n, 2), np.float32), vel=_shared((n, 2), np.float32),
                  vout=_shared((n, 2), np.float64), pout=_shared((n, 2), np.float64),
                  flags=_shared((n,), np.uint8),
                  pref=None if pref is None else np.ascontiguousarray(pref, np.float32),
                  goals=None if goals is None else np.ascontiguousarray(goals, np.float32))
        _S["pos"][:] = pos
        _S["vel"][:] = vel
        origin, dims = O.grid_derive(_S["pos"], params.neighborDist)  # frozen grid (reading Q12)
        _S["origin"], _S["dims"] = origin, dims
        self.pool = mp.get_context("fork").Pool(self.procs)
        b = np.linspace(0, n, self.procs * 2 + 1).astype(np.int64)
        self.jobs = [(int(b[q]), int(b[q + 1])) for q in range(len(b) - 1) if b[q + 1] > b[q]]
        self.infeasible = 0

    def step(self, steps: int = 1) -> float:
        """`steps` full synchronous steps; returns the wall-clock seconds they took."""
        t0 = time.perf_counter()
        for _ in range(steps):
            self.pool.map(_work, self.jobs)
            _S["vel"][:] = _S["vout"].astype(np.float32)
            _S["pos"][:] = _S["pout"].astype(np.float32)
            self.infeasible += int(np.count_nonzero(_S["flags"] & O.FLAG_INFEASIBLE))
        return time.perf_counter() - t0

    def state(self):
        return _S["pos"].copy(), _S["vel"].copy()

    def close(self):
        self.pool.close()
        self.pool.join()
