"""Thin Python binding of liborca (include/orca.h).  Argument marshalling only: every
step of the ORCA update runs in the library's CUDA kernels.  There is no CPU fallback --
importing this module raises if liborca.so is missing or cannot be loaded.

Arrays may be numpy arrays (host) or CUDA torch tensors (device); both are passed to the
library as raw pointers, which dispatches through unified addressing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liborca.so")
# tests only: ORCA_LIB selects another build of this same library -- liborca_test.so, built
# with -DORCA_TEST_HOOKS so the multi-process tests can swap in their NCCL stand-in
LIB_PATH = os.environ.get("ORCA_LIB") or LIB_PATH

ORCA_MAX_K = 32
STATUS = {0: "ok", 1: "invalid argument", 2: "not ready", 3: "out of memory", 4: "CUDA error",
          5: "NCCL error", 6: "capacity exceeded", 7: "internal error"}

# names declared in include/orca.h (checked by tests/test_capi.py)
EXPORTS = [
    "orca_create", "orca_destroy", "orca_set_agents", "orca_set_goals", "orca_step", "orca_get_state",
    "orca_get_count", "orca_get_grid", "orca_debug_cells", "orca_debug_step", "orca_get_stats",
    "orca_reset_stats", "orca_get_stream", "orca_step_timed", "orca_status_string", "orca_last_error",
    "orca_nccl_unique_id", "orca_create_dist", "orca_get_local_state", "orca_debug_work",
    "orca_create_strips", "orca_partition_columns", "orca_get_strips", "orca_set_variant",
    "orca_set_goal_removal", "orca_get_active", "orca_set_agent_props", "orca_step_trace",
    "orca_set_lp_order", "orca_set_lp3_lanes", "orca_set_lp3_inline", "orca_set_overlap", "orca_rebalance", "orca_set_transport",
    "orca_get_transport", "orca_set_state", "orca_set_state_async", "orca_get_state_async",
    "orca_io_wait", "orca_step_io_async", "orca_get_launch_info", "orca_get_kernel_config", "orca_probe_alu", "orca_get_comm_info",
]


class OrcaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"liborca: {STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("timeStep", ctypes.c_float), ("neighborDist", ctypes.c_float),
                ("maxNeighbors", ctypes.c_int32), ("timeHorizon", ctypes.c_float),
                ("radius", ctypes.c_float), ("maxSpeed", ctypes.c_float)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("steps", "agent_updates", "infeasible", "degenerate",
                                               "coincident", "eps_parallel", "marginal", "collision_pairs",
                                               "removed", "rebalances", "regrids")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_1908_10107_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    P = ctypes.POINTER
    sig = {
        "orca_create": [P(Params), i32, P(vp)],
        "orca_destroy": [vp],
        "orca_set_agents": [vp, i64, vp, vp, vp],
        "orca_set_goals": [vp, vp, f32],
        "orca_step": [vp, i32],
        "orca_get_state": [vp, vp, vp],
        "orca_get_count": [vp, P(i64)],
        "orca_get_grid": [vp, P(ctypes.c_double), P(f32), P(i32)],
        "orca_debug_cells": [vp, vp, vp],
        "orca_debug_step": [vp, vp, vp, vp, vp],
        "orca_get_stats": [vp, P(Stats)],
        "orca_reset_stats": [vp],
        "orca_get_stream": [vp, P(vp)],
        "orca_step_timed": [vp, i32, P(ctypes.c_double)],
        "orca_status_string": [i32],
        "orca_last_error": [],
        "orca_nccl_unique_id": [vp],
        "orca_create_dist": [P(Params), i32, i32, i32, vp, P(vp)],
        "orca_get_local_state": [vp, vp, vp, vp],
        "orca_debug_work": [vp, P(i64)],
        "orca_create_strips": [P(Params), i32, i32, P(vp)],
        "orca_partition_columns": [P(i64), i32, i32, P(i32)],
        "orca_get_strips": [vp, P(i32)],
        "orca_set_variant": [vp, i32],
        "orca_set_goal_removal": [vp, f32],
        "orca_get_active": [vp, vp],
        "orca_set_agent_props": [vp, vp, vp, vp],
        "orca_step_trace": [vp, i32, vp, vp],
        "orca_set_lp_order": [vp, i32, ctypes.c_uint64, i64],
        "orca_set_lp3_lanes": [vp, i32],
        "orca_set_lp3_inline": [vp, i32],
        "orca_set_overlap": [vp, i32],
        "orca_rebalance": [vp],
        "orca_set_transport": [vp, i32],
        "orca_get_transport": [vp, P(i32)],
        "orca_set_state": [vp, vp, vp],
        "orca_set_state_async": [vp, vp, vp],
        "orca_step_io_async": [vp, vp, vp, vp, vp],
        "orca_get_state_async": [vp, vp, vp],
        "orca_io_wait": [vp],
        "orca_get_launch_info": [vp, P(i32)],
        "orca_get_kernel_config": [vp, P(i32)],
        "orca_probe_alu": [i32, P(ctypes.c_double)],
        "orca_get_comm_info": [vp, P(i32)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = i32
    L.orca_destroy.restype = None
    L.orca_status_string.restype = ctypes.c_char_p
    L.orca_last_error.restype = ctypes.c_char_p
    return L


_lib = _load()


def lib():
    return _lib


def _check(st: int):
    if st != 0:
        raise OrcaError(st, _lib.orca_last_error().decode())


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(type(a))


def _as_f32(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float32)
    return a  # torch tensors: caller supplies float32 contiguous


def _io_arg(a):
    """Buffers of the asynchronous calls are used as they are (no conversion copy that could
    be freed while the transfer is in flight)."""
    if a is None:
        return None
    dt = getattr(a, "dtype", None)
    if str(dt) not in ("float32", "torch.float32"):
        raise TypeError("asynchronous I/O buffers must be float32")
    return a


def make_params(timeStep=0.25, neighborDist=15.0, maxNeighbors=10, timeHorizon=5.0, radius=0.5,
                maxSpeed=1.33) -> Params:
    return Params(timeStep, neighborDist, maxNeighbors, timeHorizon, radius, maxSpeed)


def partition_columns(col_count, world: int):
    """Strip bounds (int32[world+1]) for per-column agent counts (host only)."""
    cc = np.ascontiguousarray(col_count, np.int64)
    b = np.zeros(world + 1, np.int32)
    _check(_lib.orca_partition_columns(cc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(cc), world,
                                       b.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return b


def probe_alu(device: int = 0) -> dict:
    """orca_probe_alu: measured FP32 / FP64 FMA lane-op rates and the SM clock they ran at."""
    out = (ctypes.c_double * 4)()
    _check(_lib.orca_probe_alu(device, out))
    return dict(fp32_lane_ops_per_s=out[0], fp64_lane_ops_per_s=out[1], sm_mhz=out[2], fp32_lanes_per_sm_clk=out[3])


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.orca_nccl_unique_id(buf))
    return buf.raw


class Orca:
    """One liborca context (orca_create / orca_create_dist ... orca_destroy)."""

    def __init__(self, params: Params | dict | None = None, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, strips: int = 0):
        if params is None:
            params = make_params()
        elif isinstance(params, dict):
            params = make_params(**params)
        self.params = params
        self._ctx = ctypes.c_void_p()
        self._io_keep = []
        self.strips = max(1, strips)
        if strips:
            _check(_lib.orca_create_strips(ctypes.byref(params), device, strips, ctypes.byref(self._ctx)))
        elif world == 1:
            _check(_lib.orca_create(ctypes.byref(params), device, ctypes.byref(self._ctx)))
        else:
            idb = ctypes.create_string_buffer(nccl_id, 128)
            _check(_lib.orca_create_dist(ctypes.byref(params), device, rank, world, idb, ctypes.byref(self._ctx)))
        self.n = 0

    def close(self):
        if self._ctx:
            _lib.orca_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state
    def set_agents(self, pos, vel, pref):
        pos, vel, pref = _as_f32(pos), _as_f32(vel), _as_f32(pref)
        n = (pos.shape[0] if pos.ndim == 2 else pos.shape[0] // 2)
        _check(_lib.orca_set_agents(self._ctx, n, _ptr(pos), _ptr(vel), _ptr(pref)))
        self.n = n

    def set_state(self, pos, vel):
        """New positions / velocities of the loaded agents (by id); everything else stays."""
        _check(_lib.orca_set_state(self._ctx, _ptr(_as_f32(pos)), _ptr(_as_f32(vel))))

    def set_state_async(self, pos, vel):
        """orca_set_state_async: enqueue the upload + re-binning without synchronising.  pos / vel
        must be float32 C-contiguous (pinned torch tensors for the overlap) and stay untouched
        until io_wait()."""
        self._io_keep.extend((_io_arg(pos), _io_arg(vel)))
        _check(_lib.orca_set_state_async(self._ctx, _ptr(pos), _ptr(vel)))

    def get_state_async(self, pos=None, vel=None):
        """orca_get_state_async: enqueue the read-back of the state after the enqueued steps into
        pos / vel (float32 C-contiguous, either None); valid after io_wait()."""
        self._io_keep.extend((_io_arg(pos), _io_arg(vel)))
        _check(_lib.orca_get_state_async(self._ctx, _ptr(pos), _ptr(vel)))

    def step_io_async(self, pos_in, vel_in, pos_out=None, vel_out=None):
        """orca_step_io_async: upload, one step and read-back in one enqueued call (float32
        C-contiguous buffers, pinned for the overlap, untouched until io_wait())."""
        self._io_keep.extend((_io_arg(pos_in), _io_arg(vel_in), _io_arg(pos_out), _io_arg(vel_out)))
        _check(_lib.orca_step_io_async(self._ctx, _ptr(pos_in), _ptr(vel_in), _ptr(pos_out), _ptr(vel_out)))

    def io_wait(self):
        """orca_io_wait: every enqueued upload, step and read-back is complete."""
        try:
            _check(_lib.orca_io_wait(self._ctx))
        finally:
            self._io_keep.clear()

    def set_goals(self, goals, pref_speed: float):
        _check(_lib.orca_set_goals(self._ctx, _ptr(_as_f32(goals)), pref_speed))

    def step(self, n_steps: int = 1):
        _check(_lib.orca_step(self._ctx, n_steps))

    def step_trace(self, n_steps: int, frames=None, vframes=None, with_vel: bool = False):
        """Run n_steps and return per-step positions (n_steps, n, 2) (and velocities): the
        paper's per-step dump for visualisation.  Pass pinned torch tensors to
        overlap the copies with the simulation."""
        if frames is None:
            frames = np.empty((n_steps, self.n, 2), np.float32)
            if with_vel:
                vframes = np.empty((n_steps, self.n, 2), np.float32)
        _check(_lib.orca_step_trace(self._ctx, n_steps, _ptr(frames), _ptr(vframes)))
        return (frames, vframes) if vframes is not None else frames

    def step_timed(self, n_steps: int):
        ms = (ctypes.c_double * 4)()
        _check(_lib.orca_step_timed(self._ctx, n_steps, ms))
        return list(ms)

    def count(self) -> int:
        n = ctypes.c_int64()
        _check(_lib.orca_get_count(self._ctx, ctypes.byref(n)))
        return n.value

    def get_state(self, pos=None, vel=None):
        """Into caller buffers (numpy or torch) if given, else new numpy arrays."""
        if pos is None and vel is None:
            pos = np.empty((self.n, 2), np.float32)
            vel = np.empty((self.n, 2), np.float32)
        _check(_lib.orca_get_state(self._ctx, _ptr(pos), _ptr(vel)))
        return pos, vel

    def get_local_state(self):
        n = self.count()
        ids = np.empty(n, np.int32)
        pos = np.empty((n, 2), np.float32)
        vel = np.empty((n, 2), np.float32)
        _check(_lib.orca_get_local_state(self._ctx, _ptr(ids), _ptr(pos), _ptr(vel)))
        return ids, pos, vel

    def strip_bounds(self):
        b = np.zeros(2 * self.strips, np.int32)
        _check(_lib.orca_get_strips(self._ctx, b.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return b.reshape(-1, 2)

    def grid(self):
        o = (ctypes.c_double * 2)()
        cs = ctypes.c_float()
        d = (ctypes.c_int32 * 2)()
        _check(_lib.orca_get_grid(self._ctx, o, ctypes.byref(cs), d))
        return np.array([o[0], o[1]], np.float64), cs.value, np.array([d[0], d[1]], np.int32)

    def debug_cells(self):
        """(cx, cy) int32[n] by id (all ids of set_agents; removed agents are -1)."""
        n = self.n
        cx = np.empty(n, np.int32)
        cy = np.empty(n, np.int32)
        _check(_lib.orca_debug_cells(self._ctx, _ptr(cx), _ptr(cy)))
        return cx, cy

    def debug_step(self):
        """(vnew (n,2) f32, flags u8, nbr (n,k) int32, cnt int32) by id for the current
        state (removed agents: NaN velocity, cnt -1)."""
        n = self.n
        k = self.params.maxNeighbors
        v = np.empty((n, 2), np.float32)
        fl = np.empty(n, np.uint8)
        nb = np.empty((n, max(k, 1)), np.int32)
        cnt = np.empty(n, np.int32)
        _check(_lib.orca_debug_step(self._ctx, _ptr(v), _ptr(fl), _ptr(nb) if k > 0 else None, _ptr(cnt)))
        return v, fl, nb[:, :k], cnt

    def work(self) -> dict:
        out = (ctypes.c_int64 * 6)()
        _check(_lib.orca_debug_work(self._ctx, out))
        return dict(cand=out[0], lines=out[1], checks=out[2], lp1=out[3], proj=out[4], stencil=out[5])

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.orca_get_stats(self._ctx, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check(_lib.orca_reset_stats(self._ctx))

    def set_agent_props(self, radius=None, max_speed=None, pref_speed=None):
        """Per-agent radius / maxSpeed / prefSpeed (float[n] by id, each optional)."""
        arrs = [None if a is None else _as_f32(np.asarray(a) if not hasattr(a, "data_ptr") else a)
                for a in (radius, max_speed, pref_speed)]
        _check(_lib.orca_set_agent_props(self._ctx, *[_ptr(a) for a in arrs]))

    def set_goal_removal(self, radius: float):
        """Remove agents within `radius` of their goal after a step; 0 disables."""
        _check(_lib.orca_set_goal_removal(self._ctx, radius))

    def set_transport(self, mode: int):
        """Strip exchange: 0 = peer memory (k_push + arrival flags, default), 1 = NCCL
        send/recv (loopback: device copies); every rank must call it together."""
        _check(_lib.orca_set_transport(self._ctx, mode))

    def transport(self) -> int:
        m = ctypes.c_int32()
        _check(_lib.orca_get_transport(self._ctx, ctypes.byref(m)))
        return m.value

    def launch_info(self) -> dict:
        """orca_get_launch_info: the kernels one step launches (first strip)."""
        out = (ctypes.c_int32 * 4)()
        _check(_lib.orca_get_launch_info(self._ctx, out))
        return dict(variant=out[0], lp3_lanes=out[1], kernels_per_step=out[2], transport=out[3])

    def kernel_config(self) -> dict:
        """orca_get_kernel_config: the step-kernel instantiation the first strip runs."""
        out = (ctypes.c_int32 * 6)()
        _check(_lib.orca_get_kernel_config(self._ctx, out))
        return dict(variant=out[0], lp3_placement=out[1], compiled_for_lp3=out[2], mono=out[3],
                    threads=out[4], min_blocks_per_sm=out[5])

    def comm_info(self) -> dict:
        """orca_get_comm_info: world, rank and the rank count of liborca's NCCL communicator."""
        out = (ctypes.c_int32 * 3)()
        _check(_lib.orca_get_comm_info(self._ctx, out))
        return dict(world=out[0], rank=out[1], comm_ranks=out[2])

    def rebalance(self):
        """Re-partition the strips from the current state (automatic when a strip nears its
        capacities; every rank must call it together)."""
        _check(_lib.orca_rebalance(self._ctx))

    def set_overlap(self, mode: int):
        """Strips: -1 automatic, 0 off, 1 on -- boundary columns first, exchange concurrent
        with the interior columns."""
        _check(_lib.orca_set_overlap(self._ctx, mode))

    def set_lp3_inline(self, mode: int):
        """-1 automatic, 0 always queue for k_lp3, 1 inside the step kernel per thread, 2 inside
        the step kernel on the block's compacted queue."""
        _check(_lib.orca_set_lp3_inline(self._ctx, mode))

    def set_lp3_lanes(self, lanes: int):
        """Lanes per infeasible agent in the LP3 kernel: -1 (auto), 1 (thread), 4, 8 or 16; same results."""
        _check(_lib.orca_set_lp3_lanes(self._ctx, lanes))

    def set_lp_order(self, mode, seed: int = 0, first_step: int = 0):
        """LP constraint order (reading Q8): 0 / False = greedy (most violated next, the
        default); 1 / True = the counter-based Fisher-Yates order of (seed, t, id), t =
        first_step for the next step and +1 per step (the oracle's lp_seed / lp_step); 2 =
        neighbour order, sequential (the oracle's default order)."""
        _check(_lib.orca_set_lp_order(self._ctx, int(mode), seed, first_step))

    def active(self):
        a = np.empty(self.n, np.uint8)
        _check(_lib.orca_get_active(self._ctx, _ptr(a)))
        return a.astype(bool)

    def set_variant(self, variant: int):
        """-1 = automatic (default), 0 = thread per agent, 1 = 8-lane group per agent,
        2 = register top-k list, 3 = work-unit LP2; all give the same results."""
        _check(_lib.orca_set_variant(self._ctx, variant))

    def stream(self) -> int:
        s = ctypes.c_void_p()
        _check(_lib.orca_get_stream(self._ctx, ctypes.byref(s)))
        return s.value or 0
