"""ctypes binding of the fp64 CPU oracle (oracle/liborca_oracle.so).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this module.  The product path
(``paper_1908_10107_b200``) never imports it and shares no code with it.

Every function here is argument marshalling over ``oracle/orca_oracle.c``; the
arithmetic (and its citations into PAPER.md) lives there.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborca_oracle.so")

FLAG_INFEASIBLE = 0x01
FLAG_G1 = 0x02
FLAG_G2 = 0x04
FLAG_G3 = 0x08
FLAG_G4 = 0x10
FLAG_DEGENERATE = 0x16  # g1 | g2 | g4 (g3 reported, not excluded: DESIGN.md Q21)
FLAG_NARROW = 0x20

BRANCH_COLLISION = 1
BRANCH_CUTOFF = 2
BRANCH_LEFT = 4
BRANCH_RIGHT = 8
BRANCH_DEGENERATE = 16


class Params(ctypes.Structure):
    _fields_ = [
        ("timeStep", ctypes.c_float),
        ("neighborDist", ctypes.c_float),
        ("maxNeighbors", ctypes.c_int32),
        ("timeHorizon", ctypes.c_float),
        ("radius", ctypes.c_float),
        ("maxSpeed", ctypes.c_float),
    ]


class Agents(ctypes.Structure):
    """or_agents: optional per-agent float[n] arrays (NULL = global value)."""
    _fields_ = [("radius", ctypes.POINTER(ctypes.c_float)), ("maxSpeed", ctypes.POINTER(ctypes.c_float)),
                ("prefSpeed", ctypes.POINTER(ctypes.c_float))]


class LpOrder(ctypes.Structure):
    """or_lp_order: randomized = 0 nearest-first, 1 Fisher-Yates per (seed, step, id)."""
    _fields_ = [("randomized", ctypes.c_int32), ("seed", ctypes.c_uint64), ("step", ctypes.c_int64)]


class Line(ctypes.Structure):
    _fields_ = [("px", ctypes.c_double), ("py", ctypes.c_double),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "orca_oracle.c")
    hdr = os.path.join(_HERE, "orca_oracle.h")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        f32p, f64p = P(ctypes.c_float), P(ctypes.c_double)
        i32p, i64p, u8p, u32p = P(ctypes.c_int32), P(ctypes.c_int64), P(ctypes.c_uint8), P(ctypes.c_uint32)
        L.or_grid_derive.argtypes = [ctypes.c_int64, f32p, ctypes.c_float, f32p, i32p]
        L.or_cells.argtypes = [ctypes.c_int64, f32p, f32p, ctypes.c_float, i32p, i32p, i32p]
        L.or_neighbors.argtypes = [ctypes.c_int64, f32p, f32p, ctypes.c_float, i32p,
                                   ctypes.c_float, ctypes.c_int32, i32p, i32p]
        L.or_orca_line.argtypes = [f32p, f32p, f32p, f32p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, P(Line)]
        L.or_lp2.argtypes = [P(Line), ctypes.c_int, ctypes.c_double, f64p, ctypes.c_int, f64p, u32p]
        L.or_lp3.argtypes = [P(Line), ctypes.c_int, ctypes.c_int, ctypes.c_double, f64p, u32p]
        L.or_lp3.restype = None
        L.or_penetration.argtypes = [P(Line), ctypes.c_int, f64p]
        L.or_penetration.restype = ctypes.c_double
        L.or_solve.argtypes = [P(Line), ctypes.c_int, ctypes.c_double, f64p, f64p, f64p]
        L.or_solve.restype = ctypes.c_uint32
        L.or_step.argtypes = [P(Params), ctypes.c_int64, f32p, f32p, f32p, f32p, ctypes.c_float, P(Agents),
                              P(LpOrder), f32p, i32p, ctypes.c_int64, i64p, f64p, f64p, u8p, f64p, i32p, i32p,
                              f64p, f64p]
        L.or_run.argtypes = [P(Params), ctypes.c_int64, f32p, f32p, f32p, f32p, ctypes.c_float, P(Agents),
                             P(LpOrder), ctypes.c_int32]
        L.or_lp_permutation.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, i32p]
        L.or_lp_permutation.restype = None
        L.or_run.restype = ctypes.c_int64
        _lib = L
    return _lib


def _p(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def make_params(timeStep=0.25, neighborDist=15.0, maxNeighbors=10, timeHorizon=5.0,
                radius=0.5, maxSpeed=1.33) -> Params:
    return Params(timeStep, neighborDist, maxNeighbors, timeHorizon, radius, maxSpeed)


def grid_derive(pos, cs):
    pos = _f32(pos).reshape(-1, 2)
    origin = np.zeros(2, np.float32)
    dims = np.zeros(2, np.int32)
    rc = lib().or_grid_derive(len(pos), _p(pos, ctypes.c_float), cs, _p(origin, ctypes.c_float),
                              _p(dims, ctypes.c_int32))
    if rc != 0:
        raise ValueError("or_grid_derive failed")
    return origin, dims


def cells(pos, origin, cs, dims):
    pos = _f32(pos).reshape(-1, 2)
    origin = _f32(origin)
    dims = np.ascontiguousarray(dims, np.int32)
    cx = np.zeros(len(pos), np.int32)
    cy = np.zeros(len(pos), np.int32)
    lib().or_cells(len(pos), _p(pos, ctypes.c_float), _p(origin, ctypes.c_float), cs,
                   _p(dims, ctypes.c_int32), _p(cx, ctypes.c_int32), _p(cy, ctypes.c_int32))
    return cx, cy


def neighbors(pos, origin, cs, dims, nd, k):
    pos = _f32(pos).reshape(-1, 2)
    origin = _f32(origin)
    dims = np.ascontiguousarray(dims, np.int32)
    n = len(pos)
    nbr = np.full((n, max(k, 1)), -1, np.int32)
    cnt = np.zeros(n, np.int32)
    lib().or_neighbors(n, _p(pos, ctypes.c_float), _p(origin, ctypes.c_float), cs,
                       _p(dims, ctypes.c_int32), nd, k, _p(nbr, ctypes.c_int32), _p(cnt, ctypes.c_int32))
    return nbr[:, :k], cnt


def orca_line(pi, vi, pj, vj, idi, idj, radius, tau, dt, rj=None):
    """Returns ((px, py, dx, dy), branch_mask).  radius = r_i; rj = r_j (default r_i)."""
    out = Line()
    a = [_f32(x) for x in (pi, vi, pj, vj)]
    br = lib().or_orca_line(*[_p(x, ctypes.c_float) for x in a], idi, idj, radius,
                            radius if rj is None else rj, tau, dt, ctypes.byref(out))
    return (out.px, out.py, out.dx, out.dy), br


def _lines(lines):
    lines = np.asarray(lines, np.float64).reshape(-1, 4)
    arr = (Line * max(len(lines), 1))()
    for i, (px, py, dx, dy) in enumerate(lines):
        arr[i] = Line(px, py, dx, dy)
    return arr, len(lines)


def lp2(lines, r, opt, dirOpt=False):
    """Returns (processed_count, v, diag)."""
    arr, n = _lines(lines)
    o = np.ascontiguousarray(opt, np.float64)
    v = np.zeros(2, np.float64)
    diag = ctypes.c_uint32(0)
    f = lib().or_lp2(arr, n, r, _p(o, ctypes.c_double), int(dirOpt), _p(v, ctypes.c_double),
                     ctypes.byref(diag))
    return f, v, diag.value


def lp3(lines, begin, r, v0):
    arr, n = _lines(lines)
    v = np.ascontiguousarray(v0, np.float64).copy()
    diag = ctypes.c_uint32(0)
    lib().or_lp3(arr, n, begin, r, _p(v, ctypes.c_double), ctypes.byref(diag))
    return v, diag.value


def solve(lines, r, pref):
    """LP2 then LP3 from the failure index.  Returns (v, infeasible, diag)."""
    n = len(np.asarray(lines).reshape(-1, 4))
    f, v, d = lp2(lines, r, pref, False)
    if f < n:
        v, d3 = lp3(lines, f, r, v)
        return v, True, d | d3
    return v, False, d


def solve_classify(lines, r, pref):
    """or_solve: the step's solve of one agent plus its flags (INFEASIBLE, G2, G3, G4).
    Returns (v, flags, delta)."""
    arr, n = _lines(lines)
    o = np.ascontiguousarray(pref, np.float64)
    v = np.zeros(2, np.float64)
    d = ctypes.c_double(0.0)
    fl = lib().or_solve(arr, n, r, _p(o, ctypes.c_double), _p(v, ctypes.c_double), ctypes.byref(d))
    return v, int(fl), d.value


def penetration(lines, v):
    arr, n = _lines(lines)
    vv = np.ascontiguousarray(v, np.float64)
    return lib().or_penetration(arr, n, _p(vv, ctypes.c_double))


def lp_permutation(seed, step, agent_id, c):
    """The randomized LP order: idx[slot] = neighbour-order index processed at `slot`."""
    idx = np.zeros(max(c, 1), np.int32)
    lib().or_lp_permutation(seed, step, agent_id, c, _p(idx, ctypes.c_int32))
    return idx[:c]


def _order(lp_seed, lp_step):
    return None if lp_seed is None else ctypes.byref(LpOrder(1, lp_seed, lp_step))


def _agents(props):
    """props: None or dict(radius=, maxSpeed=, prefSpeed=) of float[n] (any may be None)."""
    if not props:
        return None, []
    keep = []
    arrs = []
    for key in ("radius", "maxSpeed", "prefSpeed"):
        v = props.get(key)
        if v is None:
            arrs.append(None)
        else:
            a = np.ascontiguousarray(v, np.float32)
            keep.append(a)
            arrs.append(_p(a, ctypes.c_float))
    return ctypes.byref(Agents(*arrs)), keep


def step(params: Params, pos, vel, pref=None, goals=None, pref_speed=1.0, origin=None, dims=None,
         agents=None, want_nbrs=False, props=None, lp_seed=None, lp_step=0, vtest=None):
    """One synchronous step from the given fp32 state.  If origin/dims are None the grid is
    derived from `pos` (as at set_agents).  props: optional per-agent radius / maxSpeed /
    prefSpeed arrays.  lp_seed: None = nearest-first LP order, else the randomized
    order of (lp_seed, lp_step, id) (reading Q8).  Returns a dict of numpy arrays indexed like `agents` (or by
    id)."""
    agp, _keep = _agents(props)
    pos = _f32(pos).reshape(-1, 2)
    vel = _f32(vel).reshape(-1, 2)
    n = len(pos)
    pref = None if pref is None else _f32(pref).reshape(-1, 2)
    goals = None if goals is None else _f32(goals).reshape(-1, 2)
    if origin is None:
        origin, dims = grid_derive(pos, params.neighborDist)
    origin = _f32(origin)
    dims = np.ascontiguousarray(dims, np.int32)
    if agents is None:
        m = n
        ag = None
    else:
        ag = np.ascontiguousarray(agents, np.int64)
        m = len(ag)
    k = params.maxNeighbors
    vnew = np.zeros((m, 2), np.float64)
    pnew = np.zeros((m, 2), np.float64)
    flags = np.zeros(m, np.uint8)
    delta = np.zeros(m, np.float64)
    nbr = np.full((m, max(k, 1)), -1, np.int32) if want_nbrs else None
    cnt = np.zeros(m, np.int32) if want_nbrs else None
    vt = None if vtest is None else np.ascontiguousarray(vtest, np.float64).reshape(m, 2)
    dt = None if vtest is None else np.zeros(m, np.float64)
    rc = lib().or_step(ctypes.byref(params), n, _p(pos, ctypes.c_float), _p(vel, ctypes.c_float),
                       _p(pref, ctypes.c_float), _p(goals, ctypes.c_float), pref_speed, agp,
                       _order(lp_seed, lp_step), _p(origin, ctypes.c_float), _p(dims, ctypes.c_int32), m, _p(ag, ctypes.c_int64),
                       _p(vnew, ctypes.c_double), _p(pnew, ctypes.c_double), _p(flags, ctypes.c_uint8),
                       _p(delta, ctypes.c_double), _p(nbr, ctypes.c_int32), _p(cnt, ctypes.c_int32),
                       _p(vt, ctypes.c_double), _p(dt, ctypes.c_double))
    if rc != 0:
        raise ValueError("or_step failed")
    out = dict(vel=vnew, pos=pnew, flags=flags, delta=delta, origin=origin, dims=dims)
    if vtest is not None:
        out["dtest"] = dt
    if want_nbrs:
        out["nbr"] = nbr[:, :k]
        out["cnt"] = cnt
    return out


def run(params: Params, pos, vel, pref=None, goals=None, pref_speed=1.0, steps=1, props=None,
        lp_seed=None, lp_step=0):
    """nsteps full steps on fp32 state; returns (pos, vel, infeasible_agent_steps)."""
    agp, _keep = _agents(props)
    pos = _f32(pos).reshape(-1, 2).copy()
    vel = _f32(vel).reshape(-1, 2).copy()
    pref = None if pref is None else _f32(pref).reshape(-1, 2)
    goals = None if goals is None else _f32(goals).reshape(-1, 2)
    r = lib().or_run(ctypes.byref(params), len(pos), _p(pos, ctypes.c_float), _p(vel, ctypes.c_float),
                     _p(pref, ctypes.c_float), _p(goals, ctypes.c_float), pref_speed, agp,
                     _order(lp_seed, lp_step), steps)
    if r < 0:
        raise ValueError("or_run failed")
    return pos, vel, int(r)
