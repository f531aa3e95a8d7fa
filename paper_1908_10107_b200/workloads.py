"""Seeded synthetic crowd generators (numpy only).

This module is the ONE piece shared by the CUDA path's tests/bench and the oracle: it
holds no ORCA arithmetic, only input recipes (DESIGN.md §6 "Input recipe").  Every array
is float32 (the ABI's state type), x,y interleaved, shape (n, 2).

Mapping to the paper's workloads (§4):
  * ``circle``   -- convergent multi-directional flow (the 8-way / vortex idea) at
                    small scale; goal-seeking pref, paper pedestrian r/speeds.
  * ``corridor`` -- the 2-way crossing structure: two opposing flows, ids
                    alternate direction; held-constant pref, no goals/removal.
  * ``uniform``  -- generic uniform crowds for throughput, as in the averaged timing runs
                    (P:156); density rho in agents/m^2.
Start positions never overlap ("Random spawn locations are chosen so that there is
no overlap"): a jittered lattice with spacing s = rho^-1/2 and jitter +-0.99 (s-2r)/2.
Agent ids (= array index) are a random permutation of lattice order, so storage order
is uncorrelated with position and the binning stage does real work.
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 190810107

# Global parameters (reading Q1 in DESIGN.md): dt 0.25, k 10 (BASELINE configs); nd 15,
# tau 5; paper pedestrian radius 0.5 m, max speed 1.33 m/s, desired 1.0 m/s.
DEFAULT_PARAMS = dict(timeStep=0.25, neighborDist=15.0, maxNeighbors=10, timeHorizon=5.0,
                      radius=0.5, maxSpeed=1.33)
DESIRED_SPEED = 1.0

CONFIGS = {
    # name: index for the seed
    "circle": 0,
    "corridor": 1,
    "uniform": 2,
    "uniform_1m": 3,
    "dense": 4,
    "uniform_4m": 5,
}


def _rng(config: str, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(BASE_SEED + CONFIGS[config] + 1000 * salt))


def _jittered_lattice(rng, nx: int, ny: int, spacing: float, radius: float, x0: float, y0: float):
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    base = np.stack([x0 + (ix.ravel() + 0.5) * spacing, y0 + (iy.ravel() + 0.5) * spacing], axis=1)
    amp = max(0.0, 0.99 * (spacing - 2.0 * radius) / 2.0)
    return base + rng.uniform(-amp, amp, size=base.shape)


def circle(n: int = 100, ring: float = 50.0, salt: int = 0):
    """C0: agents on a radius-`ring` circle walking to their antipodes; vel0 = 0.
    pref is computed from goals each step (orca_set_goals, prefSpeed = 1.0)."""
    a = 2.0 * np.pi * np.arange(n, dtype=np.float64) / n
    pos = (ring * np.stack([np.cos(a), np.sin(a)], axis=1)).astype(np.float32)
    goals = (-pos.astype(np.float64)).astype(np.float32)
    vel = np.zeros_like(pos)
    return dict(name="circle", pos=pos, vel=vel, pref=np.zeros_like(pos), goals=goals,
                pref_speed=DESIRED_SPEED, params=dict(DEFAULT_PARAMS), steps=1000)


def corridor(n: int = 10_000, length: float = 400.0, width: float = 100.0, salt: int = 0):
    """C1: bidirectional corridor, rho = n/(length*width); even ids +x, odd ids -x."""
    rng = _rng("corridor", salt)
    rho = n / (length * width)
    s = 1.0 / math.sqrt(rho)
    nx = int(math.ceil(length / s))
    ny = int(math.ceil(n / nx))
    pts = _jittered_lattice(rng, nx, ny, s, DEFAULT_PARAMS["radius"], 0.0, 0.0)
    pick = rng.permutation(len(pts))[:n]
    pos = pts[pick].astype(np.float32)
    pref = np.zeros((n, 2), np.float32)
    pref[0::2, 0] = DESIRED_SPEED
    pref[1::2, 0] = -DESIRED_SPEED
    return dict(name="corridor", pos=pos, vel=pref.copy(), pref=pref, goals=None,
                pref_speed=DESIRED_SPEED, params=dict(DEFAULT_PARAMS), steps=600)


def uniform(n: int = 100_000, rho: float = 0.25, salt: int = 0, config: str = "uniform"):
    """C2/C2'/C3/C4: random-uniform crowd at density rho in a square; pref = random unit
    heading x 1.0 m/s (held constant); vel0 = pref."""
    rng = _rng(config, salt)
    s = 1.0 / math.sqrt(rho)
    m = int(math.ceil(math.sqrt(n)))
    pts = _jittered_lattice(rng, m, m, s, DEFAULT_PARAMS["radius"], 0.0, 0.0)
    pick = rng.permutation(len(pts))[:n]
    pos = pts[pick].astype(np.float32)
    th = rng.uniform(0.0, 2.0 * np.pi, size=n)
    pref = (DESIRED_SPEED * np.stack([np.cos(th), np.sin(th)], axis=1)).astype(np.float32)
    return dict(name=f"{config}_n{n}_rho{rho}", pos=pos, vel=pref.copy(), pref=pref, goals=None,
                pref_speed=DESIRED_SPEED, params=dict(DEFAULT_PARAMS), steps=100)


def two_way(n: int = 2500, rho: float = 0.25, gap: float = 60.0, salt: int = 0):
    """E1a, the paper's 2-way crossing (Fig. 3): two crowds of n/2 start in a left
    and a right region; "the starting region of one group of people is the same area as
    the goal region of the other" -- each agent's goal is its mirror point in the opposite
    region.  Regions: square, density rho, `gap` metres apart.  Goal seeking at the
    desired 1.0 m/s, removal at the goal left to the caller."""
    rng = np.random.default_rng(BASE_SEED + 10 + 1000 * salt)
    half = n // 2
    side = math.sqrt(half / rho)
    s = 1.0 / math.sqrt(rho)
    m = int(math.ceil(side / s))
    left = _jittered_lattice(rng, m, m, s, DEFAULT_PARAMS["radius"], 0.0, 0.0)
    right = _jittered_lattice(rng, m, m, s, DEFAULT_PARAMS["radius"], side + gap, 0.0)
    left = left[rng.permutation(len(left))[:half]]
    right = right[rng.permutation(len(right))[:n - half]]
    width = 2 * side + gap
    pos = np.concatenate([left, right])
    goals = pos.copy()
    goals[:, 0] = width - pos[:, 0]  # mirror into the other region
    perm = rng.permutation(n)
    pos, goals = pos[perm].astype(np.float32), goals[perm].astype(np.float32)
    return dict(name=f"two_way_n{n}", pos=pos, vel=np.zeros_like(pos), pref=np.zeros_like(pos), goals=goals,
                pref_speed=DESIRED_SPEED, params=dict(DEFAULT_PARAMS), steps=2000)


def eight_way(n: int = 10_000, rho: float = 0.25, ring: float = 120.0, turn_deg: float = 135.0, salt: int = 0):
    """E1c, the paper's 8-way crossing (Fig. 5): eight crowds of n/8 in square
    regions around a ring; each crowd's goal region is its own region turned by
    `turn_deg` about the centre ("navigate 135 deg across the environment";
    P:151 says "to the opposite end" = 180, reading Q17).  Goal seeking at 1.0 m/s."""
    rng = np.random.default_rng(BASE_SEED + 11 + 1000 * salt)
    per = n // 8
    side = math.sqrt(per / rho)
    s = 1.0 / math.sqrt(rho)
    m = int(math.ceil(side / s))
    pos, goals = [], []
    t = math.radians(turn_deg)
    rot = np.array([[math.cos(t), -math.sin(t)], [math.sin(t), math.cos(t)]])
    for c in range(8):
        cnt = per if c < 7 else n - 7 * per
        a = 2 * math.pi * c / 8
        cx, cy = ring * math.cos(a), ring * math.sin(a)
        blk = _jittered_lattice(rng, m, m, s, DEFAULT_PARAMS["radius"], cx - side / 2, cy - side / 2)
        blk = blk[rng.permutation(len(blk))[:cnt]]
        pos.append(blk)
        goals.append(blk @ rot.T)
    pos, goals = np.concatenate(pos), np.concatenate(goals)
    perm = rng.permutation(n)
    pos, goals = pos[perm].astype(np.float32), goals[perm].astype(np.float32)
    return dict(name=f"eight_way_n{n}", pos=pos, vel=np.zeros_like(pos), pref=np.zeros_like(pos), goals=goals,
                pref_speed=DESIRED_SPEED, params=dict(DEFAULT_PARAMS), steps=3000)


def make(config: str, n: int | None = None, rho: float | None = None, salt: int = 0):
    """Named BASELINE.json configs."""
    if config == "circle":
        return circle(n or 100, salt=salt)
    if config == "corridor":
        return corridor(n or 10_000, salt=salt)
    if config == "uniform":
        return uniform(n or 100_000, rho if rho is not None else 0.25, salt=salt, config="uniform")
    if config == "uniform_1m":
        return uniform(n or 1_000_000, rho if rho is not None else 0.25, salt=salt, config="uniform_1m")
    if config == "dense":
        return uniform(n or 500_000, rho if rho is not None else 0.5, salt=salt, config="dense")
    if config == "uniform_4m":
        return uniform(n or 4_000_000, rho if rho is not None else 0.25, salt=salt, config="uniform_4m")
    if config == "two_way":
        return two_way(n or 2500, salt=salt)
    if config == "eight_way":
        return eight_way(n or 10_000, salt=salt)
    raise KeyError(config)


def tie_lattice(side: int = 30):
    """Integer lattice with id = side*x + y (tie-breaking fixture)."""
    ix, iy = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    pos = np.stack([ix.ravel(), iy.ravel()], axis=1).astype(np.float32)
    return pos
