"""Independent checkers that pin the oracle to something other than itself.

Nothing here calls oracle/ or the CUDA path: each function is a textbook definition or a
brute-force search, written directly from the mathematics the paper states:
  * cell floor as an exact rational (Fig. 2 bins; reading Q11),
  * neighbour sets by O(N^2) enumeration ("brute-force read all approach"),
  * the truncated velocity obstacle VO^tau (Fig. 1(b)) by its set definition,
  * the 2-D LP optimum by vertex enumeration (the feasible-case definition),
  * the least-penetration value by dense grid search over the speed disc.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


# ----------------------------------------------------------------------------- cells
def exact_cell(x: float, x0: float, cs: float, nc: int) -> int:
    """floor((x - x0)/cs) in exact rational arithmetic, clamped to [0, nc-1]."""
    q = (Fraction(float(x)) - Fraction(float(x0))) / Fraction(float(cs))
    c = math.floor(q)
    return min(max(c, 0), nc - 1)


# ------------------------------------------------------------------------ neighbours
def brute_neighbors(pos: np.ndarray, nd: float, k: int):
    """All-pairs k nearest strictly within nd, ordered by (kappa, id).
    kappa = dx*dx + dy*dy in fp64 from fp32 inputs, each op separately rounded (numpy
    elementwise ops never contract)."""
    pos = np.asarray(pos, np.float32).astype(np.float64)
    n = len(pos)
    nd2 = np.float64(nd) * np.float64(nd)
    nbr = np.full((n, k), -1, np.int64)
    cnt = np.zeros(n, np.int64)
    ids = np.arange(n)
    for i in range(n):
        dx = pos[:, 0] - pos[i, 0]
        dy = pos[:, 1] - pos[i, 1]
        key = dx * dx + dy * dy
        ok = (key < nd2) & (ids != i)
        cand = ids[ok]
        order = np.lexsort((cand, key[ok]))
        sel = cand[order][:k]
        nbr[i, :len(sel)] = sel
        cnt[i] = len(sel)
    return nbr, cnt


# ------------------------------------------------------------------ velocity obstacle
def vo_gap(v, rel_p, R, tau):
    """min_{t in [0,tau]} |t*v - rel_p| - R : negative iff v in VO^tau (Fig. 1(b)),
    i.e. the relative velocity v brings the discs into contact within tau.
    v may be (..., 2)."""
    v = np.asarray(v, np.float64)
    rel_p = np.asarray(rel_p, np.float64)
    vv = np.sum(v * v, axis=-1)
    with np.errstate(invalid="ignore", divide="ignore"):
        t = np.where(vv > 0, (v @ rel_p) / np.where(vv > 0, vv, 1.0), 0.0)
    t = np.clip(t, 0.0, tau)
    d = t[..., None] * v - rel_p
    return np.hypot(d[..., 0], d[..., 1]) - R


def distance_to_vo_boundary(v_rel, rel_p, R, tau, n_dir=720, s_max=8.0, n_steps=4000):
    """Shortest distance from v_rel to the boundary of VO^tau by vectorised ray marching +
    bisection over n_dir directions (Fig. 1(c) "the shortest vector to the edge of the
    obstacle")."""
    v_rel = np.asarray(v_rel, np.float64)
    inside0 = vo_gap(v_rel, rel_p, R, tau) < 0
    th = np.linspace(0, 2 * np.pi, n_dir, endpoint=False)
    e = np.stack([np.cos(th), np.sin(th)], axis=1)                 # (D, 2)
    s = np.linspace(0.0, s_max, n_steps + 1)[1:]                    # (S,)
    pts = v_rel[None, None, :] + s[None, :, None] * e[:, None, :]    # (D, S, 2)
    flip = (vo_gap(pts, rel_p, R, tau) < 0) != inside0              # (D, S)
    has = flip.any(axis=1)
    if not has.any():
        return np.inf
    first = np.argmax(flip, axis=1)
    lo = np.where(first > 0, s[np.maximum(first - 1, 0)], 0.0)[has]
    hi = s[first][has]
    ee = e[has]
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        f = (vo_gap(v_rel[None, :] + mid[:, None] * ee, rel_p, R, tau) < 0) != inside0
        hi = np.where(f, mid, hi)
        lo = np.where(f, lo, mid)
    return float(hi.min())


# ------------------------------------------------------------------------------- LP
def _halfplane_form(lines):
    """(point, unit direction) with permitted det(d, p - v) <= 0  ->  (n, s) with
    permitted n.v >= s, n = (-d.y, d.x)."""
    lines = np.asarray(lines, np.float64).reshape(-1, 4)
    n = np.stack([-lines[:, 3], lines[:, 2]], axis=1)
    s = n[:, 0] * lines[:, 0] + n[:, 1] * lines[:, 1]
    return n, s


def lp_vertex_enumeration(lines, r, pref, tol=1e-9):
    """argmin |v - pref| over {|v| <= r} intersect half-planes, by enumerating the finite
    candidate set that must contain the optimum of a strictly convex objective over a
    polygon-with-arc: pref clipped to the disc, projections of pref on each line, pairwise
    line intersections, line/circle intersections.  Returns None if infeasible."""
    n, s = _halfplane_form(lines)
    pref = np.asarray(pref, np.float64)
    cands = []
    lp = np.hypot(*pref)
    cands.append(pref if lp <= r else pref / lp * r)
    m = len(s)
    for i in range(m):
        # projection of pref on line i
        cands.append(pref + (s[i] - n[i] @ pref) * n[i])
        # line i with the circle
        d = np.array([n[i, 1], -n[i, 0]])
        base = s[i] * n[i]
        disc = r * r - s[i] * s[i]
        if disc >= 0:
            sq = math.sqrt(disc)
            cands.append(base + sq * d)
            cands.append(base - sq * d)
        for j in range(i + 1, m):
            A = np.array([n[i], n[j]])
            det = np.linalg.det(A)
            if abs(det) > 1e-14:
                cands.append(np.linalg.solve(A, np.array([s[i], s[j]])))
    best, bestd = None, np.inf
    for c in cands:
        if np.hypot(*c) > r + tol:
            continue
        if m and np.any(n @ c - s < -tol):
            continue
        d = np.hypot(*(c - pref))
        if d < bestd:
            best, bestd = c, d
    return best


def penetration_np(lines, v):
    n, s = _halfplane_form(lines)
    v = np.asarray(v, np.float64)
    if len(s) == 0:
        return 0.0
    return float(max(0.0, np.max(s - n @ v)))


def lp3_grid_search(lines, r, res=801):
    """min over a dense grid of the speed disc of the maximum penetration (P:80
    "select a velocity that least penetrates the set of half-planes")."""
    n, s = _halfplane_form(lines)
    g = np.linspace(-r, r, res)
    X, Y = np.meshgrid(g, g, indexing="ij")
    inside = X * X + Y * Y <= r * r
    V = np.stack([X[inside], Y[inside]], axis=1)
    pen = np.max(s[None, :] - V @ n.T, axis=1)
    pen = np.maximum(pen, 0.0)
    q = int(np.argmin(pen))
    return float(pen[q]), V[q]
