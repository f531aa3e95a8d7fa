"""Pins of the fp64 oracle against things other than itself.

CPU only (no GPU marker).  Each test names the passage of PAPER.md / SPEC.md it pins.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import pins
from paper_1908_10107_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------------- cells (Fig. 2)
def test_cells_match_exact_rational_floor(oracle):
    """Cell = exact floor((x-x0)/cs) clamped (P:94 bins; reading Q11)."""
    rng = np.random.default_rng(1)
    cs = np.float32(15.0)
    x0 = np.float32(-15.0)
    xs = list(rng.uniform(-40, 4100, 3000).astype(np.float32))
    # exact multiples of cs and their fp32 neighbours (edges -> higher cell)
    for m in range(0, 280, 7):
        e = np.float32(x0 + np.float32(m) * cs)
        xs += [e, np.nextafter(e, np.float32(-1e9)), np.nextafter(e, np.float32(1e9))]
    xs = np.array(xs, np.float32)
    pos = np.stack([xs, xs[::-1]], axis=1)
    dims = np.array([270, 270], np.int32)
    cx, cy = oracle.cells(pos, np.array([x0, x0], np.float32), cs, dims)
    for i in range(len(xs)):
        assert cx[i] == pins.exact_cell(pos[i, 0], x0, cs, 270)
        assert cy[i] == pins.exact_cell(pos[i, 1], x0, cs, 270)


def test_cells_spec_examples(oracle):
    """S:251 (7,7)/(20,7) with r_obs 15 -> adjacent bins; S:252 edge -> higher cell."""
    pos = np.array([[7, 7], [20, 7], [15, 0]], np.float32)
    cx, cy = oracle.cells(pos, np.zeros(2, np.float32), 15.0, np.array([4, 4], np.int32))
    assert list(cx) == [0, 1, 1] and list(cy) == [0, 0, 0]


def test_grid_derive_margin(oracle):
    """Frozen grid (reading Q12): origin = fl32(min - cs) (fp32 rounding may put the
    minimum agent in cell 0 or 1); dims leave one empty margin cell above the maximum."""
    w = W.make("uniform", n=5000, rho=0.1)
    origin, dims = oracle.grid_derive(w["pos"], 15.0)
    for a in range(2):
        assert origin[a] == np.float32(w["pos"][:, a].min() - np.float32(15.0))
    cx, cy = oracle.cells(w["pos"], origin, 15.0, dims)
    for c, d, a in ((cx, dims[0], 0), (cy, dims[1], 1)):
        assert c.min() >= 0 and c.max() <= d - 2
        # the maximum agent is in the last non-margin cell
        i = int(np.argmax(w["pos"][:, a]))
        assert c[i] == d - 2 == pins.exact_cell(w["pos"][i, a], origin[a], 15.0, 10**9)


# --------------------------------------------------------------- neighbours
@pytest.mark.parametrize("n,rho,k", [(1500, 0.25, 10), (1200, 0.5, 10), (800, 0.02, 7), (600, 0.3, 32),
                                     (300, 0.25, 0), (1, 0.1, 10)])
def test_neighbors_equal_brute_force(oracle, n, rho, k):
    """Bins + 3x3 read + r_obs filter == all-pairs definition."""
    w = W.uniform(n=n, rho=rho, salt=3)
    pos = w["pos"]
    origin, dims = oracle.grid_derive(pos, 15.0)
    nbr, cnt = oracle.neighbors(pos, origin, 15.0, dims, 15.0, k)
    bn, bc = pins.brute_neighbors(pos, 15.0, k)
    assert np.array_equal(cnt, bc)
    assert np.array_equal(nbr.astype(np.int64), bn)


def test_neighbors_clustered_and_duplicates(oracle):
    """Coincident positions (exact key ties) and agents outside the frozen grid."""
    rng = np.random.default_rng(7)
    base = rng.uniform(0, 60, (200, 2)).astype(np.float32)
    pos = np.concatenate([base, base[:50], base[:20] + np.float32(15.0)]).astype(np.float32)
    origin, dims = oracle.grid_derive(pos[:200], 15.0)
    # move some agents outside the frozen grid (clamped to edge cells)
    pos[-5:] = np.array([[-100, 5], [500, 30], [30, -90], [30, 400], [-50, -50]], np.float32)
    for k in (10, 32):
        nbr, cnt = oracle.neighbors(pos, origin, 15.0, dims, 15.0, k)
        bn, bc = pins.brute_neighbors(pos, 15.0, k)
        assert np.array_equal(cnt, bc)
        assert np.array_equal(nbr.astype(np.int64), bn)


def test_tie_lattice_golden(oracle):
    g = _load("tie_lattice.json")
    pos = W.tie_lattice(g["side"])
    origin, dims = oracle.grid_derive(pos, g["nd"])
    nbr, cnt = oracle.neighbors(pos, origin, g["nd"], dims, g["nd"], g["k"])
    assert list(nbr[g["agent"]]) == g["neighbors"]


# ------------------------------------------------------------ ORCA lines (Fig. 1)
def _n_s(line):
    px, py, dx, dy = line
    n = np.array([-dy, dx])
    return n, float(n @ np.array([px, py]))


BRANCH = {"collision": 1, "cutoff": 2, "left": 4, "right": 8}


def test_orca_closed_forms(oracle):
    g = _load("orca_closed_forms.json")
    for c in g["cases"]:
        line, br = oracle.orca_line(c["pi"], c["vi"], c["pj"], c["vj"], 0, 1, c["radius"], c["tau"], c["dt"])
        assert br & BRANCH[c["branch"]], c["name"]
        if "point" in c:
            n, s = _n_s(line)
            assert np.allclose(n, c["normal"], atol=1e-12), c["name"]
            assert abs(s - float(np.dot(n, c["point"]))) < 1e-9, c["name"]
            assert abs(float(np.array(c["point"]) @ n) - s) < 1e-9
        if "line_x" in c:
            n, s = _n_s(line)
            assert np.allclose(n, [-1, 0], atol=1e-12) and abs(-s - c["line_x"]) < 1e-12
        if "vstar" in c:
            v, inf, _ = oracle.solve([line], c["maxSpeed"], c["pref"])
            assert not inf
            assert np.allclose(v, c["vstar"], atol=1e-12), (c["name"], v)


def test_head_on_closed_form_family(oracle):
    """Head-on pair: v*_a = (v(1-R^2/4d^2), -vR sqrt(4d^2-R^2)/4d^2), v*_b = -v*_a,
    |v*| = v sqrt(1 - R^2/D^2) (hand-derived from Fig. 1)."""
    for d, v, r, tau in [(5, 1, 0.5, 10), (3, 0.8, 0.3, 20), (10, 1.2, 0.75, 12)]:
        R = 2 * r
        la, _ = oracle.orca_line([-d, 0], [v, 0], [d, 0], [-v, 0], 0, 1, r, tau, 0.25)
        lb, _ = oracle.orca_line([d, 0], [-v, 0], [-d, 0], [v, 0], 1, 0, r, tau, 0.25)
        va, _, _ = oracle.solve([la], 5.0, [v, 0])
        vb, _, _ = oracle.solve([lb], 5.0, [-v, 0])
        D = 2 * d
        exp = np.array([v * (1 - R * R / (4 * d * d)), -v * R * math.sqrt(4 * d * d - R * R) / (4 * d * d)])
        assert np.allclose(va, exp, atol=1e-6), (va, exp)
        assert np.allclose(vb, -exp, atol=1e-6)
        assert abs(np.hypot(*va) - v * math.sqrt(1 - R * R / (D * D))) < 1e-6


def _random_pairs(rng, m):
    out = []
    while len(out) < m:
        pi = rng.uniform(-8, 8, 2)
        pj = rng.uniform(-8, 8, 2)
        vi = rng.uniform(-1.5, 1.5, 2)
        vj = rng.uniform(-1.5, 1.5, 2)
        out.append([np.float32(x) for x in (pi, vi, pj, vj)])
    return out


def test_reciprocity(oracle):
    """u_ab = -u_ba (responsibility 1/2 on both sides, reading Q2)."""
    rng = np.random.default_rng(11)
    for pi, vi, pj, vj in _random_pairs(rng, 3000):
        la, _ = oracle.orca_line(pi, vi, pj, vj, 0, 1, 0.5, 5.0, 0.25)
        lb, _ = oracle.orca_line(pj, vj, pi, vi, 1, 0, 0.5, 5.0, 0.25)
        ua = 2 * (np.array(la[:2]) - vi.astype(np.float64))
        ub = 2 * (np.array(lb[:2]) - vj.astype(np.float64))
        assert np.allclose(ua, -ub, atol=1e-12)


def test_u_is_shortest_vector_to_vo_boundary(oracle):
    """Fig. 1(c): 'u is the shortest vector to the edge of the obstacle from the vector of
    velocities'; v_rel + u lies on the VO^tau boundary and the normal points out of the
    obstacle.  Checked against the VO set definition by ray marching (tests/pins.py)."""
    rng = np.random.default_rng(5)
    tau, r = 5.0, 0.5
    checked = 0
    for pi, vi, pj, vj in _random_pairs(rng, 60):
        rel_p = pj.astype(np.float64) - pi.astype(np.float64)
        if np.hypot(*rel_p) <= 2 * r:
            continue
        line, br = oracle.orca_line(pi, vi, pj, vj, 0, 1, r, tau, 0.25)
        v_rel = vi.astype(np.float64) - vj.astype(np.float64)
        u = 2 * (np.array(line[:2]) - vi.astype(np.float64))
        # on the boundary
        assert abs(pins.vo_gap(v_rel + u, rel_p, 2 * r, tau)) < 1e-9
        # shortest
        dist = pins.distance_to_vo_boundary(v_rel, rel_p, 2 * r, tau)
        # shortest: no sampled boundary point is closer than v_rel + u, which itself lies
        # on the boundary (so |u| >= the true distance)
        assert np.hypot(*u) <= dist + 1e-9
        # the permitted side is outside the obstacle
        n, s = _n_s(line)
        assert pins.vo_gap(v_rel + u + 1e-4 * n, rel_p, 2 * r, tau) > 0
        checked += 1
    assert checked > 40


def test_pairwise_no_collision_guarantee(oracle):
    """P:77 'By selecting a velocity not restricted by this half-plane, the two agents are
    guaranteed to not collide within time tau'."""
    rng = np.random.default_rng(21)
    tau, r = 5.0, 0.5
    viol = 0
    tested = 0
    for pi, vi, pj, vj in _random_pairs(rng, 4000):
        rel_p = pj.astype(np.float64) - pi.astype(np.float64)
        if np.hypot(*rel_p) <= 2 * r:
            continue
        la, _ = oracle.orca_line(pi, vi, pj, vj, 0, 1, r, tau, 0.25)
        lb, _ = oracle.orca_line(pj, vj, pi, vi, 1, 0, r, tau, 0.25)
        pa = rng.uniform(-1.3, 1.3, 2)
        pb = rng.uniform(-1.3, 1.3, 2)
        va, ia, _ = oracle.solve([la], 50.0, pa)
        vb, ib, _ = oracle.solve([lb], 50.0, pb)
        assert not ia and not ib
        # min distance over [0, tau] of p_rel + (vb - va) t
        dv = vb - va
        dd = float(dv @ dv)
        t = 0.0 if dd == 0 else min(max(-float(rel_p @ dv) / dd, 0.0), tau)
        gap = np.hypot(*(rel_p + t * dv)) - 2 * r
        viol += gap < -1e-9
        tested += 1
    assert tested > 3000 and viol == 0


def test_collision_branch_separates(oracle):
    """Reading Q4: overlapping agents get a one-step separation constraint; after taking
    their constrained velocities the centre distance grows (S:189 'post-step separation')."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        pi = rng.uniform(-0.4, 0.4, 2).astype(np.float32)
        pj = (pi + rng.uniform(-0.6, 0.6, 2)).astype(np.float32)
        vi = rng.uniform(-1, 1, 2).astype(np.float32)
        vj = rng.uniform(-1, 1, 2).astype(np.float32)
        la, br = oracle.orca_line(pi, vi, pj, vj, 0, 1, 0.5, 5.0, 0.25)
        if not br & 1:
            continue
        lb, _ = oracle.orca_line(pj, vj, pi, vi, 1, 0, 0.5, 5.0, 0.25)
        va, _, _ = oracle.solve([la], 50.0, vi)
        vb, _, _ = oracle.solve([lb], 50.0, vj)
        d0 = np.hypot(*(pj.astype(np.float64) - pi))
        d1 = np.hypot(*(pj + 0.25 * vb - pi - 0.25 * va))
        assert d1 >= min(1.0, d0) - 1e-9


def test_coincident_agents_deterministic(oracle):
    """Reading Q15: coincident agents with equal velocity -> lower id pushed to -x."""
    la, br = oracle.orca_line([1, 1], [0.5, 0], [1, 1], [0.5, 0], 3, 9, 0.5, 5.0, 0.25)
    lb, brb = oracle.orca_line([1, 1], [0.5, 0], [1, 1], [0.5, 0], 9, 3, 0.5, 5.0, 0.25)
    assert br & 16 and brb & 16
    va, _, _ = oracle.solve([la], 10.0, [0.5, 0])
    vb, _, _ = oracle.solve([lb], 10.0, [0.5, 0])
    assert va[0] < 0.5 - 1.0 and vb[0] > 0.5 + 1.0
    assert np.allclose(va - 0.5 * np.array([1, 0]), -(vb - 0.5 * np.array([1, 0])), atol=1e-12)


# ------------------------------------------------------------------ LP
def test_spec_lp_examples(oracle):
    g = _load("spec_lp_examples.json")
    for c in g["cases"]:
        lines = c["lines"]
        if lines == "triangle":
            lines = []
            for deg in (90, 210, 330):
                n = np.array([math.cos(math.radians(deg)), math.sin(math.radians(deg))])
                lines.append([0.5 * n[0], 0.5 * n[1], n[1], -n[0]])
        v, inf, _ = oracle.solve(lines, c["r"], c["pref"])
        assert inf == (not c["feasible"]), c["name"]
        if "v" in c:
            assert np.allclose(v, c["v"], atol=1e-12), (c["name"], v)
        if "vx" in c:
            assert abs(v[0] - c["vx"]) < 1e-12
        if "delta" in c:
            assert abs(oracle.penetration(lines, v) - c["delta"]) < 1e-12, c["name"]
        assert np.hypot(*v) <= c["r"] + 1e-12


def _random_lp(rng, m, r=1.33):
    ang = rng.uniform(0, 2 * np.pi, m)
    n = np.stack([np.cos(ang), np.sin(ang)], 1)
    s = rng.uniform(-1.0, 0.6, m)
    pts = s[:, None] * n
    d = np.stack([n[:, 1], -n[:, 0]], 1)
    lines = np.concatenate([pts + rng.uniform(-2, 2, (m, 1)) * d, d], axis=1)
    pref = rng.uniform(-2, 2, 2)
    return lines, pref


def test_lp2_vertex_enumeration(oracle):
    """Feasible optimum = argmin |v - pref| over the disc and half-planes, by vertex
    enumeration; classification agrees except on marginal (tolerance-width) problems."""
    rng = np.random.default_rng(2)
    agree = 0
    for trial in range(1500):
        m = int(rng.integers(0, 33))
        lines, pref = _random_lp(rng, m)
        v, inf, _ = oracle.solve(lines, 1.33, pref)
        ref = pins.lp_vertex_enumeration(lines, 1.33, pref)
        if ref is None:
            assert inf or oracle.penetration(lines, v) < 1e-9
        else:
            if inf:
                # only allowed when the feasible set has tolerance width
                assert pins.penetration_np(lines, ref) < 1e-9 and oracle.penetration(lines, v) < 1e-8
                continue
            assert np.allclose(v, ref, atol=1e-9), (trial, v, ref)
            agree += 1
    assert agree > 300


def test_lp2_feasibility_and_order_invariance(oracle):
    """feasible solutions satisfy every line within 1e-9 and |v| <= r; the
    optimum does not depend on the constraint order (strictly convex objective)."""
    rng = np.random.default_rng(4)
    for _ in range(800):
        m = int(rng.integers(1, 20))
        lines, pref = _random_lp(rng, m)
        v, inf, _ = oracle.solve(lines, 1.33, pref)
        if inf:
            continue
        assert pins.penetration_np(lines, v) <= 1e-9
        assert np.hypot(*v) <= 1.33 + 1e-9
        perm = rng.permutation(m)
        v2, inf2, _ = oracle.solve(lines[perm], 1.33, pref)
        assert not inf2 and np.allclose(v, v2, atol=1e-9)


def test_lp3_grid_search(oracle):
    """P:80 least penetration: delta(v_oracle) <= grid-search best (801^2) and within its
    resolution bound; the result stays in the speed disc."""
    rng = np.random.default_rng(8)
    tested = 0
    while tested < 120:
        m = int(rng.integers(2, 16))
        ang = rng.uniform(0, 2 * np.pi, m)
        n = np.stack([np.cos(ang), np.sin(ang)], 1)
        s = rng.uniform(0.2, 1.2, m)  # outward-ish constraints: often infeasible
        d = np.stack([n[:, 1], -n[:, 0]], 1)
        lines = np.concatenate([s[:, None] * n, d], axis=1)
        v, inf, _ = oracle.solve(lines, 1.33, rng.uniform(-1, 1, 2))
        if not inf:
            continue
        dl = oracle.penetration(lines, v)
        gbest, _ = pins.lp3_grid_search(lines, 1.33, res=401)
        assert dl <= gbest + 1e-12
        assert dl >= gbest - 2 * (2 * 1.33 / 400) * 1.0 - 1e-9
        assert np.hypot(*v) <= 1.33 + 1e-9
        tested += 1


# ----------------------------------------------------------------- whole step
def _params(oracle, **kw):
    p = dict(W.DEFAULT_PARAMS)
    p.update(kw)
    return oracle.make_params(**p)


def _lines_for(oracle, w, i, nbrs, p):
    out = []
    for j in nbrs:
        l, _ = oracle.orca_line(w["pos"][i], w["vel"][i], w["pos"][j], w["vel"][j], i, j, p.radius,
                                p.timeHorizon, p.timeStep)
        out.append(l)
    return out


@pytest.mark.parametrize("config,n,rho", [("uniform", 1500, 0.5), ("corridor", 2000, None), ("uniform", 1500, 0.05)])
def test_step_invariants(oracle, config, n, rho):
    """Every new velocity satisfies all its ORCA lines within 1e-9 when feasible, |v| <=
    maxSpeed always; infeasible agents report delta = max penetration; p' = p + dt v'."""
    w = W.make(config, n=n, rho=rho) if rho else W.corridor(n=n, length=n / (0.25 * 25.0), width=25.0)
    p = _params(oracle)
    r = oracle.step(p, w["pos"], w["vel"], pref=w["pref"], want_nbrs=True)
    origin, dims = oracle.grid_derive(w["pos"], p.neighborDist)
    nb, cnt = oracle.neighbors(w["pos"], origin, p.neighborDist, dims, p.neighborDist, p.maxNeighbors)
    assert np.array_equal(r["nbr"], nb) and np.array_equal(r["cnt"], cnt)
    for i in range(0, n, 7):
        lines = _lines_for(oracle, w, i, nb[i, :cnt[i]], p)
        v = r["vel"][i]
        assert np.hypot(*v) <= p.maxSpeed + 1e-9
        pen = pins.penetration_np(lines, v) if lines else 0.0
        if r["flags"][i] & oracle.FLAG_INFEASIBLE:
            assert abs(pen - r["delta"][i]) < 1e-12 and pen > 0
        else:
            assert pen <= 1e-9
            ref = pins.lp_vertex_enumeration(lines, p.maxSpeed, w["pref"][i].astype(np.float64))
            assert ref is not None and np.allclose(v, ref, atol=1e-9)
        assert np.allclose(r["pos"][i], w["pos"][i].astype(np.float64) + p.timeStep * v, atol=0, rtol=0)
    deg = np.count_nonzero(r["flags"] & oracle.FLAG_DEGENERATE)
    assert deg <= max(2, 0.001 * n)


def test_free_agent_moves_pref(oracle):
    """A lone agent takes pref clipped to maxSpeed (LP with no constraints)."""
    p = _params(oracle)
    pos = np.array([[0, 0], [100, 100]], np.float32)
    vel = np.zeros((2, 2), np.float32)
    pref = np.array([[2.0, 0.0], [0.3, -0.4]], np.float32)
    r = oracle.step(p, pos, vel, pref=pref)
    assert np.allclose(r["vel"][0], [1.33, 0], atol=1e-7)
    assert np.allclose(r["vel"][1], pref[1].astype(np.float64), atol=0)
    assert np.allclose(r["pos"][0], [0.25 * 1.33, 0], atol=1e-7)


def test_step_subset_equals_full(oracle):
    w = W.make("uniform", n=3000, rho=0.25)
    p = _params(oracle)
    full = oracle.step(p, w["pos"], w["vel"], pref=w["pref"])
    ag = np.array([0, 5, 17, 2999, 1234])
    sub = oracle.step(p, w["pos"], w["vel"], pref=w["pref"], agents=ag)
    assert np.array_equal(sub["vel"], full["vel"][ag])
    assert np.array_equal(sub["flags"], full["flags"][ag])


def test_circle_all_arrive(oracle):
    """C0: all 100 agents reach their antipodes within 1000 steps with the
    paper's pedestrian parameters; speed cap holds every step."""
    w = W.make("circle")
    p = _params(oracle)
    pos, vel = w["pos"].copy(), w["vel"].copy()
    for chunk in range(10):
        pos, vel, _ = oracle.run(p, pos, vel, goals=w["goals"], pref_speed=1.0, steps=100)
        assert np.all(np.hypot(vel[:, 0], vel[:, 1]) <= p.maxSpeed * (1 + 1e-6))
    dist = np.hypot(*(pos - w["goals"]).T)
    assert np.all(dist < p.radius)


def test_degenerate_rate_small(oracle):
    """BASELINE north_star: degenerate LPs must stay below 0.1 % (dense cold start)."""
    w = W.make("dense", n=4000)
    p = _params(oracle)
    r = oracle.step(p, w["pos"], w["vel"], pref=w["pref"])
    assert np.count_nonzero(r["flags"] & oracle.FLAG_DEGENERATE) <= 4


# ------------------------------------------- heterogeneous agents (§8(f2))
def test_head_on_unequal_radii_closed_form(oracle):
    """The head-on closed form depends on R = r_a + r_b only (Fig. 1(a)): unequal radii give
    the same v* as equal radii with the same sum."""
    d, v, tau = 5.0, 1.0, 10.0
    for ra, rb in [(0.5, 1.0), (0.75, 0.25), (1.0, 1.0)]:
        R = ra + rb
        la, _ = oracle.orca_line([-d, 0], [v, 0], [d, 0], [-v, 0], 0, 1, ra, tau, 0.25, rj=rb)
        lb, _ = oracle.orca_line([d, 0], [-v, 0], [-d, 0], [v, 0], 1, 0, rb, tau, 0.25, rj=ra)
        va, _, _ = oracle.solve([la], 5.0, [v, 0])
        vb, _, _ = oracle.solve([lb], 5.0, [-v, 0])
        exp = np.array([v * (1 - R * R / (4 * d * d)), -v * R * math.sqrt(4 * d * d - R * R) / (4 * d * d)])
        assert np.allclose(va, exp, atol=1e-6) and np.allclose(vb, -exp, atol=1e-6)


def test_unequal_radii_reciprocity_and_no_collision(oracle):
    rng = np.random.default_rng(31)
    viol = 0
    for pi, vi, pj, vj in _random_pairs(rng, 2000):
        ra, rb = rng.choice([0.5, 0.75, 1.0], 2)
        rel_p = pj.astype(np.float64) - pi.astype(np.float64)
        la, _ = oracle.orca_line(pi, vi, pj, vj, 0, 1, ra, 5.0, 0.25, rj=rb)
        lb, _ = oracle.orca_line(pj, vj, pi, vi, 1, 0, rb, 5.0, 0.25, rj=ra)
        ua = 2 * (np.array(la[:2]) - vi.astype(np.float64))
        ub = 2 * (np.array(lb[:2]) - vj.astype(np.float64))
        assert np.allclose(ua, -ub, atol=1e-12)
        if np.hypot(*rel_p) <= ra + rb:
            continue
        va, _, _ = oracle.solve([la], 50.0, rng.uniform(-2, 2, 2))
        vb, _, _ = oracle.solve([lb], 50.0, rng.uniform(-2, 2, 2))
        dv = vb - va
        dd = float(dv @ dv)
        t = 0.0 if dd == 0 else min(max(-float(rel_p @ dv) / dd, 0.0), 5.0)
        viol += np.hypot(*(rel_p + t * dv)) - (ra + rb) < -1e-9
    assert viol == 0


def test_heterogeneous_step_invariants(oracle):
    """Per-agent maxSpeed caps every velocity; lines use r_i + r_j; per-agent desired speed
    with goals (max = 125 % of desired)."""
    w = W.make("uniform", n=2000, rho=0.15)
    rng = np.random.default_rng(5)
    radius = rng.choice([0.5, 0.75, 1.0], 2000).astype(np.float32)
    desired = rng.choice([1.0, 1.33, 2.0], 2000).astype(np.float32)
    props = dict(radius=radius, maxSpeed=(1.25 * desired).astype(np.float32), prefSpeed=desired)
    goals = (w["pos"] + rng.uniform(-50, 50, w["pos"].shape)).astype(np.float32)
    p = _params(oracle)
    r = oracle.step(p, w["pos"], w["vel"], goals=goals, props=props, want_nbrs=True)
    sp = np.hypot(*r["vel"].T)
    assert np.all(sp <= props["maxSpeed"].astype(np.float64) + 1e-9)
    for i in range(0, 2000, 13):
        lines = [oracle.orca_line(w["pos"][i], w["vel"][i], w["pos"][j], w["vel"][j], i, j, radius[i],
                                  p.timeHorizon, p.timeStep, rj=radius[j])[0] for j in r["nbr"][i][:r["cnt"][i]]]
        pen = pins.penetration_np(lines, r["vel"][i]) if lines else 0.0
        if not r["flags"][i] & oracle.FLAG_INFEASIBLE:
            assert pen <= 1e-9
            g = goals[i].astype(np.float64) - w["pos"][i]
            pref = g * min(1.0, desired[i] / np.hypot(*g))
            ref = pins.lp_vertex_enumeration(lines, float(props["maxSpeed"][i]), pref)
            assert ref is not None and np.allclose(r["vel"][i], ref, atol=1e-9)


# ------------------------------------------- randomized constraint order (§8(f3), reading Q8)
def test_lp_permutation_is_a_uniform_permutation(oracle):
    """P:82 "randomized incremental": every order is a permutation of the c lines, and the
    Fisher-Yates shuffle of the counter-based hash is uniform (chi-square over the 6 orders
    of 3 lines; every line equally likely at every slot for c = 10)."""
    for c in (0, 1, 2, 5, 10, 32):
        for key in range(50):
            idx = oracle.lp_permutation(12345, key % 7, key * 977, c)
            assert sorted(idx.tolist()) == list(range(c))
    counts = {}
    for agent in range(6000):
        t = tuple(oracle.lp_permutation(7, 3, agent, 3).tolist())
        counts[t] = counts.get(t, 0) + 1
    assert len(counts) == 6
    chi2 = sum((v - 1000.0) ** 2 / 1000.0 for v in counts.values())
    assert chi2 < 20.5  # p = 0.001 at 5 dof
    slot = np.zeros((10, 10))
    for agent in range(5000):
        for s, q in enumerate(oracle.lp_permutation(99, agent % 3, agent, 10)):
            slot[s, q] += 1
    assert np.all(np.abs(slot - 500.0) < 5 * math.sqrt(500 * 0.9))
    # the order depends on every key component
    base = oracle.lp_permutation(1, 2, 3, 16)
    for args in [(2, 2, 3), (1, 3, 3), (1, 2, 4)]:
        assert not np.array_equal(base, oracle.lp_permutation(*args, 16))


def test_randomized_order_same_optimum(oracle):
    """The LP optimum does not depend on the constraint order (a strictly convex
    objective over a convex region has one minimiser; the 3-D fallback has one minimal
    penetration): with the randomized order every feasible agent reaches the vertex-
    enumeration optimum and every infeasible one the same delta as nearest-first."""
    w = W.make("uniform", n=3000, rho=0.5)
    p = _params(oracle)
    a = oracle.step(p, w["pos"], w["vel"], pref=w["pref"], want_nbrs=True)
    b = oracle.step(p, w["pos"], w["vel"], pref=w["pref"], want_nbrs=True, lp_seed=2024, lp_step=5)
    assert np.array_equal(a["nbr"], b["nbr"])
    inf = (a["flags"] & oracle.FLAG_INFEASIBLE) != 0
    assert np.array_equal(inf, (b["flags"] & oracle.FLAG_INFEASIBLE) != 0)
    assert np.count_nonzero(inf) > 10
    feas = ~inf
    assert np.allclose(a["vel"][feas], b["vel"][feas], atol=1e-9)
    assert np.allclose(a["delta"][inf], b["delta"][inf], atol=1e-9)
    deg = (a["flags"] | b["flags"]) & oracle.FLAG_DEGENERATE
    same_v = np.all(np.isclose(a["vel"], b["vel"], atol=1e-9), axis=1)
    assert np.all(same_v | (deg != 0) | inf)
    # but the solver really saw another order: the processed sequence differs
    moved = sum(not np.array_equal(oracle.lp_permutation(2024, 5, i, int(c)), np.arange(c))
                for i, c in enumerate(b["cnt"]) if c > 1)
    assert moved > 0.9 * np.count_nonzero(b["cnt"] > 1)


# --------------------------------------- degenerate classes g2 / g4
def _rot_line(line, th, q):
    """`line` (point, unit direction) rotated by th about the point q (which it contains)."""
    c, s = math.cos(th), math.sin(th)
    dx, dy = line[2], line[3]
    return [q[0], q[1], c * dx - s * dy, s * dx + c * dy]


def _argmin_diameter(lines, r, slack, res=801):
    """Diameter of {v in the disc : max penetration(v) <= grid best + slack} on a dense grid:
    large iff the least-penetration argmin is not unique (up to the grid)."""
    n, s = pins._halfplane_form(lines)
    g = np.linspace(-r, r, res)
    X, Y = np.meshgrid(g, g, indexing="ij")
    inside = X * X + Y * Y <= r * r
    V = np.stack([X[inside], Y[inside]], axis=1)
    pen = np.maximum(np.max(s[None, :] - V @ n.T, axis=1), 0.0)
    near = V[pen <= pen.min() + slack]
    return float(np.max(np.ptp(near, axis=0)))


def test_g4_fires_on_non_unique_lp3_argmin(oracle):
    """g4: a least-penetration problem whose argmin is a segment.  The
    S:123 pair {x >= 1, x <= -1} is minimised (delta = 1) by every point of x = 0 in the
    disc; likewise {y >= 0.5, y <= -0.5, x <= 1.5} along y = 0.  The grid search confirms
    the argmin set is a long segment, and the oracle flags g4."""
    cases = [
        [[1.0, 0.0, 0.0, -1.0], [-1.0, 0.0, 0.0, 1.0]],
        [[0.0, 0.5, 1.0, 0.0], [0.0, -0.5, -1.0, 0.0], [1.5, 0.0, 0.0, 1.0]],
    ]
    for lines in cases:
        assert _argmin_diameter(lines, 2.0, 1e-9) > 1.0  # independent: non-unique argmin
        v, fl, d = oracle.solve_classify(lines, 2.0, [0.3, 0.1])
        assert fl & oracle.FLAG_INFEASIBLE
        assert fl & oracle.FLAG_G4, (lines, fl)
        assert abs(d - pins.penetration_np(lines, v)) < 1e-12
        assert abs(d - (1.0 if len(lines) == 2 else 0.5)) < 1e-9


def test_g4_silent_on_unique_lp3_argmin(oracle):
    """A unique least-penetration argmin never raises g4: the symmetric empty triangle (S:125,
    v = 0, delta = 0.5) and 200 generic random infeasible problems, whose near-argmin sets
    (grid, slack 1e-3) stay a few grid cells wide."""
    tri = []
    for a in (90.0, 210.0, 330.0):
        n = np.array([math.cos(math.radians(a)), math.sin(math.radians(a))])
        tri.append([0.5 * n[0], 0.5 * n[1], n[1], -n[0]])
    v, fl, d = oracle.solve_classify(tri, 1.33, [0.2, 0.1])
    assert fl & oracle.FLAG_INFEASIBLE and not fl & oracle.FLAG_G4
    assert np.hypot(*v) < 1e-9 and abs(d - 0.5) < 1e-9
    assert _argmin_diameter(tri, 1.33, 1e-3) < 0.02
    rng = np.random.default_rng(44)
    tested = 0
    while tested < 200:
        m = int(rng.integers(3, 12))
        ang = rng.uniform(0, 2 * np.pi, m)
        n = np.stack([np.cos(ang), np.sin(ang)], 1)
        s = rng.uniform(0.2, 1.2, m)
        lines = np.concatenate([s[:, None] * n, np.stack([n[:, 1], -n[:, 0]], 1)], axis=1)
        v, fl, d = oracle.solve_classify(lines, 1.33, rng.uniform(-1, 1, 2))
        if not fl & oracle.FLAG_INFEASIBLE:
            continue
        assert not fl & oracle.FLAG_G4, lines
        if tested < 40:
            assert _argmin_diameter(lines, 1.33, 1e-3, res=401) < 0.2
        tested += 1


def test_g2_near_parallel_crossing_inside_disc(oracle):
    """g2 (reading Q9): lines 5e-6 rad apart crossing INSIDE the speed disc.  A solver with
    the GPU's parallel tolerance (|det| <= 1e-5 -> "parallel": fail if the point lies on the
    wrong side, else skip) declares LP1 infeasible here, while the exact problem is
    feasible (vertex enumeration) -- the decision can flip, so the agent is flagged."""
    A = [0.5, 0.0, 0.0, -1.0]                      # permitted x >= 0.5
    q = np.array([0.5, 0.2])                       # the crossing, |q| < r
    B = _rot_line(A, 5e-6, q)
    B[0] -= 0.1 * B[2]                             # B's point 0.1 along B from the crossing
    B[1] -= 0.1 * B[3]
    den = A[2] * B[3] - A[3] * B[2]                 # det(D_A, D_B)
    num = A[2] * (B[1] - A[1]) - A[3] * (B[0] - A[0])  # det(D_A, P_B - P_A)
    assert abs(den) <= 1e-5 and num < 0.0          # the eps-solver's "parallel, pointing away"
    assert pins.lp_vertex_enumeration([A, B], 1.33, [0.0, 0.0]) is not None  # exactly feasible
    f, v, diag = oracle.lp2([A, B], 1.33, [0.0, 0.0])
    assert f == 2 and diag & oracle.FLAG_G2
    ve = pins.lp_vertex_enumeration([A, B], 1.33, [0.0, 0.0])
    assert np.allclose(v, ve, atol=1e-9)
    # the same pair, the other way round, in the least-penetration LP (same-direction pair
    # whose bisector crosses the disc) with a third line making the problem infeasible
    C = [-0.5, 0.0, 0.0, 1.0]
    v3, d3 = oracle.lp3([A, C, B], 2, 1.33, np.array([0.0, 0.0]))
    assert d3 & oracle.FLAG_G2


def test_g2_silent_when_crossing_outside_disc_or_angle_large(oracle):
    """No g2 when (a) the lines are as nearly parallel (5e-6 rad) but cross far outside the
    disc -- the eps-solver's parallel rule and the exact crossing then decide alike -- or
    (b) they cross inside the disc at 3e-5 rad, above the GPU tolerance (both solvers
    intersect)."""
    A = [0.5, 0.0, 0.0, -1.0]
    for q, th in (((0.5, 100.0), 5e-6), ((0.5, -100.0), -5e-6), ((0.5, 0.2), 3e-5), ((0.5, 0.2), -3e-5)):
        B = _rot_line(A, th, q)
        # move B's point to the disc (the crossing stays at q)
        t = -(B[0] * B[2] + B[1] * B[3])
        B = [B[0] + t * B[2], B[1] + t * B[3], B[2], B[3]]
        den = A[2] * B[3] - A[3] * B[2]
        num = A[2] * (B[1] - A[1]) - A[3] * (B[0] - A[0])
        cross_in_disc = math.hypot(*q) < 1.33
        if abs(den) <= 1e-5:
            assert not cross_in_disc
            # the eps rule (fail iff num < 0) agrees with the exact feasibility of {A, B}
            # on B's chord: exact LP1 on B clipped by A
            exact_ok = pins.lp_vertex_enumeration([A, B], 1.33, [B[0], B[1]]) is not None
            assert exact_ok == (num >= 0.0)
        for order in ([A, B], [B, A]):
            for pref in ([0.0, 0.0], [1.0, 0.3], [-1.0, -0.5]):
                f, v, diag = oracle.lp2(order, 1.33, pref)
                assert not diag & oracle.FLAG_G2, (q, th, pref)
