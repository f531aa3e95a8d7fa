"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the same
seeded inputs.

Bar (BASELINE.json north_star / DESIGN.md §4):
  * grid, cells and neighbour id lists: bit-exact;
  * single-step new velocities within 1e-4 m/s absolute (max-norm per component) for
    every agent the oracle does not flag degenerate (g1|g2|g4); degenerate < 0.1 %;
  * infeasible agents: max penetration of the GPU velocity, evaluated in fp64 on the
    oracle's lines, <= delta*_oracle + 1e-4;
  * positions within dt*1e-4 + 1 ulp_fp32(|p|) of p + dt v (oracle);
  * |v| <= maxSpeed (fp32 rounding slack 1e-6 relative).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle_par
import pins
from paper_1908_10107_b200 import workloads as W

pytestmark = pytest.mark.gpu

VTOL = 1e-4


@pytest.fixture(scope="module")
def orca():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1908_10107_b200 import build
    build.build()
    from paper_1908_10107_b200 import orca as O
    return O


def _ctx(orca, w, **over):
    p = dict(w["params"])
    p.update(over)
    o = orca.Orca(p)
    o.set_agents(w["pos"], w["vel"], w["pref"])
    if w.get("goals") is not None:
        o.set_goals(w["goals"], w["pref_speed"])
    return o, p


def _oracle_params(oracle, p):
    return oracle.make_params(**p)


def compare_step(orca, oracle, w, agents=None, max_deg=None, lp=None, variant=None, lp3_lanes=None, order=None,
                 **over):
    """One step from the state in w on both sides; returns a report dict and asserts the
    bar.  agents: optional sample of ids for large inputs (oracle computes one by one).
    lp: optional (seed, step) of the randomized LP order (reading Q8)."""
    o, p = _ctx(orca, w, **over)
    if variant is not None:
        o.set_variant(variant)
    if lp3_lanes is not None:
        o.set_lp3_lanes(lp3_lanes)
    if lp is not None:
        o.set_lp_order(True, lp[0], lp[1])
    if order is not None:
        o.set_lp_order(order)
    op = _oracle_params(oracle, p)
    origin, cs, dims = o.grid()
    oorigin, odims = oracle.grid_derive(w["pos"], op.neighborDist)
    assert np.array_equal(origin, oorigin.astype(np.float64)) and np.array_equal(dims, odims)
    # cells (bit-exact)
    cx, cy = o.debug_cells()
    ocx, ocy = oracle.cells(w["pos"], oorigin, op.neighborDist, odims)
    assert np.array_equal(cx, ocx) and np.array_equal(cy, ocy)
    # one step (dry) on the GPU
    v, fl, nb, cnt = o.debug_step()
    ids = np.arange(len(w["pos"])) if agents is None else np.asarray(agents)
    ref = oracle_par.step(op, w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"),
                          pref_speed=w.get("pref_speed", 1.0), agents=agents, want_nbrs=True,
                          lp_seed=None if lp is None else lp[0], lp_step=0 if lp is None else lp[1],
                          vtest=v[ids].astype(np.float64))
    # neighbours (bit-exact)
    assert np.array_equal(cnt[ids], ref["cnt"])
    assert np.array_equal(nb[ids], ref["nbr"])
    # the automatic kernel choice (variant -1) and the one-thread-per-agent kernel (0) agree
    # bit for bit, so the oracle comparison below covers both
    if variant is None:
        o.set_variant(0)
        v0, fl0, nb0, cnt0 = o.debug_step()
        o.set_variant(-1)
        assert np.array_equal(v0, v) and np.array_equal(nb0, nb) and np.array_equal(cnt0, cnt)
        assert np.array_equal(fl0 & 1, fl & 1)
    # velocities
    ov = ref["vel"]
    gv = v[ids].astype(np.float64)
    err = np.max(np.abs(gv - ov), axis=1)
    deg = (ref["flags"] & oracle.FLAG_DEGENERATE) != 0
    bad = (err > VTOL) & ~deg
    k = p["maxNeighbors"]
    # infeasible: penetration of the GPU answer on the oracle's own lines (every agent)
    inf = (ref["flags"] & oracle.FLAG_INFEASIBLE) != 0
    worst_pen_gap = float((ref["dtest"] - ref["delta"])[inf].max()) if inf.any() else 0.0
    speed = np.hypot(gv[:, 0], gv[:, 1])
    report = dict(n=len(ids), max_err=float(err[~deg].max()) if (~deg).any() else 0.0,
                  n_bad=int(bad.sum()), n_deg=int(deg.sum()), n_inf=int(inf.sum()),
                  gpu_inf=int(((fl[ids] & 1) != 0).sum()), worst_pen_gap=worst_pen_gap,
                  max_speed=float(speed.max()) if len(speed) else 0.0)
    assert report["n_bad"] == 0, (report, np.nonzero(bad)[0][:10])
    assert report["n_deg"] <= (max(1, 0.001 * len(ids)) if max_deg is None else max_deg), report
    assert worst_pen_gap <= VTOL, report
    assert np.all(speed <= p["maxSpeed"] * (1 + 1e-6) + 1e-7), report
    # a real step agrees with the dry step and moves p + dt v
    o.step(1)
    pos1, vel1 = o.get_state()
    assert np.array_equal(vel1, v)
    pexp = ref["pos"]
    ptol = p["timeStep"] * VTOL + np.spacing(np.abs(pexp).max(axis=1).astype(np.float32)).astype(np.float64)
    perr = np.max(np.abs(pos1[ids].astype(np.float64) - pexp), axis=1)
    assert np.all((perr <= ptol + 1e-12) | deg), perr.max()
    o.close()
    return report


# --------------------------------------------------------------------------- cases
@pytest.mark.parametrize("config,n,rho", [
    ("uniform", 3000, 0.25), ("uniform", 3000, 0.5), ("uniform", 2000, 0.01), ("uniform", 2500, 0.1),
    ("corridor", 3000, None), ("dense", 4000, None),
])
def test_step_parity_small(orca, oracle, config, n, rho):
    if config == "corridor":
        w = W.corridor(n=n, length=n / (0.25 * 30.0), width=30.0)
    else:
        w = W.make(config, n=n, rho=rho)
    compare_step(orca, oracle, w)


def test_step_parity_circle_goals(orca, oracle):
    w = W.make("circle")
    compare_step(orca, oracle, w)


@pytest.mark.parametrize("warm", [5, 20])
def test_step_parity_warm_state(orca, oracle, warm):
    """State warmed up by the ORACLE (fp32 state between steps), then one step on both."""
    w = W.make("uniform", n=2000, rho=0.5)
    op = oracle.make_params(**w["params"])
    pos, vel, _ = oracle.run(op, w["pos"], w["vel"], pref=w["pref"], steps=warm)
    w2 = dict(w, pos=pos, vel=vel)
    compare_step(orca, oracle, w2)


def test_step_parity_corridor_warm(orca, oracle):
    w = W.corridor(n=3000, length=400.0, width=30.0)
    op = oracle.make_params(**w["params"])
    pos, vel, _ = oracle.run(op, w["pos"], w["vel"], pref=w["pref"], steps=15)
    compare_step(orca, oracle, dict(w, pos=pos, vel=vel))


def test_circle_warm_goals(orca, oracle):
    """The circle's central crush (many infeasible agents, overlaps) at oracle step 300."""
    w = W.make("circle")
    op = oracle.make_params(**w["params"])
    pos, vel, _ = oracle.run(op, w["pos"], w["vel"], goals=w["goals"], pref_speed=1.0, steps=300)
    compare_step(orca, oracle, dict(w, pos=pos, vel=vel))


@pytest.mark.parametrize("k", [0, 1, 7, 32])
def test_step_parity_k(orca, oracle, k):
    w = W.make("uniform", n=1500, rho=0.3)
    compare_step(orca, oracle, w, maxNeighbors=k)


def test_tie_lattice_neighbors(orca, oracle):
    pos = W.tie_lattice(30)
    w = dict(pos=pos, vel=np.zeros_like(pos), pref=np.zeros_like(pos), goals=None,
             params=dict(W.DEFAULT_PARAMS, neighborDist=2.5, radius=0.2))
    compare_step(orca, oracle, w)


@pytest.mark.parametrize("ulp", [False, True])
def test_subcell_boundary_lattice(orca, oracle, ulp):
    """Agents exactly on the sort's fine-column (cs/4) and sub-row (cs/8) boundaries -- and one
    fp32 ulp either side of them -- with many exact distance ties: the search windows of the
    sub-cell runs still give the bit-exact cells and (kappa, id) neighbour lists."""
    cs = 4.0
    xs = np.arange(40, dtype=np.float32) * np.float32(cs / 4)
    ys = np.arange(40, dtype=np.float32) * np.float32(cs / 8)
    pos = np.stack(np.meshgrid(xs, ys, indexing="ij"), -1).reshape(-1, 2).astype(np.float32)
    pos += np.float32(cs)  # the grid origin is min - cs: boundaries at whole multiples
    if ulp:
        rng = np.random.default_rng(4)
        pick = rng.random(pos.shape) < 0.3
        up = rng.random(pos.shape) < 0.5
        pos = np.where(pick, np.where(up, np.nextafter(pos, np.float32(np.inf)),
                                      np.nextafter(pos, np.float32(-np.inf))), pos).astype(np.float32)
    rng = np.random.default_rng(5)
    pref = rng.uniform(-1, 1, pos.shape).astype(np.float32)
    w = dict(pos=pos, vel=np.zeros_like(pos), pref=pref, goals=None,
             params=dict(W.DEFAULT_PARAMS, neighborDist=cs, radius=0.2))
    rep = compare_step(orca, oracle, w)
    print("subcell lattice", ulp, rep)


def test_coincident_agents(orca, oracle):
    """Coincident agents with equal velocity (reading Q15, g1): deterministic +-x push."""
    rng = np.random.default_rng(9)
    pos = rng.uniform(0, 40, (400, 2)).astype(np.float32)
    pos[300:310] = pos[0]  # ten coincident copies of agent 0
    vel = np.zeros_like(pos)
    pref = rng.uniform(-1, 1, (400, 2)).astype(np.float32)
    w = dict(pos=pos, vel=vel, pref=pref, goals=None, params=dict(W.DEFAULT_PARAMS))
    rep = compare_step(orca, oracle, w, max_deg=11)
    assert rep["n_deg"] == 11


def test_empty_and_single(orca, oracle):
    o = orca.Orca(W.DEFAULT_PARAMS)
    e = np.zeros((0, 2), np.float32)
    o.set_agents(e, e, e)
    o.step(3)
    p, v = o.get_state()
    assert p.shape == (0, 2)
    one = np.array([[1.0, 2.0]], np.float32)
    o.set_agents(one, np.zeros_like(one), np.array([[3.0, 0.0]], np.float32))
    o.step(1)
    p, v = o.get_state()
    assert np.allclose(v, [[1.33, 0.0]], atol=1e-6) and np.allclose(p, [[1.0 + 0.25 * 1.33, 2.0]], atol=1e-6)
    o.close()


def test_not_ready_and_nan(orca):
    o = orca.Orca(W.DEFAULT_PARAMS)
    with pytest.raises(orca.OrcaError) as e:
        o.step(1)
    assert e.value.status == 2
    bad = np.array([[np.nan, 0.0]], np.float32)
    with pytest.raises(orca.OrcaError) as e:
        o.set_agents(bad, np.zeros_like(bad), np.zeros_like(bad))
    assert e.value.status == 1
    o.close()


def test_device_pointer_inputs(orca, oracle):
    """torch CUDA tensors in, torch CUDA tensors out: same result as host arrays."""
    import torch
    w = W.make("uniform", n=2000, rho=0.25)
    a, _ = _ctx(orca, w)
    a.step(3)
    pa, va = a.get_state()
    b = orca.Orca(w["params"])
    tp = torch.from_numpy(w["pos"]).cuda()
    tv = torch.from_numpy(w["vel"]).cuda()
    tq = torch.from_numpy(w["pref"]).cuda()
    b.set_agents(tp, tv, tq)
    b.step(3)
    op = torch.empty_like(tp)
    ov = torch.empty_like(tv)
    b.get_state(op, ov)
    assert np.array_equal(op.cpu().numpy(), pa) and np.array_equal(ov.cpu().numpy(), va)
    a.close()
    b.close()


def test_deterministic_and_graph_equals_timed(orca):
    w = W.make("uniform", n=20000, rho=0.25)
    a, _ = _ctx(orca, w)
    b, _ = _ctx(orca, w)
    c, _ = _ctx(orca, w)
    a.step(10)
    b.step(10)
    c.step_timed(10)
    pa, va = a.get_state()
    pb, vb = b.get_state()
    pc, vc = c.get_state()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)
    assert np.array_equal(pa, pc) and np.array_equal(va, vc)
    for o in (a, b, c):
        o.close()


def test_multistep_invariants_circle(orca):
    """C0 on the GPU: speed cap every step; all agents reach their goals by step 1000."""
    w = W.make("circle")
    o, p = _ctx(orca, w)
    for _ in range(20):
        o.step(50)
        pos, vel = o.get_state()
        assert np.all(np.hypot(vel[:, 0], vel[:, 1]) <= p["maxSpeed"] * (1 + 1e-6))
    dist = np.hypot(*(pos - w["goals"]).T)
    assert np.all(dist < p["radius"]), np.sort(dist)[-5:]
    st = o.stats()
    assert st["steps"] == 1000 and st["infeasible"] > 0
    o.close()


# ------------------------------------------------------- full sizes, every agent
def check_warm_state(o, oracle, p, pref=None, goals=None, pref_speed=1.0, props=None, label=""):
    """The context's CURRENT state (after real GPU steps: the history search radius, the
    bench's automatic kernel choice and launch configuration) against the oracle on that
    same fp32 state and frozen grid, for EVERY active agent: cells and neighbour lists
    bit-exact, velocities within 1e-4 outside the degenerate set, infeasible agents'
    penetration on the oracle's lines, a real step equal to the dry step, positions.  Ids of
    removed agents (NaN) are left out on both sides: the oracle steps the active crowd."""
    pos, vel = o.get_state()
    act = np.isfinite(pos[:, 0])
    aid = np.nonzero(act)[0]
    origin, cs, dims = o.grid()
    origin32 = np.asarray(origin, np.float32)
    op = oracle.make_params(**p)
    cx, cy = o.debug_cells()
    ocx, ocy = oracle.cells(pos[aid], origin32, op.neighborDist, np.asarray(dims, np.int32))
    assert np.array_equal(cx[aid], ocx) and np.array_equal(cy[aid], ocy), label
    v, fl, nb, cnt = o.debug_step()
    sub = lambda a: None if a is None else np.ascontiguousarray(a[aid])
    sprops = None if props is None else {k_: sub(v_) for k_, v_ in props.items()}
    ref = oracle_par.step(op, pos[aid], vel[aid], pref=sub(pref), goals=sub(goals), pref_speed=pref_speed,
                          origin=origin32, dims=np.asarray(dims, np.int32), want_nbrs=True, props=sprops,
                          vtest=v[aid].astype(np.float64))
    onb = np.where(ref["nbr"] >= 0, aid[np.maximum(ref["nbr"], 0)], -1)  # compacted -> global ids
    assert np.array_equal(cnt[aid], ref["cnt"]), label
    assert np.array_equal(nb[aid], onb), label
    gv = v[aid].astype(np.float64)
    err = np.max(np.abs(gv - ref["vel"]), axis=1)
    deg = (ref["flags"] & oracle.FLAG_DEGENERATE) != 0
    inf = (ref["flags"] & oracle.FLAG_INFEASIBLE) != 0
    bad = (err > VTOL) & ~deg
    gap = float((ref["dtest"] - ref["delta"])[inf].max()) if inf.any() else 0.0
    vmax = np.float64(p["maxSpeed"]) if props is None else props["maxSpeed"][aid].astype(np.float64)
    speed = np.hypot(gv[:, 0], gv[:, 1])
    report = dict(label=label, n=len(aid), max_err=float(err[~deg].max()) if (~deg).any() else 0.0,
                  n_bad=int(bad.sum()), excluded_degenerate=int(deg.sum()), n_inf=int(inf.sum()),
                  gpu_inf=int(((fl[aid] & 1) != 0).sum()), worst_pen_gap=gap,
                  g1=int(((ref["flags"] & oracle.FLAG_G1) != 0).sum()),
                  g2=int(((ref["flags"] & oracle.FLAG_G2) != 0).sum()),
                  g4=int(((ref["flags"] & oracle.FLAG_G4) != 0).sum()))
    print("parity", report)
    assert report["n_bad"] == 0, (report, aid[np.nonzero(bad)[0][:10]])
    assert report["excluded_degenerate"] <= max(1, 0.001 * len(aid)), report
    assert gap <= VTOL, report
    assert np.all(speed <= vmax * (1 + 1e-6) + 1e-7), report
    o.step(1)
    pos1, vel1 = o.get_state()
    still = np.isfinite(pos1[aid, 0])  # (removal after this step)
    assert np.array_equal(vel1[aid][still], v[aid][still]), label
    pexp = ref["pos"]
    ptol = p["timeStep"] * VTOL + np.spacing(np.abs(pexp).max(axis=1).astype(np.float32)).astype(np.float64)
    perr = np.max(np.abs(pos1[aid].astype(np.float64) - pexp), axis=1)
    assert np.all((perr <= ptol + 1e-12) | deg | ~still), perr[still].max()
    return report


@pytest.mark.parametrize("config", ["uniform", "dense", "uniform_1m"])
def test_full_size_every_agent(orca, oracle, config):
    """BASELINE sizes (C2 100k, C3 500k, C2' 1M) in the bench's launch configuration (the
    automatic kernel choice: inline LP3 at 100k, k_step + k_lp3 above), from a state warmed
    by 20 real GPU steps (history search radius), every agent against the oracle."""
    w = W.make(config)
    o, p = _ctx(orca, w)
    o.step(20)
    rep = check_warm_state(o, oracle, p, pref=w["pref"], label=config)
    assert rep["n"] == len(w["pos"])
    o.close()


def test_full_size_heterogeneous_goals_removal(orca, oracle):
    """§8(f1)+(f2) at the C2 size: 100k agents with per-agent radius / maxSpeed / desired
    speed, goal seeking and removal at the goal, after 20 GPU steps in which
    agents have left; the oracle steps the remaining crowd, every agent compared."""
    w = W.make("uniform")
    n = len(w["pos"])
    rng = np.random.default_rng(31)
    goals = (w["pos"] + rng.uniform(-12, 12, w["pos"].shape)).astype(np.float32)
    props = _het_props(n, seed=13)
    o, p = _ctx(orca, dict(w, goals=goals, pref_speed=1.0))
    o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
    o.set_goal_removal(0.75)
    o.step(20)
    assert 0 < o.stats()["removed"] < n // 2
    n_active = o.count()
    rep = check_warm_state(o, oracle, p, pref=w["pref"], goals=goals, props=props, label="het+goals+removal 100k")
    assert rep["n"] == n_active
    o.close()


def test_max_speed_zero(orca, oracle):
    """maxSpeed = 0 (allowed by orca_create): the speed disc is a point, every agent's LP is
    infeasible unless all its half-planes admit v = 0; both sides return v = 0 exactly and
    nobody moves."""
    w = W.make("uniform", n=3000, rho=0.3)
    rep = compare_step(orca, oracle, w, maxSpeed=0.0)
    o, p = _ctx(orca, w, maxSpeed=0.0)
    o.step(3)
    pos, vel = o.get_state()
    assert np.all(vel == 0.0) and np.array_equal(pos, w["pos"])
    o.close()
    print("maxSpeed=0", rep)


def test_c4_4m_eight_strips_bit_identical_and_oracle(orca, oracle):
    """C4 (BASELINE configs[4]): 4M agents in 8 loopback strips (halo + migration through the
    exchange buffers) equal one strip bit for bit over 72 steps; the final
    state is then checked against the oracle for every agent."""
    w = W.make("uniform_4m")
    n = len(w["pos"])
    a, p = _ctx(orca, w)
    b = orca.Orca(p, strips=8)
    b.set_agents(w["pos"], w["vel"], w["pref"])
    for chunk in (1, 7, 64):
        a.step(chunk)
        b.step(chunk)
        pa, va = a.get_state()
        pb, vb = b.get_state()
        assert np.array_equal(pa, pb) and np.array_equal(va, vb), chunk
    assert b.count() == n
    sa, sb = a.stats(), b.stats()
    for key in ("infeasible", "degenerate", "collision_pairs"):
        assert sa[key] == sb[key], key
    b.close()
    rep = check_warm_state(a, oracle, p, pref=w["pref"], label="C4 4M")
    assert rep["n"] == n
    a.close()


def test_history_bound_path_consistent(orca):
    """After real steps the query uses the previous k-th distance as its search bound; a
    fresh context holding the same state uses the density guess.  Both are exact, so the
    neighbour lists and velocities must agree bit for bit (self-consistency, not an oracle
    claim), and the lists must equal brute force on that state (tests/pins.py)."""
    w = W.make("uniform", n=6000, rho=0.4)
    a, p = _ctx(orca, w)
    a.step(7)
    pos, vel = a.get_state()
    v1, f1, nb1, c1 = a.debug_step()
    b = orca.Orca(p)
    b.set_agents(pos, vel, w["pref"])
    # the fresh context re-derives the grid from the current positions; only compare if equal
    v2, f2, nb2, c2 = b.debug_step()
    assert np.array_equal(nb1, nb2) and np.array_equal(c1, c2)
    assert np.array_equal(v1, v2)
    bn, bc = pins.brute_neighbors(pos, p["neighborDist"], p["maxNeighbors"])
    assert np.array_equal(c1, bc) and np.array_equal(nb1.astype(np.int64), bn)
    a.close()
    b.close()


# ------------------------------------------------------------ strips
@pytest.mark.parametrize("strips,config,n", [(2, "uniform", 20000), (3, "corridor", 10000), (4, "uniform", 30000),
                                             (8, "uniform", 60000)])
def test_strips_bit_identical(orca, strips, config, n):
    """The strip decomposition (halo + migration through the same exchange buffers NCCL
    moves) gives bit-identical state to one strip: the same ordered neighbour lists with
    global-id ties feed the same arithmetic."""
    w = W.make(config, n=n) if config != "corridor" else W.corridor(n=n)
    a, p = _ctx(orca, w)
    b = orca.Orca(p, strips=strips)
    b.set_agents(w["pos"], w["vel"], w["pref"])
    bounds = b.strip_bounds()
    assert bounds[0, 0] == 0 and bounds[-1, 1] == a.grid()[2][0]
    assert np.all(bounds[1:, 0] == bounds[:-1, 1])
    va, fa, na, ca = a.debug_step()
    vb, fb, nb, cb = b.debug_step()
    assert np.array_equal(na, nb) and np.array_equal(va, vb) and np.array_equal(fa, fb)
    for chunk in (1, 9, 30):
        a.step(chunk)
        b.step(chunk)
        pa, wa = a.get_state()
        pb, wb = b.get_state()
        assert np.array_equal(pa, pb) and np.array_equal(wa, wb), chunk
    assert b.count() == n
    sa, sb = a.stats(), b.stats()
    for key in ("infeasible", "degenerate", "collision_pairs"):
        assert sa[key] == sb[key], key
    ids, lp, lv = b.get_local_state()
    assert np.array_equal(np.sort(ids), np.arange(n))
    a.close()
    b.close()


@pytest.mark.parametrize("strips,transport", [(2, 0), (4, 0), (4, 1), (8, 0)])
def test_strips_overlap_bit_identical(orca, strips, transport):
    """Halo overlap (orca_set_overlap): boundary columns first, the exchange and
    k_receive on a second stream while the interior columns step -- bit-identical to the
    un-overlapped strips and to one strip, with both transports; the step launches the step
    kernel twice per overlapping strip."""
    import os
    w = W.make("uniform", n=80000)
    a, p = _ctx(orca, w)
    runs = []
    os.environ["ORCA_ONE_STREAM"] = "1"  # loopback strips on one stream (else they overlap anyway)
    try:
        for mode in (0, 1):
            b = orca.Orca(p, strips=strips)
            b.set_agents(w["pos"], w["vel"], w["pref"])
            b.set_transport(transport)
            b.set_overlap(mode)
            runs.append(b)
        k0, k1 = runs[0].launch_info()["kernels_per_step"], runs[1].launch_info()["kernels_per_step"]
        assert k1 == k0 + strips  # every strip here has >= 4 columns
        for chunk in (1, 9, 30):
            a.step(chunk)
            ref = a.get_state()
            for b in runs:
                b.step(chunk)
                st = b.get_state()
                assert np.array_equal(ref[0], st[0]) and np.array_equal(ref[1], st[1]), chunk
    finally:
        del os.environ["ORCA_ONE_STREAM"]
    sa = a.stats()
    for b in runs:
        sb = b.stats()
        for key in ("infeasible", "degenerate", "collision_pairs"):
            assert sa[key] == sb[key], key
        b.close()
    a.close()


@pytest.mark.parametrize("strips", [2, 4, 8])
def test_strips_own_streams_bit_identical(orca, strips):
    """Loopback strips on one stream per strip (peer-memory exchange ordered by the arrival
    flags and step-parity buffers across streams) equal one strip and the
    single-stream strips bit for bit, over steps that cross a 64-step graph chunk."""
    import os
    w = W.make("uniform", n=60000)
    a, p = _ctx(orca, w)
    b = orca.Orca(p, strips=strips)
    b.set_agents(w["pos"], w["vel"], w["pref"])
    os.environ["ORCA_ONE_STREAM"] = "1"
    try:
        c = orca.Orca(p, strips=strips)
        c.set_agents(w["pos"], w["vel"], w["pref"])
        for chunk in (1, 70):
            c.step(chunk)
    finally:
        del os.environ["ORCA_ONE_STREAM"]
    for chunk in (1, 70):
        a.step(chunk)
        b.step(chunk)
    ra, rb, rc = a.get_state(), b.get_state(), c.get_state()
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
    assert np.array_equal(ra[0], rc[0]) and np.array_equal(ra[1], rc[1])
    assert a.stats()["infeasible"] == b.stats()["infeasible"]
    for o in (a, b, c):
        o.close()


def test_strips_goals_circle(orca):
    """Goal seeking through the strips (the circle's agents cross every strip)."""
    w = W.make("circle")
    a, p = _ctx(orca, w)
    b = orca.Orca(p, strips=3)
    b.set_agents(w["pos"], w["vel"], w["pref"])
    b.set_goals(w["goals"], w["pref_speed"])
    a.step(400)
    b.step(400)
    pa, va = a.get_state()
    pb, vb = b.get_state()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)
    a.close()
    b.close()


@pytest.mark.parametrize("order", [0, 2])
@pytest.mark.parametrize("config,n,rho", [("uniform", 20000, 0.25), ("dense", 20000, None), ("uniform", 5000, 0.02)])
def test_variants_bit_identical(orca, config, n, rho, order):
    """Thread-per-agent with a shared-memory (0) or register (2) top-k list, the
    8-lane-group-per-agent kernel (1), the work-unit LP2 (3) and two lanes per agent (4): same
    neighbours, velocities
    and trajectories bit for bit (exact comparators; the group and work-unit LPs use exact
    min/max reductions), in the greedy LP order (0, default) and the sequential neighbour
    order (2, where variant 3 runs the work units).  The work-unit LP also reproduces every
    flag and work counter."""
    w = W.make(config, n=n, rho=rho) if rho else W.make(config, n=n)
    ctxs = []
    for v in (0, 1, 2, 3, 4):
        o, p = _ctx(orca, w)
        o.set_variant(v)
        o.set_lp_order(order)
        ctxs.append(o)
    r = [o.debug_step() for o in ctxs]
    for q in (1, 2, 3, 4):
        assert np.array_equal(r[0][2], r[q][2]) and np.array_equal(r[0][3], r[q][3])
        assert np.array_equal(r[0][0], r[q][0])
        assert np.array_equal(r[0][1] & 1, r[q][1] & 1)
    assert np.array_equal(r[0][1], r[3][1])
    assert ctxs[0].work() == ctxs[3].work()
    # the lane-pair variant (4; greedy order only, else it runs as 0) reproduces every flag and
    # work counter too
    assert np.array_equal(r[0][1], r[4][1])
    assert ctxs[0].work() == ctxs[4].work()
    for o in ctxs:
        o.step(25)
    s = [o.get_state() for o in ctxs]
    for q in (1, 2, 3, 4):
        assert np.array_equal(s[0][0], s[q][0]) and np.array_equal(s[0][1], s[q][1])
    for o in ctxs:
        o.close()


@pytest.mark.parametrize("n,het", [(170000, False), (170000, True), (100000, False), (60000, False)])
def test_specialised_kernels_bit_identical(orca, n, het):
    """The default configurations run k_step instantiations compiled for them (DESIGN.md §10,
    r02ai-au): LP3 placement fixed (k_lp3 above one wave, the block queue below it, 256-thread
    blocks with an 85-register budget while one wave of those fits), one homogeneous strip
    (MONO), the lane pair with its own register budget.  Each must equal the general kernels --
    variant 2 (register top-k list) and variant 3 (work-unit template, greedy order) run the
    general instantiation -- in dry-step velocities, flags and lists and in 12 real steps (state
    and statistics), with per-agent properties too (the non-MONO specialisation)."""
    w = W.make("uniform", n=n)
    ctxs = []
    for v in (-1, 2, 3):
        o, _ = _ctx(orca, w)
        o.set_variant(v)
        if het:
            props = _het_props(n, seed=9)
            o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
        ctxs.append(o)
    kc = [o.kernel_config() for o in ctxs]
    exp = {170000: dict(variant=0, lp3_placement=0, compiled_for_lp3=0, threads=128),
           100000: dict(variant=0, lp3_placement=2, compiled_for_lp3=2, threads=256, min_blocks_per_sm=3),
           60000: dict(variant=4, lp3_placement=2, compiled_for_lp3=2, threads=128, min_blocks_per_sm=6)}[n]
    assert {q: kc[0][q] for q in exp} == exp, kc[0]
    assert kc[0]["mono"] == (0 if het else 1)
    assert kc[1]["compiled_for_lp3"] == -1 and kc[2]["compiled_for_lp3"] == -1  # the general kernels
    r = [o.debug_step() for o in ctxs]
    assert np.count_nonzero(r[0][1] & 1) > 0  # infeasible agents: the LP3 placement is exercised
    for q in (1, 2):
        assert np.array_equal(r[0][0], r[q][0]), q  # velocities
        assert np.array_equal(r[0][2], r[q][2]) and np.array_equal(r[0][3], r[q][3]), q  # lists
        assert np.array_equal(r[0][1] & 1, r[q][1] & 1), q  # infeasible
    assert np.array_equal(r[0][1], r[2][1])  # every flag (the same half-plane and LP code)
    for o in ctxs:
        o.step(12)
    s = [o.get_state() for o in ctxs]
    st = [o.stats() for o in ctxs]
    for q in (1, 2):
        assert np.array_equal(s[0][0], s[q][0]) and np.array_equal(s[0][1], s[q][1]), q
        assert st[0] == st[q], q
    for o in ctxs:
        o.close()


# ---------------------------------------------------- goals + removal (§8(f1))
def test_removal_one_step_vs_oracle(orca, oracle):
    """After one step an agent is removed iff its new position is strictly within R of its
    goal; compared with the oracle's p' = p + dt v' outside an fp32 band."""
    rng = np.random.default_rng(17)
    w = W.make("uniform", n=3000, rho=0.2)
    R = 0.6
    goals = (w["pos"] + rng.uniform(-1.2, 1.2, w["pos"].shape)).astype(np.float32)
    o, p = _ctx(orca, dict(w, goals=goals, pref_speed=1.0))
    o.set_goal_removal(R)
    ref = oracle.step(oracle.make_params(**p), w["pos"], w["vel"], goals=goals, pref_speed=1.0)
    o.step(1)
    act = o.active()
    dg = np.hypot(*(goals.astype(np.float64) - ref["pos"]).T)
    sure_in, sure_out = dg < R - 1e-4, dg > R + 1e-4
    assert np.all(~act[sure_in]) and np.all(act[sure_out])
    assert o.count() == int(act.sum()) and o.stats()["removed"] == int((~act).sum())
    pos, vel = o.get_state()
    assert np.all(np.isnan(pos[~act])) and np.all(np.isfinite(pos[act]))
    # removed agents are no longer observed: next step's neighbour lists only hold active ids
    v, fl, nb, cnt = o.debug_step()
    ids = nb[act][nb[act] >= 0]
    assert np.all(act[ids])
    o.close()


@pytest.mark.parametrize("strips", [1, 3])
def test_circle_all_removed(orca, strips):
    """C0 with removal at the goal: the simulation ends (count 0) within 1000 steps."""
    w = W.make("circle")
    o = orca.Orca(w["params"], strips=strips if strips > 1 else 0)
    o.set_agents(w["pos"], w["vel"], w["pref"])
    o.set_goals(w["goals"], w["pref_speed"])
    o.set_goal_removal(w["params"]["radius"])
    last = o.count()
    for _ in range(20):
        o.step(50)
        c = o.count()
        assert c <= last
        last = c
    assert last == 0 and o.stats()["removed"] == 100
    o.close()


def test_two_way_crossing_runs(orca):
    """E1a: 2,500 agents cross and are removed at their goals."""
    w = W.make("two_way")
    o, p = _ctx(orca, w)
    o.set_goal_removal(p["radius"])
    o.step(1500)
    st = o.stats()
    assert st["removed"] >= 0.9 * 2500, st
    o.close()


# ------------------------------------------ heterogeneous crowds (§8(f2))
def _het_props(n, seed=5):
    rng = np.random.default_rng(seed)
    radius = rng.choice([0.5, 0.75, 1.0], n).astype(np.float32)
    desired = rng.choice([1.0, 1.33, 2.0], n).astype(np.float32)
    return dict(radius=radius, maxSpeed=(1.25 * desired).astype(np.float32), prefSpeed=desired)


@pytest.mark.parametrize("goals", [False, True])
def test_heterogeneous_step_parity(orca, oracle, goals):
    """Per-agent radius (R = r_i + r_j), maxSpeed and desired speed vs the oracle."""
    w = W.make("uniform", n=4000, rho=0.15)
    props = _het_props(len(w["pos"]))
    if goals:
        rng = np.random.default_rng(8)
        w = dict(w, goals=(w["pos"] + rng.uniform(-40, 40, w["pos"].shape)).astype(np.float32), pref_speed=1.0)
    o, p = _ctx(orca, w)
    o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
    v, fl, nb, cnt = o.debug_step()
    ref = oracle.step(oracle.make_params(**p), w["pos"], w["vel"], pref=w["pref"], goals=w.get("goals"),
                      pref_speed=1.0, want_nbrs=True, props=props)
    assert np.array_equal(nb, ref["nbr"]) and np.array_equal(cnt, ref["cnt"])
    deg = (ref["flags"] & oracle.FLAG_DEGENERATE) != 0
    err = np.abs(v.astype(np.float64) - ref["vel"]).max(axis=1)
    assert np.all((err <= VTOL) | deg), err[~deg].max()
    assert deg.sum() <= max(1, 0.001 * len(deg))
    sp = np.hypot(*v.T.astype(np.float64))
    assert np.all(sp <= props["maxSpeed"].astype(np.float64) * (1 + 1e-6) + 1e-7)
    o.step(1)
    _, vel1 = o.get_state()
    assert np.array_equal(vel1, v)
    o.close()


def test_heterogeneous_strips_and_history(orca):
    """Heterogeneous crowd through 3 strips (radii travel with migrants and halos) equals
    one strip bit for bit, and its history-bound query equals a fresh context's."""
    w = W.make("uniform", n=20000, rho=0.15)
    props = _het_props(len(w["pos"]), seed=9)
    a, p = _ctx(orca, w)
    a.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
    b = orca.Orca(p, strips=3)
    b.set_agents(w["pos"], w["vel"], w["pref"])
    b.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
    a.step(30)
    b.step(30)
    pa, va = a.get_state()
    pb, vb = b.get_state()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)
    c = orca.Orca(p)
    c.set_agents(pa, va, w["pref"])
    c.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
    r1, r2 = a.debug_step(), c.debug_step()
    assert np.array_equal(r1[2], r2[2]) and np.array_equal(r1[0], r2[0])
    for o in (a, b, c):
        o.close()


def test_step_trace_frames(orca):
    """Trace dump: frames equal get_state after every step; removed agents
    read NaN; pinned torch buffers work (copy engine overlapped)."""
    import torch
    w = W.make("circle")
    a, p = _ctx(orca, w)
    b, _ = _ctx(orca, w)
    a.set_goal_removal(0.5)
    b.set_goal_removal(0.5)
    frames = a.step_trace(120)
    for s in range(120):
        b.step(1)
        pb, _ = b.get_state()
        assert np.array_equal(frames[s], pb, equal_nan=True), s
    fr = torch.empty((30, 100, 2), dtype=torch.float32).pin_memory()
    vf = torch.empty((30, 100, 2), dtype=torch.float32).pin_memory()
    a.step_trace(30, fr, vf)
    b.step(30)
    pb, vb = b.get_state()
    assert np.array_equal(fr[-1].numpy(), pb, equal_nan=True) and np.array_equal(vf[-1].numpy(), vb, equal_nan=True)
    a.close()
    b.close()


# ------------------------------------- randomized LP constraint order (§8(f3), Q8)
@pytest.mark.parametrize("config,n,rho,lp", [("uniform", 3000, 0.5, (2024, 0)), ("dense", 4000, None, (7, 123456)),
                                             ("uniform", 2500, 0.1, (2 ** 64 - 1, 99))])
def test_randomized_order_parity(orca, oracle, config, n, rho, lp):
    """The same counter-based Fisher-Yates order on both sides: velocities within the bar,
    including the infeasible agents whose least-penetration answer may depend on order."""
    w = W.make(config, n=n, rho=rho) if rho else W.make(config, n=n)
    r = compare_step(orca, oracle, w, lp=lp)
    assert r["n_inf"] > 0


def test_randomized_order_circle_crush(orca, oracle):
    """The circle's central crush (order-sensitive infeasible LPs) with a randomized order."""
    w = W.make("circle")
    op = oracle.make_params(**w["params"])
    pos, vel, _ = oracle.run(op, w["pos"], w["vel"], goals=w["goals"], pref_speed=1.0, steps=300,
                             lp_seed=5, lp_step=0)
    compare_step(orca, oracle, dict(w, pos=pos, vel=vel), lp=(5, 300))


def test_randomized_order_resume_and_strips(orca):
    """t advances by one per step and survives set_agents (checkpoint/resume reproduces the
    uninterrupted run bit for bit); strips and the register-list variant agree bit for bit;
    nearest-first and randomized runs share every feasible velocity."""
    w = W.make("uniform", n=20000, rho=0.4)
    a, p = _ctx(orca, w)
    a.set_lp_order(True, 11, 40)
    a.step(6)
    b, _ = _ctx(orca, w)  # resumed: 2 steps, reload the state, 4 more
    b.set_lp_order(True, 11, 40)
    b.step(2)
    pos2, vel2 = b.get_state()
    b.set_agents(pos2, vel2, w["pref"])
    b.step(4)
    c = orca.Orca(p)  # fresh context from the step-2 checkpoint at t = 42
    c.set_agents(pos2, vel2, w["pref"])
    c.set_lp_order(True, 11, 42)
    c.step(4)
    d = orca.Orca(p, strips=3)
    d.set_agents(w["pos"], w["vel"], w["pref"])
    d.set_lp_order(True, 11, 40)
    d.step(6)
    e, _ = _ctx(orca, w)
    e.set_variant(2)
    e.set_lp_order(True, 11, 40)
    e.step(6)
    ref = a.get_state()
    for o in (b, c, d, e):
        s = o.get_state()
        assert np.array_equal(ref[0], s[0]) and np.array_equal(ref[1], s[1])
    # a different t changes the order: some infeasible agent moves differently, while the
    # feasible ones (unique optimum) are unchanged
    f, _ = _ctx(orca, w)
    g, _ = _ctx(orca, w)
    f.set_lp_order(True, 11, 0)
    g.set_lp_order(True, 11, 1)
    vf, ff, _, _ = f.debug_step()
    vg, fg, _, _ = g.debug_step()
    h, _ = _ctx(orca, w)
    vh, fh, _, _ = h.debug_step()
    feas = ((ff | fg | fh) & 0x7) == 0  # feasible, no g1/g2 event on any side
    assert np.array_equal(ff & 1, fh & 1) and np.array_equal(ff & 1, fg & 1)
    assert np.max(np.abs(vf[feas] - vh[feas])) < VTOL
    assert np.max(np.abs(vf[feas] - vg[feas])) < VTOL
    with pytest.raises(Exception):
        a.set_lp_order(True, 1, -1)
    with pytest.raises(Exception):
        a.set_lp_order(True, 1, 2 ** 31)
    for o in (a, b, c, d, e, f, g, h):
        o.close()


# ------------------------------------------------ work-unit LP2 (§8(f3))
@pytest.mark.parametrize("order", [0, 2])
@pytest.mark.parametrize("case", ["dense", "circle_crush", "k32"])
def test_lp_orders_vs_oracle(orca, oracle, case, order):
    """The greedy LP order (0, default: most violated half-plane next, in LP2 and LP3) and the
    sequential neighbour order (2, the oracle's) both reach the oracle's optimum within 1e-4 and
    its least penetration on the LP-heaviest inputs (reading Q8)."""
    if case == "dense":
        r = compare_step(orca, oracle, W.make("dense", n=4000), variant=0, order=order)
    elif case == "k32":
        r = compare_step(orca, oracle, W.make("uniform", n=3000, rho=0.5), variant=0, order=order, maxNeighbors=32)
    else:
        w = W.make("circle")
        op = oracle.make_params(**w["params"])
        pos, vel, _ = oracle.run(op, w["pos"], w["vel"], goals=w["goals"], pref_speed=1.0, steps=300)
        r = compare_step(orca, oracle, dict(w, pos=pos, vel=vel), variant=0, order=order)
    assert r["n_inf"] > 0


@pytest.mark.parametrize("case", ["dense", "circle_crush", "k32"])
def test_work_unit_lp_parity(orca, oracle, case):
    """Variant 3 (idle lanes evaluate other lanes' LP1 constraints) against the oracle on the
    LP-heaviest inputs: the dense crowd, the circle's central crush and k = 32 (segments of
    32 lanes, one problem per round)."""
    if case == "dense":
        compare_step(orca, oracle, W.make("dense", n=4000), variant=3, order=2)
    elif case == "k32":
        compare_step(orca, oracle, W.make("uniform", n=3000, rho=0.5), variant=3, order=2, maxNeighbors=32)
    else:
        w = W.make("circle")
        op = oracle.make_params(**w["params"])
        pos, vel, _ = oracle.run(op, w["pos"], w["vel"], goals=w["goals"], pref_speed=1.0, steps=300)
        compare_step(orca, oracle, dict(w, pos=pos, vel=vel), variant=3, order=2)


def test_work_unit_lp_bit_identical_k_sweep(orca):
    """Bit-identity of variant 3 with variant 0 (velocities, flags, work counters) over k,
    including k not a power of two and a ragged last warp."""
    w = W.make("uniform", n=4099, rho=0.6)
    for k in (1, 2, 3, 5, 9, 16, 17, 31, 32):
        a, _ = _ctx(orca, w, maxNeighbors=k)
        b, _ = _ctx(orca, w, maxNeighbors=k)
        a.set_variant(0)
        b.set_variant(3)
        for o in (a, b):  # the work-unit loop runs in the sequential orders
            o.set_lp_order(2)
        ra, rb = a.debug_step(), b.debug_step()
        for x, y in zip(ra, rb):
            assert np.array_equal(x, y), k
        assert a.work() == b.work(), k
        a.close()
        b.close()


# ------------------------------------------------ group LP3 kernel
@pytest.mark.parametrize("config,n,k", [("dense", 20000, 10), ("uniform", 6000, 32), ("uniform", 3001, 3)])
def test_lp3_lanes_bit_identical(orca, config, n, k):
    """The least-penetration kernel with 1 (thread), 4, 8 or 16 lanes per agent: the same
    velocities, flags, work counters, trajectories and statistics bit for bit (k = 32 runs
    LP1/projection chunks beyond one group width).  These sizes would run LP3 inside the step
    kernel, so the queued path is forced (orca_set_lp3_inline(0)) for the lane settings; the
    last context keeps the automatic (inline) choice, which must agree as well."""
    w = W.make(config, n=n) if config == "dense" else W.make(config, n=n, rho=0.6)
    ctxs = []
    for lanes in (1, 4, 8, 16, -1):  # -1: automatic
        o, _ = _ctx(orca, w, maxNeighbors=k)
        o.set_lp3_lanes(lanes)
        o.set_lp3_inline(0)
        assert o.launch_info()["lp3_lanes"] == (1 if lanes == -1 else lanes)
        ctxs.append(o)
    o, _ = _ctx(orca, w, maxNeighbors=k)
    li = o.launch_info()
    assert li["lp3_lanes"] == (1 if li["variant"] == 1 else 0)  # inline unless the group variant
    ctxs.append(o)
    r = [o.debug_step() for o in ctxs]
    assert np.count_nonzero(r[0][1] & 1) > 0
    wk = [o.work() for o in ctxs]
    for q in range(1, len(ctxs)):
        for x, y in zip(r[0], r[q]):
            assert np.array_equal(x, y), q
        assert wk[0] == wk[q], q
    for o in ctxs:
        o.step(20)
    s = [o.get_state() for o in ctxs]
    st = [o.stats() for o in ctxs]
    for q in range(1, len(ctxs)):
        assert np.array_equal(s[0][0], s[q][0]) and np.array_equal(s[0][1], s[q][1]), q
        assert st[0] == st[q], q
    with pytest.raises(Exception):
        ctxs[0].set_lp3_lanes(3)
    for o in ctxs:
        o.close()


@pytest.mark.parametrize("config,n,k,het", [("dense", 20000, 10, False), ("uniform", 30000, 32, True),
                                            ("uniform", 3001, 3, False), ("dense", 40000, 10, True)])
def test_lp3_modes_bit_identical(orca, config, n, k, het):
    """Where LP3 runs -- the k_lp3 kernel (0), per thread inside k_step (1), k_step's block-local
    compacted queue (2, several rounds when more than half a block is infeasible) -- changes
    nothing, for the thread-per-agent (0) and the lane-pair (4; k <= 14) kernels: dry-step velocities / flags / lists / work counters and 15 real steps (state and
    statistics) bit for bit, with heterogeneous agents and goals too."""
    w = W.make(config, n=n) if config == "dense" else W.make(config, n=n, rho=0.6)
    rng = np.random.default_rng(3)
    ctxs = []
    for mode, variant in ((0, 0), (1, 0), (2, 0), (0, 4), (2, 4)):
        o, _ = _ctx(orca, w, maxNeighbors=k)
        o.set_variant(variant)
        if het:
            props = _het_props(n, seed=21)
            o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
            o.set_goals((w["pos"] + rng.uniform(-30, 30, w["pos"].shape)).astype(np.float32), 1.0)
            rng = np.random.default_rng(3)
        o.set_lp3_inline(mode)
        assert o.launch_info()["lp3_lanes"] == (1 if mode == 0 else 0)
        ctxs.append(o)
    r = [o.debug_step() for o in ctxs]
    assert np.count_nonzero(r[0][1] & 1) > 0
    wk = [o.work() for o in ctxs]
    for q in range(1, len(ctxs)):
        for x, y in zip(r[0], r[q]):
            assert np.array_equal(x, y), q
        assert wk[0] == wk[q], q
    for o in ctxs:
        o.step(15)
    s = [o.get_state() for o in ctxs]
    st = [o.stats() for o in ctxs]
    for q in range(1, len(ctxs)):
        assert np.array_equal(s[0][0], s[q][0]) and np.array_equal(s[0][1], s[q][1]), q
        assert st[0] == st[q], q
    for o in ctxs:
        o.close()


@pytest.mark.parametrize("lanes", [4, 16])
def test_lp3_group_vs_oracle(orca, oracle, lanes):
    """The group LP3 kernels against the oracle on the dense crowd (many infeasible LPs)."""
    r = compare_step(orca, oracle, W.make("dense", n=4000), lp3_lanes=lanes)
    assert r["n_inf"] > 0


def test_graph_cache_across_set_agents(orca):
    """Cached step graphs survive orca_set_agents only while every captured argument is
    unchanged (graph_key): reloading the same layout reuses them, a new grid or capacity
    re-captures; either way the trajectory equals a fresh context's bit for bit."""
    w1 = W.make("uniform", n=20000, rho=0.25)
    w2 = W.make("uniform", n=30000, rho=0.4)
    a, p = _ctx(orca, w1)
    a.step(3)
    a.set_agents(w2["pos"], w2["vel"], w2["pref"])  # other grid and capacity
    a.step(3)
    b = orca.Orca(p)
    b.set_agents(w2["pos"], w2["vel"], w2["pref"])
    b.step(3)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    for _ in range(3):  # the e2e pattern: reload the same state, step, read back
        a.set_agents(w2["pos"], w2["vel"], w2["pref"])
        a.step(3)
        sa = a.get_state()
        assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    a.set_agents(w1["pos"], w1["vel"], w1["pref"])  # smaller input into the larger buffers
    a.step(3)
    c, _ = _ctx(orca, w1)
    c.step(3)
    sa, sc = a.get_state(), c.get_state()
    assert np.array_equal(sa[0], sc[0]) and np.array_equal(sa[1], sc[1])
    # same n, unrelated state: the kept search-radius hints are wrong, the result is exact
    w3 = W.make("uniform", n=20000, rho=0.6, salt=3)
    a.set_agents(w3["pos"], w3["vel"], w3["pref"])
    va, fa, na, ca = a.debug_step()
    a.step(3)
    d, _ = _ctx(orca, w3)
    vd, fd, nd, cd = d.debug_step()
    d.step(3)
    assert np.array_equal(na, nd) and np.array_equal(ca, cd) and np.array_equal(va, vd)
    sa, sd = a.get_state(), d.get_state()
    assert np.array_equal(sa[0], sd[0]) and np.array_equal(sa[1], sd[1])
    for o in (a, b, c, d):
        o.close()


# ------------------------------------------------ strip rebalance
def test_strips_rebalance_carries_state(orca):
    """orca_rebalance mid-run (heterogeneous agents, goals, removal at the goal, randomized LP
    order): the strips are re-partitioned and the trajectory stays bit-identical to one strip."""
    w = W.make("uniform", n=30000, rho=0.3)
    n = len(w["pos"])
    rng = np.random.default_rng(11)
    goals = (w["pos"] + rng.uniform(-60, 60, w["pos"].shape)).astype(np.float32)
    props = _het_props(n, seed=9)
    ctxs = []
    for strips in (0, 4):
        o = orca.Orca(w["params"], strips=strips)
        o.set_agents(w["pos"], w["vel"], w["pref"])
        o.set_goals(goals, 1.0)
        o.set_goal_removal(2.0)
        o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
        o.set_lp_order(True, 5, 0)
        ctxs.append(o)
    a, b = ctxs
    for o in ctxs:
        o.step(20)
    b.rebalance()
    assert b.stats()["rebalances"] >= 1
    for o in ctxs:
        o.step(30)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0], equal_nan=True) and np.array_equal(sa[1], sb[1], equal_nan=True)
    assert np.array_equal(a.active(), b.active()) and a.count() == b.count() < n
    ta, tb = a.stats(), b.stats()
    for key in ("infeasible", "degenerate", "collision_pairs", "removed"):
        assert ta[key] == tb[key], key
    for o in ctxs:
        o.close()


def test_strips_rebalance_convergent_crowd(orca):
    """A crowd converging on one point piles into the middle strips: the automatic rebalance
    re-partitions before any strip outgrows its buffers, and the run stays bit-identical to
    one strip (no overflow error)."""
    w = W.make("uniform", n=20000, rho=0.25)
    centre = w["pos"].mean(axis=0)
    goals = np.repeat(centre[None].astype(np.float32), len(w["pos"]), axis=0)
    a = orca.Orca(w["params"])
    b = orca.Orca(w["params"], strips=5)
    for o in (a, b):
        o.set_agents(w["pos"], w["vel"], w["pref"])
        o.set_goals(goals, 1.0)
    for _ in range(12):
        a.step(64)
        b.step(64)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    assert b.stats()["rebalances"] >= 1
    # the crowd really converged: most agents within 80 m of the centre
    assert np.mean(np.hypot(*(sa[0] - centre).T) < 80.0) > 0.8
    for o in (a, b):
        o.close()


def test_strips_transports_bit_identical(orca):
    """Loopback strips with the peer-memory exchange (k_push + arrival flags, default) and with
    whole-buffer device copies: identical trajectories, also across a switch mid-run."""
    w = W.make("uniform", n=30000, rho=0.35)
    a = orca.Orca(w["params"], strips=4)
    b = orca.Orca(w["params"], strips=4)
    b.set_transport(1)
    for o in (a, b):
        o.set_agents(w["pos"], w["vel"], w["pref"])
        o.step(40)
    a.set_transport(1)
    b.set_transport(0)
    for o in (a, b):
        o.step(30)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    c, _ = _ctx(orca, w)
    c.step(70)
    sc = c.get_state()
    assert np.array_equal(sa[0], sc[0]) and np.array_equal(sa[1], sc[1])
    for o in (a, b, c):
        o.close()


@pytest.mark.parametrize("offset", [(-3.0e4, 1.7e4), (6.5e4, -6.5e4)])
def test_far_from_origin(orca, oracle, offset):
    """A crowd tens of km from the origin (fp32 ulp of the coordinates ~ 4-8 mm, negative and
    positive): cells and neighbour lists stay bit-exact, velocities within the bar."""
    w = W.make("uniform", n=3000, rho=0.4)
    pos = (w["pos"].astype(np.float64) + np.array(offset)).astype(np.float32)
    compare_step(orca, oracle, dict(w, pos=pos))


def test_grid_capacity_and_recovery(orca):
    """A domain too large for the sort bins (two agents 10^7 m apart -> > 2^28 bins) is refused
    with ORCA_ERR_CAPACITY; the context stays usable with a valid crowd afterwards."""
    o = orca.Orca(W.DEFAULT_PARAMS)
    far = np.array([[0.0, 0.0], [1.0e7, 1.0e7]], np.float32)
    with pytest.raises(orca.OrcaError) as e:
        o.set_agents(far, np.zeros_like(far), np.zeros_like(far))
    assert e.value.status == 6
    w = W.make("uniform", n=500, rho=0.2)
    o.set_agents(w["pos"], w["vel"], w["pref"])
    o.step(3)
    assert o.count() == 500
    o.close()


@pytest.mark.parametrize("strips", [0, 3])
def test_expanding_crowd_regrids(orca, strips):
    """An open crowd spreads beyond the grid frozen at set_agents: when an agent reaches the
    outer cell ring the grid is re-derived (reading Q12), so the step stays fast, and the state
    steps exactly like a fresh context loaded with it (same neighbour lists and velocities)."""
    import time
    w = W.make("uniform", n=20000, rho=0.25)
    a = orca.Orca(w["params"], strips=strips)
    a.set_agents(w["pos"], w["vel"], w["pref"])
    a.step(64)
    a.count()
    t0 = time.perf_counter()
    a.step(64)
    a.count()
    early = time.perf_counter() - t0
    for _ in range(6):
        a.step(64)
    st = a.stats()
    assert st["regrids"] >= 1
    t0 = time.perf_counter()
    a.step(64)
    a.count()
    late = time.perf_counter() - t0
    assert late < 3.0 * early + 0.05, (early, late)
    pos, vel = a.get_state()
    origin, cs, dims = a.grid()
    assert np.all(pos >= origin.astype(np.float32)) and np.all(pos < origin + cs * dims)  # nobody clamped
    b = orca.Orca(w["params"])
    b.set_agents(pos, vel, w["pref"])
    va, fa, na, ca = a.debug_step()
    vb, fb, nb, cb = b.debug_step()
    assert np.array_equal(na, nb) and np.array_equal(ca, cb) and np.array_equal(va, vb)
    a.close()
    b.close()


def test_long_step_call_regrids_while_running(orca):
    """One orca_step(600) call on the spreading corridor re-derives the grid while it runs
    (the flag of chunk q-2 is read before chunk q is queued), and the trajectory equals stepping
    in short calls bit for bit (results never depend on the grid).  Agents that were clamped
    into the edge bins in between still find their exact neighbours (the search windows are
    clamped like the bins)."""
    import time
    w = W.make("corridor")
    a, b = orca.Orca(w["params"]), orca.Orca(w["params"])
    for o in (a, b):
        o.set_agents(w["pos"], w["vel"], w["pref"])
    a.count()
    t0 = time.perf_counter()
    a.step(600)
    a.count()
    long_call = time.perf_counter() - t0
    for _ in range(10):
        b.step(60)
    assert a.stats()["regrids"] >= 1  # (a re-derived grid keeps ~512 steps of walking as margin)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    assert long_call < 0.6, long_call  # ~0.05 ms per step; an unre-gridded run took ~0.3 ms
    a.close()
    b.close()


@pytest.mark.parametrize("strips", [0, 3])
def test_set_state_keeps_the_rest(orca, strips):
    """orca_set_state with the current state continues the run bit for bit (goals, removal,
    per-agent properties, randomized LP order, counters all kept); with another state it
    steps exactly like a fresh context configured the same way."""
    w = W.make("uniform", n=12000, rho=0.3)
    n = len(w["pos"])
    rng = np.random.default_rng(21)
    goals = (w["pos"] + rng.uniform(-40, 40, w["pos"].shape)).astype(np.float32)
    props = _het_props(n, seed=4)

    def make():
        o = orca.Orca(w["params"], strips=strips)
        o.set_agents(w["pos"], w["vel"], w["pref"])
        o.set_goals(goals, 1.0)
        o.set_goal_removal(1.5)
        o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
        o.set_lp_order(True, 9, 0)
        return o

    a, b = make(), make()
    a.step(30)
    b.step(30)
    pos, vel = b.get_state()
    b.set_state(pos, vel)  # removed agents read NaN: ignored
    a.step(20)
    b.step(20)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0], equal_nan=True) and np.array_equal(sa[1], sb[1], equal_nan=True)
    assert a.count() == b.count() < n
    ta, tb = a.stats(), b.stats()
    for key in ("infeasible", "collision_pairs", "removed"):
        assert ta[key] == tb[key], key
    # a present agent with NaN is refused
    bad = sb[0].copy()
    bad[np.nonzero(b.active())[0][0]] = np.nan
    with pytest.raises(orca.OrcaError):
        b.set_state(bad, sb[1])
    for o in (a, b):
        o.close()


def test_set_state_new_state_equals_fresh_context(orca):
    w = W.make("uniform", n=8000, rho=0.3)
    w2 = W.make("uniform", n=8000, rho=0.45, salt=2)
    a, p = _ctx(orca, w)
    a.step(5)
    a.set_state(w2["pos"], w2["vel"])  # the grid is re-derived if needed
    b = orca.Orca(p)
    b.set_agents(w2["pos"], w2["vel"], w["pref"])
    ra, rb = a.debug_step(), b.debug_step()
    for x, y in zip(ra, rb):
        assert np.array_equal(x, y)
    a.step(10)
    b.step(10)
    sa, sb = a.get_state(), b.get_state()
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])
    a.close()
    b.close()


def test_group_variant_heterogeneous_and_random_order(orca):
    """The 8-lane group kernel (variant 1, the automatic choice for small crowds) handles
    per-agent radii/speeds and the randomized LP order bit-identically to variant 0."""
    w = W.make("uniform", n=9000, rho=0.35)
    n = len(w["pos"])
    rng = np.random.default_rng(17)
    goals = (w["pos"] + rng.uniform(-50, 50, w["pos"].shape)).astype(np.float32)
    props = _het_props(n, seed=12)
    ctxs = []
    for v in (0, 1):
        o, _ = _ctx(orca, w)
        o.set_variant(v)
        o.set_goals(goals, 1.0)
        o.set_agent_props(props["radius"], props["maxSpeed"], props["prefSpeed"])
        o.set_lp_order(True, 77, 3)
        ctxs.append(o)
    r = [o.debug_step() for o in ctxs]
    assert np.array_equal(r[0][2], r[1][2]) and np.array_equal(r[0][3], r[1][3])
    assert np.array_equal(r[0][0], r[1][0]) and np.array_equal(r[0][1] & 1, r[1][1] & 1)
    for o in ctxs:
        o.step(25)
    s = [o.get_state() for o in ctxs]
    assert np.array_equal(s[0][0], s[1][0]) and np.array_equal(s[0][1], s[1][1])
    for o in ctxs:
        o.close()
