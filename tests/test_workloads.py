"""Seeded input recipes: non-overlapping starts, densities, goals."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1908_10107_b200 import workloads as W


def _min_sep(pos):
    from scipy.spatial import cKDTree
    d, _ = cKDTree(pos.astype(np.float64)).query(pos.astype(np.float64), k=2)
    return d[:, 1].min()


@pytest.mark.parametrize("cfg,kw", [("uniform", dict(n=20000, rho=0.5)), ("corridor", {}), ("dense", dict(n=20000)),
                                    ("two_way", {}), ("eight_way", {}), ("uniform", dict(n=5000, rho=0.01))])
def test_no_initial_overlap(cfg, kw):
    w = W.make(cfg, **kw)
    assert w["pos"].dtype == np.float32 and w["pos"].shape[1] == 2
    assert _min_sep(w["pos"]) >= 2 * W.DEFAULT_PARAMS["radius"]


def test_deterministic():
    a = W.make("uniform", n=1000)
    b = W.make("uniform", n=1000)
    assert np.array_equal(a["pos"], b["pos"]) and np.array_equal(a["pref"], b["pref"])
    c = W.make("uniform", n=1000, salt=1)
    assert not np.array_equal(a["pos"], c["pos"])


def test_uniform_density_and_headings():
    w = W.make("uniform", n=40000, rho=0.25)
    ext = w["pos"].max(0) - w["pos"].min(0)
    assert abs(40000 / (ext[0] * ext[1]) - 0.25) < 0.02
    sp = np.hypot(*w["pref"].T)
    assert np.allclose(sp, W.DESIRED_SPEED, atol=1e-6)


def test_two_way_goals_swap_regions():
    """each group's start region is the other's goal region."""
    w = W.make("two_way")
    p, g = w["pos"], w["goals"]
    mid = 0.5 * (p[:, 0].min() + p[:, 0].max())
    left = p[:, 0] < mid
    assert abs(left.mean() - 0.5) < 0.01
    assert np.all(g[left, 0] > mid) and np.all(g[~left, 0] < mid)
    # goal set of the left group lies inside the right group's start region (bounding box)
    rb = p[~left].min(0), p[~left].max(0)
    assert np.all(g[left] >= rb[0] - 2.0) and np.all(g[left] <= rb[1] + 2.0)


def test_eight_way_turn():
    """goals are the start regions turned by 135 degrees about the centre."""
    w = W.eight_way(n=8000, turn_deg=135.0)
    p, g = w["pos"].astype(np.float64), w["goals"].astype(np.float64)
    ap = np.arctan2(p[:, 1], p[:, 0])
    ag = np.arctan2(g[:, 1], g[:, 0])
    d = np.angle(np.exp(1j * (ag - ap)), deg=True)
    assert np.allclose(d, 135.0, atol=1e-3)
    assert np.allclose(np.hypot(*p.T), np.hypot(*g.T), rtol=1e-5)
