"""Pins for the oracle's per-layer circle/triangle intersection (steps 1-6).

Against: the hand-worked SPEC S:235 example, and an independent segment/circle
quadratic (|E0 + t (E1-E0)|^2 = rho^2, t in [0,1]) that counts crossings of a
circle with the slice segment directly.
"""
import numpy as np
import pytest


def test_spec_example_beta0(oracle_mod):
    s = oracle_mod.segment([1, -2, -1], [1, -2, 2], [1, 2, -1], 0.0)
    assert np.allclose(s["E0"], [1, -2])
    assert np.allclose(s["E1"], [1, 2 / 3])
    assert s["rc"] == pytest.approx(1.0)
    assert s["rmin"] == pytest.approx(np.sqrt(13) / 3)
    assert s["rmax"] == pytest.approx(np.sqrt(5))


def test_outside_extent_and_half_open(oracle_mod):
    tri = ([0, 0, 0], [1, 0, 1], [0, 1, 2])
    assert oracle_mod.segment(*tri, -0.1) is None
    assert oracle_mod.segment(*tri, 2.0) is None          # beta == z_max excluded (G5)
    assert oracle_mod.segment(*tri, 0.0) is None          # beta == z_min: a single point, zero length
    assert oracle_mod.segment(*tri, 1.0) is not None      # beta == z_mid: uses edge (b,c)
    flat = ([0, 0, 1], [1, 0, 1], [0, 1, 1])
    assert oracle_mod.segment(*flat, 1.0) is None          # coplanar triangle (G6)


def _quadratic_count(e0, e1, rho):
    d = e1 - e0
    a = d @ d
    b = 2 * e0 @ d
    c = e0 @ e0 - rho * rho
    disc = b * b - 4 * a * c
    if disc < 0:
        return 0
    sq = np.sqrt(disc)
    ts = [(-b - sq) / (2 * a), (-b + sq) / (2 * a)]
    return sum(1 for t in ts if 0 <= t <= 1)


def test_ranges_match_quadratic(oracle_mod):
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(3000):
        tri = rng.uniform(-1, 1, (3, 3))
        beta = rng.uniform(-1, 1)
        s = oracle_mod.segment(tri[0], tri[1], tri[2], beta)
        if s is None:
            continue
        e0, e1 = np.asarray(s["E0"]), np.asarray(s["E1"])
        for rho in rng.uniform(0, 1.5, 8):
            want = _quadratic_count(e0, e1, rho)
            got = 0
            if s["rc"] is not None and s["rc"] <= rho < s["rmin"]:
                got = 2
            elif s["rmin"] <= rho < s["rmax"]:
                got = 1
            # skip exact ties (measure zero)
            if min(abs(rho - s["rmin"]), abs(rho - s["rmax"]), abs(rho - (s["rc"] or -9))) < 1e-9:
                continue
            assert got == want
            checked += 1
    assert checked > 1000
