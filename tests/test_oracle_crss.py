"""Pins for the oracle's CRSS distance (Eq. 7, Listing 1) and ranks.

Against: the hand-evaluated Listing 1 example (golden fixture), algebraic
identities of Eq. 7 (self distance 0, all-zero needle 0, invariance to per-row
constant offsets of the haystack, the clutter-ignoring property), an expanded
form sum M*Dn^2 - 2 sum M*Dn*Dh + sum M*Dh^2 evaluated with numpy matrix
algebra, and ranks against a sort-based brute force.
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    d = {}
    with open(os.path.join(GOLDEN, "crss_listing1_example.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                d[k] = [int(x) for x in v]
    return d


def test_listing1_hand_example(oracle_mod):
    g = _golden()
    n = np.array(g["needle"], np.uint16).reshape(3, 3)
    h = np.array(g["haystack"], np.uint16).reshape(3, 3)
    assert oracle_mod.crss(n, h) == g["crss"][0]
    assert oracle_mod.crss(h, n) == g["crss_reversed"][0]     # asymmetric


def _rand_imgs(rng, k, N=64, hi=12, density=0.3):
    a = rng.integers(0, hi, (k, N, N))
    a[rng.random((k, N, N)) > density] = 0
    return a.astype(np.uint16)


def test_identities(oracle_mod):
    rng = np.random.default_rng(0)
    A = _rand_imgs(rng, 6)
    for x in A:
        assert oracle_mod.crss(x, x) == 0
        assert oracle_mod.crss(np.zeros_like(x), x) == 0
        off = rng.integers(0, 50, (64, 1)).astype(np.uint16)
        for y in A:
            assert oracle_mod.crss(x, y) == oracle_mod.crss(x, y + off)   # per-row constant


def test_clutter_ignoring_property(oracle_mod):
    """Editing the haystack only where the needle is flat on both sides of a pixel
    leaves CRSS unchanged (SPEC 'clutter-ignoring property')."""
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = _rand_imgs(rng, 1, density=0.05)[0].astype(np.int64)
        h = _rand_imgs(rng, 1)[0].astype(np.int64)
        d = np.zeros_like(n)
        d[:, 1:] = n[:, 1:] - n[:, :-1]
        flat = np.zeros_like(n, bool)
        flat[:, :-1] = (d[:, :-1] == 0) & (d[:, 1:] == 0)
        flat[:, -1] = d[:, -1] == 0
        h2 = h.copy()
        h2[flat] += rng.integers(0, 30, flat.sum())
        assert oracle_mod.crss(n.astype(np.uint16), h.astype(np.uint16)) == \
            oracle_mod.crss(n.astype(np.uint16), h2.astype(np.uint16))


def test_expanded_form_matrix(oracle_mod):
    rng = np.random.default_rng(2)
    A = _rand_imgs(rng, 20, hi=300, density=0.4)
    B = _rand_imgs(rng, 30, hi=300, density=0.6)
    D = oracle_mod.crss_matrix(A, B)
    da = np.diff(A.astype(np.int64), axis=2).reshape(20, -1)
    db = np.diff(B.astype(np.int64), axis=2).reshape(30, -1)
    M = (da != 0).astype(np.int64)
    want = (M * da * da).sum(1)[:, None] - 2 * (da @ db.T) + M @ (db * db).T
    assert np.array_equal(D.astype(np.int64), want)


def test_large_values_exact(oracle_mod):
    """uint16 extremes: per-term squares reach (2*65535)^2 > 2^32 (G9)."""
    n = np.zeros((64, 64), np.uint16)
    h = np.zeros((64, 64), np.uint16)
    n[:, 1::2] = 65535
    h[:, 0::2] = 65535
    got = oracle_mod.crss(n, h)
    # every column c>=1 has needle delta +-65535 and haystack delta -+65535
    assert got == 64 * 63 * (2 * 65535) ** 2


def test_rank_tie_example(oracle_mod):
    """S:441's distances [5,2,2,9] with a correspondent at distance 2.  Under the paper's
    best-tie rule ("we use the highest (best) rank") and 0-based ranks (P:388,
    0 <= rank <= |CD|-1) nothing is strictly closer, so the rank is 0; S:441 prints 1,
    which contradicts its own post-condition S:440 (a SPEC defect, G10).
    Replacing the tied 2 by a 3 gives rank 1."""
    N = 4
    needle = np.zeros((N, N), np.uint16)
    needle[0, 1:] = 1                     # needle deltas: +1 at (0,1) and (1,1) only
    needle[1, 1:] = 1
    # CRSS = (1 - hd0)^2 + (1 - hd1)^2 with hd_r = h[r,1] - h[r,0]
    # hd pairs (0,-1) -> 5, (0,0) -> 2, (0,0) -> 2, (-2,1) -> 9
    rows = [((0, 0), (1, 0)), ((0, 0), (0, 0)), ((0, 0), (0, 0)), ((2, 0), (0, 1))]
    hay = np.zeros((4, N, N), np.uint16)
    for j, (r0, r1) in enumerate(rows):
        hay[j, 0, :2] = r0
        hay[j, 1, :2] = r1
    assert list(oracle_mod.crss_matrix(needle, hay)[0]) == [5, 2, 2, 9]
    thr = np.array([oracle_mod.crss(needle, hay[2])], np.uint64)   # correspondent = 2
    assert oracle_mod.count_below(needle[None], hay, thr)[0] == 0
    hay[2, 0, :2] = (1, 0)                 # hd0 = -1 -> (1+1)^2 = 4
    hay[2, 1, :2] = (0, 1)                 # hd1 = +1 -> (1-1)^2 = 0; total 4
    d = list(oracle_mod.crss_matrix(needle, hay)[0])
    assert d == [5, 2, 4, 9]
    thr = np.array([d[2]], np.uint64)
    assert oracle_mod.count_below(needle[None], hay, thr)[0] == 1


def test_ranks_vs_sort(oracle_mod):
    rng = np.random.default_rng(4)
    A = _rand_imgs(rng, 25, N=16, hi=4, density=0.3)
    H = np.concatenate([A, _rand_imgs(rng, 15, N=16, hi=4, density=0.3)])
    H[3] = H[7]                                       # duplicate -> ties
    r = oracle_mod.ranks(A, H)
    D = oracle_mod.crss_matrix(A, H)
    for i in range(A.shape[0]):
        s = np.sort(D[i])
        assert r[i] == np.searchsorted(s, D[i, i], side="left")
