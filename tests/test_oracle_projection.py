"""Pins for the oracle's spin frame and projection (Eqs. 1-5).

Pinned against things other than the oracle itself: the SPEC's hand examples
(S:159-161), the isometry alpha^2+beta^2 = |P-S_v|^2, beta = (P-S_v).n
(the closed-form meaning of the spin frame), and an independent orthonormal
frame built from cross products (the "direct approach" of fig:directRotation,
P:154), which gives the same (alpha, beta) for any frame rotated about S_n.
"""
import numpy as np
import pytest


def test_frame_examples(oracle_mod):
    # S:159-161
    f, ok = oracle_mod.spin_frame([0, 0, 1])
    assert ok and np.allclose(f, [1, 0, 0, 1])            # identity rotations
    f, ok = oracle_mod.spin_frame([1, 0, 0])
    assert np.allclose(f, [1, 0, 1, 0])
    f, ok = oracle_mod.spin_frame(np.array([1, 1, 1]) / np.sqrt(3))
    assert np.allclose(f, [1 / np.sqrt(2), 1 / np.sqrt(2), np.sqrt(2 / 3), 1 / np.sqrt(3)])


def test_zero_normal_is_invalid(oracle_mod):
    _, ok = oracle_mod.spin_frame([0, 0, 0])
    assert not ok


@pytest.mark.parametrize("origin,point,expect", [
    ([0, 0, 0, 0, 0, 1], [3, 4, 5], (5, 5)),
    ([1, 1, 1, 0, 0, 1], [1, 1, 4], (0, 3)),
    ([0, 0, 0, 1, 0, 0], [2, 3, 0], (3, 2)),
    ([0, 0, 0, 0, 0, -1], [3, 4, 5], (5, -5)),   # G2: n = -z flips beta
])
def test_projection_examples(oracle_mod, origin, point, expect):
    a, b = oracle_mod.project(origin, point)
    assert a == pytest.approx(expect[0], abs=1e-12)
    assert b == pytest.approx(expect[1], abs=1e-12)


def _direct(origin, p):
    """fig:directRotation-style frame: e3 = n, e1 from a cross product, e2 = e3 x e1."""
    s, n = np.asarray(origin[:3], float), np.asarray(origin[3:], float)
    n = n / np.linalg.norm(n)
    helper = np.array([0.0, 0.0, 1.0]) if abs(n[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
    e1 = np.cross(helper, n)
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(n, e1)
    d = np.asarray(p, float) - s
    return np.hypot(d @ e1, d @ e2), d @ n


def test_projection_matches_direct_frame_random(oracle_mod):
    rng = np.random.default_rng(1)
    normals = rng.normal(size=(400, 3))
    # the identity-rotation branches (S_nx=S_ny=0 and S_ny=S_nz=0)
    normals[:10] = [0, 0, 1]
    normals[10:20] = [0, 0, -1]
    normals[20:30] = [1, 0, 0]
    normals[30:40] = [-1, 0, 0]
    normals[40:50] = [0, -1, 0]
    for k in range(normals.shape[0]):
        origin = np.concatenate([rng.uniform(-2, 2, 3), normals[k]])
        p = rng.uniform(-3, 3, 3)
        a, b = oracle_mod.project(origin, p)
        ea, eb = _direct(origin, p)
        assert a == pytest.approx(ea, abs=1e-12)
        assert b == pytest.approx(eb, abs=1e-12)
        # isometry (rotations preserve distance): alpha^2 + beta^2 = |P - S_v|^2
        assert a * a + b * b == pytest.approx(np.sum((p - origin[:3]) ** 2), rel=1e-12)


def test_printed_eq1_is_not_what_the_rotations_need():
    """G1: Eq. 1 as printed (N_b = Normalize[S_nx, S_nz]) fails to map S_n onto +z
    for n = (0,1,0); the corrected N_b (x after the first rotation) succeeds."""
    n = np.array([0.0, 1.0, 0.0])
    nax, nay = n[0] / np.hypot(n[0], n[1]), n[1] / np.hypot(n[0], n[1])
    qx = nax * n[0] + nay * n[1]

    def tz(nbx, nbz):
        return nbx * qx + nbz * n[2]
    lit = np.array([n[0], n[2]])
    lit = lit / np.linalg.norm(lit) if np.linalg.norm(lit) > 0 else np.array([0.0, 1.0])
    cor = np.array([qx, n[2]]) / np.hypot(qx, n[2])
    assert abs(tz(*lit) - 1.0) > 0.5          # printed reading: n does not land on +z
    assert tz(*cor) == pytest.approx(1.0)     # corrected reading
