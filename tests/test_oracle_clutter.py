"""Pins for the oracle's Eq. 8 clutter fraction (reading G17: area inside the RICI
support cylinder, r <= R and |beta| <= R/2, by a Q x Q barycentric quadrature).

Against: closed-form areas of planes cut by the cylinder (pi R^2 for a plane through S_v
perpendicular to S_n, 2R x R for a plane containing the axis), exact cases of Eq. 8 (a lone
reference -> 0, a coincident duplicate -> 1/2, clutter outside the volume -> 0), and a
triangle fully inside the volume (area exact)."""
import numpy as np
import pytest

import synth


def _grid_plane(h, extent, axis="z"):
    """Finely triangulated square plane through the origin (normal along `axis`)."""
    k = int(round(2 * extent / h))
    u = np.linspace(-extent, extent, k + 1)
    U, V = np.meshgrid(u, u, indexing="ij")
    Z = np.zeros_like(U)
    P = np.stack([U, V, Z], -1) if axis == "z" else np.stack([U, Z, V], -1)
    verts = P.reshape(-1, 3).astype(np.float32)
    i, j = np.meshgrid(np.arange(k), np.arange(k), indexing="ij")
    a = (i * (k + 1) + j).ravel()
    b, c, d = a + (k + 1), a + (k + 2), a + 1
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)]).astype(np.int32)
    return verts, tris


ORIGIN = np.array([[0, 0, 0, 0, 0, 1]], np.float32)


@pytest.mark.parametrize("axis,expect", [("z", np.pi * 0.3 ** 2), ("y", 2 * 0.3 * 0.3)])
def test_plane_areas_converge_to_closed_forms(oracle_mod, axis, expect):
    R = 0.3
    errs = []
    for h in (0.04, 0.02, 0.01):
        v, t = _grid_plane(h, 0.5, axis)
        frac, aa, ao = oracle_mod.clutter_fraction(v, t, np.ones(len(t), np.uint8), ORIGIN, R, q=4)
        assert frac[0] == 0.0 and aa[0] == ao[0]
        errs.append(abs(aa[0] - expect) / expect)
    assert errs[-1] < 0.01 and errs[-1] <= errs[0] + 1e-6      # converges (exact when grid-aligned)


def test_exact_cases(oracle_mod):
    m = synth.bumpy_torus(40, 20, key=(3,))
    o = m.origins[::17]
    tag1 = np.ones(m.n_triangles, np.uint8)
    frac, aa, _ = oracle_mod.clutter_fraction(m.vertices, m.indices, tag1, o, 0.3)
    assert (frac == 0).all() and (aa > 0).all()
    # a coincident duplicate of the object: exactly half of the area is clutter
    V = np.concatenate([m.vertices, m.vertices])
    T = np.concatenate([m.indices, m.indices + m.n_vertices])
    tag = np.concatenate([tag1, np.zeros(m.n_triangles, np.uint8)])
    frac, _, _ = oracle_mod.clutter_fraction(V, T, tag, o, 0.3)
    assert np.allclose(frac, 0.5, rtol=0, atol=1e-12)
    # clutter far outside the support volume changes nothing
    V2 = np.concatenate([m.vertices, m.vertices + np.float32(10)])
    frac, _, _ = oracle_mod.clutter_fraction(V2, T, tag, o, 0.3)
    assert (frac == 0).all()


def test_triangle_inside_counts_its_area(oracle_mod):
    V = np.array([[0.01, 0.0, 0.02], [0.05, 0.01, -0.03], [0.02, 0.06, 0.01]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    area = 0.5 * np.linalg.norm(np.cross(V[1].astype(float) - V[0], V[2].astype(float) - V[0]))
    _, aa, _ = oracle_mod.clutter_fraction(V, T, np.ones(1, np.uint8), ORIGIN, 0.3, q=5)
    assert aa[0] == pytest.approx(area, rel=1e-12)


def _quad_bound(R, d):
    """Area within distance d of a quarter circle of radius R (the band where a sub-triangle of
    diameter d can straddle the wall and be mis-assigned by a centroid quadrature)."""
    return 0.5 * np.pi * ((R + d) ** 2 - max(R - d, 0.0) ** 2) / 2


def test_wall_crossing_triangle_converges_to_exact_clip(oracle_mod):
    """A triangle that crosses the cylinder WALL (r = R): right triangle with legs 0.5 at the
    axis, in the plane beta = 0.05.  Its hypotenuse is 0.354 > R from the axis, so the exact
    clipped area is the quarter disk pi R^2 / 4.  The Q x Q centroid quadrature (G17) may only
    misplace sub-triangles that straddle the wall: |error| <= the area of the band of width d
    (the sub-triangle diameter) around the quarter circle, and the error shrinks with Q."""
    R = 0.3
    V = np.array([[0.0, 0.0, 0.05], [0.5, 0.0, 0.05], [0.0, 0.5, 0.05]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    exact = np.pi * R * R / 4
    errs = []
    for q in (8, 16, 32, 64):
        _, aa, _ = oracle_mod.clutter_fraction(V, T, np.ones(1, np.uint8), ORIGIN, R, q=q)
        d = 0.5 * np.sqrt(2) / q                     # sub-triangle diameter
        err = abs(aa[0] - exact)
        assert err <= _quad_bound(R, d), (q, aa[0], exact)
        errs.append(err)
    assert errs[-1] < 0.02 * exact and errs[-1] < errs[0]


def test_slab_crossing_triangle_converges_to_exact_clip(oracle_mod):
    """A triangle inside r <= R that crosses the SLAB walls |beta| = R/2: vertices
    (0.1, -0.1, -0.3), (0.1, 0.1, -0.3), (0.1, 0, 0.3); its width at height z is
    0.2 (0.3 - z) / 0.6, so the area with |z| <= 0.15 is (1/3) * integral (0.3 - z) dz = 0.03."""
    R = 0.3
    V = np.array([[0.1, -0.1, -0.3], [0.1, 0.1, -0.3], [0.1, 0.0, 0.3]], np.float32)
    T = np.array([[0, 1, 2]], np.int32)
    exact = 0.03
    errs = []
    for q in (5, 9, 17, 33, 65):                     # not multiples of 4: the slab walls cut sub-triangles
        _, aa, _ = oracle_mod.clutter_fraction(V, T, np.ones(1, np.uint8), ORIGIN, R, q=q)
        h = 0.6 / q                                  # sub-triangle height along z
        band = 2 * 0.2 * 2 * h                       # two walls, width <= 0.2, band +-h each
        err = abs(aa[0] - exact)
        assert err <= band, (q, aa[0], exact)
        errs.append(err)
    assert errs[0] > 1e-4 and errs[-1] < 0.02 * exact and errs[-1] < errs[0]
