"""Seeded synthetic inputs for the RICI hot path (shared by the oracle tests and the CUDA path).

This module holds NONE of the method's arithmetic: it only builds triangle
meshes, vertex normals and oriented points shaped like the paper's workloads
(P:379-387 clutterbox protocol, P:423-425 settings).  Every random choice is
derived from one master seed ("a single random seed determines all randomly
chosen parameters").  The recipe is stated in DESIGN.md "Input recipe".

Configs:
  C1 tiny     : icosphere level 1 (V=42, T=80), origins at every vertex, R=1.0, N=64
  C2 object   : bumpy torus 264x132 (V=34,848, T=69,696), R=0.3, N=64
  C3 scene    : 10 bumpy tori 316x158 in a clutterbox of side 3 (V=499,280, T=998,560)
  C4 search   : reference torus 448x224 (needles) + 9 clutter objects (haystack V=1,003,520)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MASTER_SEED = 42


@dataclass
class Mesh:
    vertices: np.ndarray          # [V,3] float32
    indices: np.ndarray           # [T,3] int32
    normals: np.ndarray           # [V,3] float32, unit
    object_id: np.ndarray = field(default=None)  # [V] int32 (clutterbox scenes)

    @property
    def origins(self) -> np.ndarray:
        """Oriented points (S_v, S_n) at every vertex: [V,6] float32 (px,py,pz,nx,ny,nz)."""
        return np.ascontiguousarray(np.concatenate([self.vertices, self.normals], axis=1), dtype=np.float32)

    @property
    def n_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def n_triangles(self) -> int:
        return int(self.indices.shape[0])


def rng_for(*key: int) -> np.random.Generator:
    """Independent stream per (config, scene, object, ...) key under the master seed."""
    return np.random.default_rng([MASTER_SEED, *[int(k) for k in key]])


# --------------------------------------------------------------------------- meshes
def vertex_normals(vertices: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """Area-weighted vertex normals (sum of un-normalised face normals)."""
    v = vertices.astype(np.float64)
    t = indices.astype(np.int64)
    fn = np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]])
    acc = np.zeros_like(v)
    for k in range(3):
        np.add.at(acc, t[:, k], fn)
    ln = np.linalg.norm(acc, axis=1, keepdims=True)
    ln[ln == 0] = 1.0
    return (acc / ln).astype(np.float32)


def icosphere(level: int = 1) -> Mesh:
    """Golden-ratio icosahedron, ``level`` midpoint subdivisions, projected to the unit sphere.
    Normals are radial (exact for the sphere)."""
    p = (1.0 + 5.0 ** 0.5) / 2.0
    verts = [(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0),
             (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
             (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
             (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
             (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
             (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    v = [np.array(x, dtype=np.float64) / np.linalg.norm(x) for x in verts]
    for _ in range(level):
        cache: dict = {}
        nf = []

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = v[a] + v[b]
                v.append(m / np.linalg.norm(m))
                cache[key] = len(v) - 1
            return cache[key]
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    V = np.array(v, dtype=np.float64).astype(np.float32)
    n = V.astype(np.float64)
    n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    return Mesh(V, np.array(faces, dtype=np.int32), n)


def normalise_unit_sphere(v: np.ndarray) -> np.ndarray:
    """Scale and translate so the object fits inside the unit sphere:
    centre = bounding-box centre, radius = max distance from it."""
    v = v.astype(np.float64)
    c = 0.5 * (v.min(0) + v.max(0))
    r = np.linalg.norm(v - c, axis=1).max()
    return (v - c) / r


def bumpy_torus(nu: int, nv: int, key: tuple = (0,), minor: float = 0.35,
                amp: float = 0.06, n_terms: int = 12, normalise: bool = True) -> Mesh:
    """Closed (watertight) torus grid nu x nv with a seeded radial displacement
    d(u,v) = sum_k amp * w_k * sin(a_k u + phi_k) * cos(b_k v + psi_k) / 3,
    a_k in 1..8, b_k in 1..6 (integers keep it periodic), w_k ~ U[0,1).
    V = nu*nv, T = 2*nu*nv.  Area-weighted vertex normals."""
    rng = rng_for(*key)
    a = rng.integers(1, 9, n_terms)
    b = rng.integers(1, 7, n_terms)
    w = rng.random(n_terms)
    phi = rng.random(n_terms) * 2 * np.pi
    psi = rng.random(n_terms) * 2 * np.pi
    u = np.arange(nu) * (2 * np.pi / nu)
    vv = np.arange(nv) * (2 * np.pi / nv)
    U, W = np.meshgrid(u, vv, indexing="ij")
    d = np.zeros_like(U)
    for k in range(n_terms):
        d += amp * w[k] * np.sin(a[k] * U + phi[k]) * np.cos(b[k] * W + psi[k]) / 3.0
    r = minor + d
    X = (1.0 + r * np.cos(W)) * np.cos(U)
    Y = (1.0 + r * np.cos(W)) * np.sin(U)
    Z = r * np.sin(W)
    verts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
    i = np.arange(nu)[:, None]
    j = np.arange(nv)[None, :]
    i1 = (i + 1) % nu
    j1 = (j + 1) % nv
    q00 = (i * nv + j).ravel()
    q10 = (i1 * nv + j).ravel()
    q11 = (i1 * nv + j1).ravel()
    q01 = (i * nv + j1).ravel()
    tris = np.concatenate([np.stack([q00, q10, q11], 1), np.stack([q00, q11, q01], 1)], 0)
    if normalise:
        verts = normalise_unit_sphere(verts)
    V = verts.astype(np.float32)
    T = tris.astype(np.int32)
    n = vertex_normals(V, T)
    # orient outward: normals should point away from the tube centre line
    vc = V.astype(np.float64) - V.astype(np.float64).mean(0)
    ang = np.arctan2(vc[:, 1], vc[:, 0])
    ring = np.stack([np.cos(ang), np.sin(ang), np.zeros_like(ang)], 1) * np.linalg.norm(vc[:, :2], axis=1).mean()
    if np.sum(np.einsum("ij,ij->i", n.astype(np.float64), vc - ring)) < 0:
        T = T[:, ::-1].copy()
        n = -n
    return Mesh(V, np.ascontiguousarray(T), n)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation from a uniform unit quaternion (G15)."""
    u1, u2, u3 = rng.random(3)
    q = np.array([np.sqrt(1 - u1) * np.sin(2 * np.pi * u2), np.sqrt(1 - u1) * np.cos(2 * np.pi * u2),
                  np.sqrt(u1) * np.sin(2 * np.pi * u3), np.sqrt(u1) * np.cos(2 * np.pi * u3)])
    x, y, z, w = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def clutterbox(objects: list[Mesh], key: tuple, box_side: float = 3.0) -> Mesh:
    """Clutterbox scene: each unit-sphere object gets a uniform random
    orientation and a centre uniform in [1, s-1]^3 so its bounding sphere fits in
    the box.  Object 0 (the reference) is placed first, so scene vertex i is
    reference vertex i for i < V_ref (G11)."""
    rng = rng_for(*key)
    vs, ts, ns, ids = [], [], [], []
    off = 0
    for k, m in enumerate(objects):
        Rm = random_rotation(rng)
        c = rng.uniform(1.0, box_side - 1.0, 3)
        v = m.vertices.astype(np.float64) @ Rm.T + c
        n = m.normals.astype(np.float64) @ Rm.T
        vs.append(v.astype(np.float32))
        ns.append((n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32))
        ts.append(m.indices + off)
        ids.append(np.full(m.n_vertices, k, dtype=np.int32))
        off += m.n_vertices
    return Mesh(np.concatenate(vs), np.concatenate(ts).astype(np.int32), np.concatenate(ns),
                np.concatenate(ids))


def place(m: Mesh, rotation: np.ndarray, translation) -> Mesh:
    """Rigidly move a mesh (vertices and normals)."""
    v = m.vertices.astype(np.float64) @ rotation.T + np.asarray(translation, dtype=np.float64)
    n = m.normals.astype(np.float64) @ rotation.T
    return Mesh(v.astype(np.float32), m.indices.copy(), n.astype(np.float32), m.object_id)


# --------------------------------------------------------------------------- hand-case meshes
def cube(half: float = 1.0) -> Mesh:
    """Axis-aligned cube [-h,h]^3, 12 triangles, outward winding; normals at the
    corners point along the body diagonal."""
    h = half
    V = np.array([[x, y, z] for x in (-h, h) for y in (-h, h) for z in (-h, h)], dtype=np.float32)
    # vertex index = 4*ix + 2*iy + iz
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    T = []
    for a, b, c, d in quads:
        T += [(a, b, c), (a, c, d)]
    n = V.astype(np.float64)
    n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    return Mesh(V, np.array(T, dtype=np.int32), n)


def tetrahedron() -> Mesh:
    """Regular tetrahedron (1,1,1),(1,-1,-1),(-1,1,-1),(-1,-1,1); radial normals."""
    V = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=np.float32)
    T = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]], dtype=np.int32)
    n = V.astype(np.float64)
    n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    return Mesh(V, T, n)


def quad(corners) -> Mesh:
    """Two-triangle quad from 4 corners (in order)."""
    V = np.array(corners, dtype=np.float32)
    T = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int32)
    return Mesh(V, T, vertex_normals(V, T))


def triangle_soup(n_tri: int, key: tuple, extent: float = 1.0, grid: float | None = None) -> Mesh:
    """Random triangles in [-extent, extent]^3; with ``grid`` the coordinates are
    snapped to multiples of ``grid`` (adversarial, tie-prone)."""
    rng = rng_for(*key)
    V = rng.uniform(-extent, extent, (3 * n_tri, 3))
    if grid:
        V = np.round(V / grid) * grid
    V = V.astype(np.float32)
    T = np.arange(3 * n_tri, dtype=np.int32).reshape(-1, 3)
    return Mesh(V, T, vertex_normals(V, T))


def random_origins(n: int, key: tuple, extent: float = 0.5) -> np.ndarray:
    """Random oriented points: positions in [-extent,extent]^3, unit normals."""
    rng = rng_for(*key)
    p = rng.uniform(-extent, extent, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([p, d], 1).astype(np.float32)


# --------------------------------------------------------------------------- configs
def config_c1() -> dict:
    m = icosphere(1)
    return {"name": "C1", "mesh": m, "origins": m.origins, "R": 1.0, "N": 64}


def config_c2() -> dict:
    m = bumpy_torus(264, 132, key=(2, 0, 0))
    return {"name": "C2", "mesh": m, "origins": m.origins, "R": 0.3, "N": 64}


def _scene_objects(n_obj: int, nu: int, nv: int, key: tuple) -> list[Mesh]:
    objs = []
    for k in range(n_obj):
        rng = rng_for(*key, k, 99)
        objs.append(bumpy_torus(nu, nv, key=(*key, k), minor=float(rng.uniform(0.2, 0.45)), amp=0.08))
    return objs


def config_c3(n_obj: int = 10, nu: int = 316, nv: int = 158, scene: int = 0) -> dict:
    objs = _scene_objects(n_obj, nu, nv, (3, scene))
    sc = clutterbox(objs, key=(3, scene, 1000))
    return {"name": "C3", "mesh": sc, "origins": sc.origins, "R": 0.3, "N": 64}


def config_c4(n_clutter: int = 9, nu: int = 448, nv: int = 224, scene: int = 0) -> dict:
    """Needles = reference object alone; haystack = scene with the reference placed first."""
    objs = _scene_objects(1 + n_clutter, nu, nv, (4, scene))
    sc = clutterbox(objs, key=(4, scene, 1000))
    ref = Mesh(sc.vertices[: objs[0].n_vertices].copy(), objs[0].indices.copy(),
               sc.normals[: objs[0].n_vertices].copy())
    return {"name": "C4", "reference": ref, "scene": sc, "R": 0.3, "N": 64}
