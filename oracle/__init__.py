"""CPU oracle for the RICI hot path (arXiv 2007.02306) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2007_02306_b200`` never imports it and shares no code with it.

The arithmetic lives in ``rici_oracle.c`` (plain double-precision loops that
follow the paper step by step, each function citing its passage).  This file
only compiles that C file with gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rici_oracle.c")
_LIB_PATH = os.path.join(_HERE, "librici_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c99",
                               "-fvisibility=hidden", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_spin_frame.argtypes = [P, P]
        lib.oracle_spin_frame.restype = ctypes.c_int
        lib.oracle_project.argtypes = [P, P, P]
        lib.oracle_project.restype = None
        lib.oracle_segment.argtypes = [P, P, P, ctypes.c_double, P]
        lib.oracle_segment.restype = ctypes.c_int
        lib.oracle_rici_generate.argtypes = [P, i64, P, i64, P, i64, ctypes.c_double, ctypes.c_int, P, P, P,
                                             ctypes.c_double]
        lib.oracle_rici_generate.restype = None
        lib.oracle_rici_definition.argtypes = [P, i64, P, i64, P, i64, ctypes.c_double, ctypes.c_int, P]
        lib.oracle_rici_definition.restype = None
        lib.oracle_crss.argtypes = [P, P, ctypes.c_int]
        lib.oracle_crss.restype = ctypes.c_uint64
        lib.oracle_crss_matrix.argtypes = [P, i64, P, i64, ctypes.c_int, P]
        lib.oracle_crss_matrix.restype = None
        lib.oracle_count_below.argtypes = [P, i64, P, i64, ctypes.c_int, P, P]
        lib.oracle_count_below.restype = None
        lib.oracle_ranks.argtypes = [P, i64, P, i64, ctypes.c_int, P]
        lib.oracle_ranks.restype = None
        lib.oracle_clutter_fraction.argtypes = [P, i64, P, i64, P, P, i64, ctypes.c_double, ctypes.c_int, P, P, P]
        lib.oracle_clutter_fraction.restype = None
        lib.oracle_num_threads.argtypes = []
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def spin_frame(normal) -> tuple[np.ndarray, bool]:
    """Eq. 1 (corrected, G1) -> (N_ax, N_ay, N_bx, N_bz), valid flag."""
    o = np.zeros(6, dtype=np.float64)
    o[3:] = normal
    out = np.zeros(4, dtype=np.float64)
    ok = _load().oracle_spin_frame(_ptr(o), _ptr(out))
    return out, bool(ok)


def project(origin, point) -> tuple[float, float]:
    """Eqs. 2-5 -> (alpha, beta) of ``point`` for the oriented point ``origin`` (6 floats)."""
    o = np.ascontiguousarray(origin, dtype=np.float64)
    p = np.ascontiguousarray(point, dtype=np.float64)
    out = np.zeros(2, dtype=np.float64)
    _load().oracle_project(_ptr(o), _ptr(p), _ptr(out))
    return float(out[0]), float(out[1])


def segment(t0, t1, t2, beta):
    """P:270-276 steps 1-6 on projected vertices.  Returns None or a dict."""
    a = [np.ascontiguousarray(t, dtype=np.float64) for t in (t0, t1, t2)]
    out = np.zeros(7, dtype=np.float64)
    ok = _load().oracle_segment(_ptr(a[0]), _ptr(a[1]), _ptr(a[2]), float(beta), _ptr(out))
    if not ok:
        return None
    return {"E0": out[0:2].copy(), "E1": out[2:4].copy(), "rmin": out[4], "rmax": out[5],
            "rc": (None if out[6] < 0 else out[6])}


def _mesh_args(vertices, indices, origins):
    v = np.ascontiguousarray(vertices, dtype=np.float32).reshape(-1, 3)
    t = np.ascontiguousarray(indices, dtype=np.int32).reshape(-1, 3)
    o = np.ascontiguousarray(origins, dtype=np.float32).reshape(-1, 6)
    return v, t, o


def rici_generate(vertices, indices, origins, support_radius: float, n_bins: int,
                  fragile: bool = False, exact: bool = False, tau_rel: float = 1e-5):
    """Paper algorithm in double on the float32 inputs.

    Returns uint16 images [n, N, N] saturated at 65535 (G9) -- or the exact
    uint32 counts when ``exact`` -- plus, when ``fragile``, a bool mask of the
    pixels whose count changes under a tau = tau_rel*R displacement of the circle
    (default 1e-5, the north-star rule),
    and stats {pairs_in_slab, segments}.
    """
    v, t, o = _mesh_args(vertices, indices, origins)
    n, N = o.shape[0], int(n_bins)
    counts = np.zeros((n, N, N), dtype=np.uint32)
    fr = np.zeros((n, N, N), dtype=np.uint8) if fragile else None
    stats = np.zeros(2, dtype=np.int64)
    _load().oracle_rici_generate(_ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(o), n,
                                 float(support_radius), N, _ptr(counts),
                                 _ptr(fr) if fragile else None, _ptr(stats), float(tau_rel))
    img = counts if exact else np.minimum(counts, 65535).astype(np.uint16)
    res = {"images": img, "pairs_in_slab": int(stats[0]), "segments": int(stats[1])}
    if fragile:
        res["fragile"] = fr.astype(bool)
    return res


def rici_definition(vertices, indices, origins, support_radius: float, n_bins: int) -> np.ndarray:
    """O-def: circle/surface intersection count per pixel from the definition."""
    v, t, o = _mesh_args(vertices, indices, origins)
    n, N = o.shape[0], int(n_bins)
    counts = np.zeros((n, N, N), dtype=np.uint32)
    _load().oracle_rici_definition(_ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(o), n,
                                   float(support_radius), N, _ptr(counts))
    return counts


def _imgs(a):
    a = np.ascontiguousarray(a, dtype=np.uint16)
    if a.ndim == 2:
        a = a[None]
    assert a.shape[1] == a.shape[2]
    return a


def crss(needle, haystack) -> int:
    """Eq. 7 / Listing 1 for one (needle, haystack) pair."""
    n, h = _imgs(needle), _imgs(haystack)
    return int(_load().oracle_crss(_ptr(n), _ptr(h), n.shape[1]))


def crss_matrix(needles, haystack) -> np.ndarray:
    n, h = _imgs(needles), _imgs(haystack)
    out = np.zeros((n.shape[0], h.shape[0]), dtype=np.uint64)
    _load().oracle_crss_matrix(_ptr(n), n.shape[0], _ptr(h), h.shape[0], n.shape[1], _ptr(out))
    return out


def count_below(needles, haystack, thresholds) -> np.ndarray:
    n, h = _imgs(needles), _imgs(haystack)
    thr = np.ascontiguousarray(thresholds, dtype=np.uint64)
    out = np.zeros(n.shape[0], dtype=np.uint32)
    _load().oracle_count_below(_ptr(n), n.shape[0], _ptr(h), h.shape[0], n.shape[1], _ptr(thr), _ptr(out))
    return out


def ranks(needles, haystack) -> np.ndarray:
    """rank_i = #{j : CRSS(n_i, h_j) < CRSS(n_i, h_i)} (G10, G11)."""
    n, h = _imgs(needles), _imgs(haystack)
    assert h.shape[0] >= n.shape[0]
    out = np.zeros(n.shape[0], dtype=np.uint32)
    _load().oracle_ranks(_ptr(n), n.shape[0], _ptr(h), h.shape[0], n.shape[1], _ptr(out))
    return out


def clutter_fraction(vertices, indices, object_tag, origins, support_radius: float, q: int = 4):
    """Eq. 8 per oriented point with a Q x Q barycentric quadrature of the area
    inside the support cylinder (G17).  Returns (fraction, area_all, area_object)."""
    v, t, o = _mesh_args(vertices, indices, origins)
    tag = np.ascontiguousarray(object_tag, dtype=np.uint8).reshape(-1)
    assert tag.shape[0] == t.shape[0]
    n = o.shape[0]
    frac = np.zeros(n)
    aa = np.zeros(n)
    ao = np.zeros(n)
    _load().oracle_clutter_fraction(_ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(tag), _ptr(o), n,
                                    float(support_radius), int(q), _ptr(frac), _ptr(aa), _ptr(ao))
    return frac, aa, ao
