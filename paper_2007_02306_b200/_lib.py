"""ctypes binding of librici.so (include/rici.h).  Argument marshalling only.

There is no fallback of any kind: if the shared library is missing or cannot be
loaded, importing the ops raises.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``python paper_2007_02306_b200/build.py``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librici.so")

SYMBOLS = ["rici_create_mesh", "rici_destroy_mesh", "rici_mesh_num_triangles", "rici_generate",
           "rici_crss_search", "rici_crss_search_ex", "rici_crss_pairs", "rici_crss_count_below", "rici_crss_distances",
           "rici_clutter_fraction", "rici_last_error", "rici_launch_count", "rici_set_kernel_timing",
           "rici_kernel_time_ms", "rici_crss_guard_stats", "rici_version"]

RICI_CRSS_SIMT = 1
RICI_CRSS_EARLY_EXIT = 2
RICI_KERNEL_GENERATE = 0
RICI_KERNEL_CRSS_MMA = 1

STATUS = {0: "RICI_OK", 1: "RICI_ERR_INVALID_ARGUMENT", 2: "RICI_ERR_CUDA",
          3: "RICI_ERR_OUT_OF_MEMORY", 4: "RICI_ERR_UNSUPPORTED"}

_lib = None


class RiciError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: the CUDA extension is not built "
                          "(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    st = ctypes.c_int
    lib.rici_create_mesh.argtypes = [P, i64, P, i64, P, ctypes.POINTER(P)]
    lib.rici_create_mesh.restype = st
    lib.rici_destroy_mesh.argtypes = [P]
    lib.rici_destroy_mesh.restype = st
    lib.rici_mesh_num_triangles.argtypes = [P]
    lib.rici_mesh_num_triangles.restype = i64
    lib.rici_generate.argtypes = [P, P, i64, ctypes.c_float, i32, P, P]
    lib.rici_generate.restype = st
    lib.rici_crss_search.argtypes = [P, i64, P, i64, i32, P, P]
    lib.rici_crss_search.restype = st
    lib.rici_crss_search_ex.argtypes = [P, i64, P, i64, i32, ctypes.c_uint32, P, P]
    lib.rici_crss_search_ex.restype = st
    lib.rici_crss_pairs.argtypes = [P, i64, P, i64, i32, P, i64, P, P]
    lib.rici_crss_pairs.restype = st
    lib.rici_crss_count_below.argtypes = [P, i64, P, i64, i32, P, P, P]
    lib.rici_crss_count_below.restype = st
    lib.rici_crss_distances.argtypes = [P, i64, P, i64, i32, P, P]
    lib.rici_crss_distances.restype = st
    lib.rici_clutter_fraction.argtypes = [P, P, P, i64, ctypes.c_float, i32, P, P, P]
    lib.rici_clutter_fraction.restype = st
    lib.rici_last_error.argtypes = []
    lib.rici_last_error.restype = ctypes.c_char_p
    lib.rici_launch_count.argtypes = []
    lib.rici_launch_count.restype = ctypes.c_uint64
    lib.rici_set_kernel_timing.argtypes = [i32]
    lib.rici_set_kernel_timing.restype = st
    lib.rici_kernel_time_ms.argtypes = [i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i64)]
    lib.rici_kernel_time_ms.restype = st
    lib.rici_crss_guard_stats.argtypes = [ctypes.POINTER(i64), i32]
    lib.rici_crss_guard_stats.restype = st
    lib.rici_version.argtypes = []
    lib.rici_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        raise RiciError(status, load().rici_last_error().decode(errors="replace"))
