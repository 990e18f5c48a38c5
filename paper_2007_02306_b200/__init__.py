"""B200-native RICI hot path (arXiv 2007.02306): Python binding of librici.so.

Same names as the C ABI (include/rici.h).  Every function here only marshals
arguments -- shapes, dtypes, pointers, the current CUDA stream -- and calls the
library; all arithmetic runs in the sm_100a kernels.  Tensors may live on the
GPU (device pointers) or the host (the library stages them, see rici.h).

    mesh = rici_create_mesh(vertices, indices)              # [V,3] f32, [T,3] i32
    imgs = rici_generate(mesh, origins, 0.3, 64)            # [n,64,64] uint16
    ranks = rici_crss_search(needles, haystack)             # [n_needles] uint32 (int32 storage)
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import RiciError, check, load

__all__ = ["Mesh", "RiciError", "rici_create_mesh", "rici_destroy_mesh", "rici_generate",
           "rici_crss_search", "rici_crss_search_ex", "rici_clutter_fraction", "rici_crss_pairs", "rici_crss_count_below", "rici_crss_distances",
           "rici_launch_count", "rici_set_kernel_timing", "rici_kernel_time_ms", "rici_crss_guard_stats",
           "rici_version",
           "library_path"]


def library_path() -> str:
    from ._lib import LIB_PATH
    return LIB_PATH


def _stream(stream, device=None) -> int:
    if stream is None:
        if not torch.cuda.is_available():
            return 0
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _as_tensor(x, dtype: torch.dtype, name: str) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor or numpy array")
    if x.dtype != dtype:
        raise TypeError(f"{name}: expected dtype {dtype}, got {x.dtype}")
    if not x.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return x


def _u16(x: torch.Tensor) -> torch.Tensor:
    """uint16 images may arrive as torch.uint16 or as an int16 bit-view."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x).view(np.int16))
    if x.dtype == torch.uint16:
        x = x.view(torch.int16)
    if x.dtype != torch.int16:
        raise TypeError("images must be uint16 (or an int16 view of uint16)")
    if not x.is_contiguous():
        raise ValueError("images must be contiguous")
    return x


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t.numel() else 0)


class Mesh:
    """Owns a ``rici_mesh`` handle (device triangle buffer)."""

    def __init__(self, handle: ctypes.c_void_p, n_triangles: int, device: int):
        self._h = handle
        self.n_triangles = n_triangles
        self.device = device

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise ValueError("mesh was destroyed")
        return self._h

    def destroy(self) -> None:
        if self._h is not None:
            check(load().rici_destroy_mesh(self._h))
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def rici_create_mesh(vertices, indices, stream=None) -> Mesh:
    """(a1) ``rici_create_mesh``: vertices [V,3] float32, indices [T,3] int32 (device or host)."""
    v = _as_tensor(vertices, torch.float32, "vertices").reshape(-1, 3)
    t = _as_tensor(indices, torch.int32, "indices").reshape(-1, 3)
    h = ctypes.c_void_p()
    check(load().rici_create_mesh(_ptr(v), v.shape[0], _ptr(t), t.shape[0],
                                  ctypes.c_void_p(_stream(stream)), ctypes.byref(h)))
    dev = v.device.index if v.is_cuda else (torch.cuda.current_device() if torch.cuda.is_available() else 0)
    return Mesh(h, int(t.shape[0]), dev)


def rici_destroy_mesh(mesh: Mesh) -> None:
    mesh.destroy()


def rici_generate(mesh: Mesh, origins, support_radius: float, n_bins: int = 64, out=None,
                  stream=None) -> torch.Tensor:
    """(a2-a8) ``rici_generate``: origins [n,6] float32 -> uint16 images [n,N,N] (int16 storage
    holding the uint16 bit pattern; ``.view(torch.uint16)`` or numpy ``.view(np.uint16)``)."""
    o = _as_tensor(origins, torch.float32, "origins").reshape(-1, 6)
    n = o.shape[0]
    if out is None:
        out = torch.empty((n, n_bins, n_bins), dtype=torch.int16, device=o.device,
                          pin_memory=(not o.is_cuda and torch.cuda.is_available()))
    out = _u16(out)
    if out.numel() != n * n_bins * n_bins:
        raise ValueError("out has the wrong size")
    check(load().rici_generate(mesh.handle, _ptr(o), n, float(support_radius), int(n_bins),
                               _ptr(out), ctypes.c_void_p(_stream(stream))))
    return out


def _images(x, n_bins):
    x = _u16(x)
    P = n_bins * n_bins
    if x.numel() % P:
        raise ValueError("image buffer is not a multiple of n_bins^2")
    return x, x.numel() // P


def _bins_of(x) -> int:
    return int(x.shape[-1])


def rici_crss_search(needles, haystack, n_bins: int | None = None, out=None, stream=None,
                     early_exit: bool = False, simt: bool = False) -> torch.Tensor:
    """(a9-a12) ``rici_crss_search`` / ``rici_crss_search_ex``: ranks with needle i <-> haystack i.
    ``early_exit`` selects rank mode (identical ranks), ``simt`` forces the SIMT kernel.
    Returns an int32 tensor holding the uint32 ranks (needles' device, or pinned host memory)."""
    from ._lib import RICI_CRSS_EARLY_EXIT, RICI_CRSS_SIMT
    N = n_bins or _bins_of(needles)
    nd, nn = _images(needles, N)
    hd, nh = _images(haystack, N)
    if out is None:
        out = torch.empty(nn, dtype=torch.int32, device=nd.device,
                          pin_memory=(not nd.is_cuda and torch.cuda.is_available()))
    flags = (RICI_CRSS_EARLY_EXIT if early_exit else 0) | (RICI_CRSS_SIMT if simt else 0)
    if flags:
        check(load().rici_crss_search_ex(_ptr(nd), nn, _ptr(hd), nh, N, flags, _ptr(out),
                                         ctypes.c_void_p(_stream(stream))))
    else:
        check(load().rici_crss_search(_ptr(nd), nn, _ptr(hd), nh, N, _ptr(out),
                                      ctypes.c_void_p(_stream(stream))))
    return out


def rici_crss_search_ex(needles, haystack, flags: int, n_bins: int | None = None, out=None, stream=None):
    """``rici_crss_search_ex`` with raw flags (RICI_CRSS_SIMT = 1, RICI_CRSS_EARLY_EXIT = 2)."""
    return rici_crss_search(needles, haystack, n_bins, out, stream, early_exit=bool(flags & 2),
                            simt=bool(flags & 1))


def rici_crss_pairs(needles, haystack, pairs, n_bins: int | None = None, out=None, stream=None) -> torch.Tensor:
    """``rici_crss_pairs``: pairs [m,2] int64 -> CRSS uint64 (int64 storage)."""
    N = n_bins or _bins_of(needles)
    nd, nn = _images(needles, N)
    hd, nh = _images(haystack, N)
    p = _as_tensor(pairs, torch.int64, "pairs").reshape(-1, 2)
    m = p.shape[0]
    if out is None:
        out = torch.empty(m, dtype=torch.int64, device=nd.device)
    check(load().rici_crss_pairs(_ptr(nd), nn, _ptr(hd), nh, N, _ptr(p), m, _ptr(out),
                                 ctypes.c_void_p(_stream(stream))))
    return out


def rici_crss_count_below(needles, haystack, thresholds, n_bins: int | None = None, out=None,
                          stream=None) -> torch.Tensor:
    """``rici_crss_count_below``: counts (int32 storage of uint32) of haystack images closer than the
    per-needle threshold (uint64 in int64 storage)."""
    N = n_bins or _bins_of(needles)
    nd, nn = _images(needles, N)
    hd, nh = _images(haystack, N)
    thr = _as_tensor(thresholds, torch.int64, "thresholds")
    if out is None:
        out = torch.empty(nn, dtype=torch.int32, device=nd.device)
    check(load().rici_crss_count_below(_ptr(nd), nn, _ptr(hd), nh, N, _ptr(thr), _ptr(out),
                                       ctypes.c_void_p(_stream(stream))))
    return out


def rici_crss_distances(needles, haystack, n_bins: int | None = None, out=None, stream=None) -> torch.Tensor:
    """``rici_crss_distances``: full [n_needles, n_haystack] CRSS matrix (uint64 in int64 storage)."""
    N = n_bins or _bins_of(needles)
    nd, nn = _images(needles, N)
    hd, nh = _images(haystack, N)
    if out is None:
        out = torch.empty((nn, nh), dtype=torch.int64, device=nd.device)
    check(load().rici_crss_distances(_ptr(nd), nn, _ptr(hd), nh, N, _ptr(out),
                                     ctypes.c_void_p(_stream(stream))))
    return out


def rici_clutter_fraction(mesh: Mesh, object_tag, origins, support_radius: float, quadrature_q: int = 4,
                          with_area: bool = False, stream=None):
    """(f4) ``rici_clutter_fraction``: Eq. 8 per oriented point.  object_tag [T] uint8 in the
    triangle order given to rici_create_mesh.  Returns float32 fractions (and A_all)."""
    t = _as_tensor(object_tag, torch.uint8, "object_tag").reshape(-1)
    o = _as_tensor(origins, torch.float32, "origins").reshape(-1, 6)
    n = o.shape[0]
    frac = torch.empty(n, dtype=torch.float32, device=o.device)
    area = torch.empty(n, dtype=torch.float32, device=o.device) if with_area else None
    check(load().rici_clutter_fraction(mesh.handle, _ptr(t), _ptr(o), n, float(support_radius), int(quadrature_q),
                                       _ptr(frac), _ptr(area) if with_area else None,
                                       ctypes.c_void_p(_stream(stream))))
    return (frac, area) if with_area else frac


def rici_launch_count() -> int:
    return int(load().rici_launch_count())


def rici_set_kernel_timing(enable: bool) -> None:
    """``rici_set_kernel_timing``: record CUDA events around the timed kernels' launches."""
    check(load().rici_set_kernel_timing(1 if enable else 0))


def rici_kernel_time_ms(kernel: int) -> tuple[float, int]:
    """``rici_kernel_time_ms``: (mean ms per recorded launch, launches) of kernel id
    RICI_KERNEL_GENERATE (0) or RICI_KERNEL_CRSS_MMA (1); clears the record."""
    ms, n = ctypes.c_float(0.0), ctypes.c_int64(0)
    check(load().rici_kernel_time_ms(int(kernel), ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def rici_version() -> str:
    return load().rici_version().decode()


def rici_crss_guard_stats(reset: bool = False) -> dict:
    """Guard coverage of the tensor-core CRSS path on the current device (include/rici.h)."""
    out = (ctypes.c_int64 * 5)()
    check(load().rici_crss_guard_stats(out, int(bool(reset))))
    keys = ("needles", "needles_outside_guard", "haystack", "haystack_outside_guard", "needles_not_2_4")
    return dict(zip(keys, (int(x) for x in out)))
