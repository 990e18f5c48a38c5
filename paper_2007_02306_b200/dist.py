"""Data-parallel sharding of the RICI hot path over the GPUs of one node.

Construction (a2-a8): the oriented points are split into contiguous blocks, one per rank;
the mesh is replicated; no collective -- each rank's image block IS its haystack shard.

Search (a9-a12): the haystack is split into contiguous blocks; the needle set is on
every rank (broadcast once); the only exchange steps are
  * thresholds t_i = CRSS(n_i, h_i): computed by the rank that owns h_i (a10), combined
    with all_reduce(MAX) (non-owners contribute 0), and
  * ranks: each rank counts haystack images closer than t_i in its shard (a11 + a12),
    then all_reduce(SUM) of the per-needle partial counts.
Integer counts summed exactly, so ranks are identical for every world size.

The compute calls default to the CUDA library; ``ops`` lets the CPU tests drive the same
host logic (sharding arithmetic, collectives) under the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ``n`` items for ``rank`` of ``world`` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class SearchOps:
    """Compute primitives used by :func:`search_sharded` (defaults: librici.so)."""
    pairs: Callable        # (needles, haystack_shard, pairs[m,2] int64) -> uint64 CRSS (int64 storage)
    count_below: Callable  # (needles, haystack_shard, thresholds) -> per-needle counts (int32)


def cuda_ops() -> SearchOps:
    from . import rici_crss_count_below, rici_crss_pairs
    return SearchOps(pairs=rici_crss_pairs, count_below=rici_crss_count_below)


def _world_rank(group=None) -> tuple[int, int]:
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def generate_sharded(mesh, origins: torch.Tensor, support_radius: float, n_bins: int = 64,
                     group=None, generate: Callable | None = None, out: torch.Tensor | None = None):
    """Each rank generates the images of its block of ``origins`` (the full [n,6] array; the
    mesh is replicated, no collective).  ``out`` (optional) receives the block: [hi-lo, N, N].
    Returns (images of the block, (lo, hi))."""
    world, rank = _world_rank(group)
    lo, hi = shard_range(origins.shape[0], world, rank)
    if generate is None:
        from . import rici_generate as generate
    if out is not None:
        return generate(mesh, origins[lo:hi].contiguous(), support_radius, n_bins, out=out), (lo, hi)
    return generate(mesh, origins[lo:hi].contiguous(), support_radius, n_bins), (lo, hi)


def all_gather_images(images: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """In place: ``images`` [n_total, N, N] holds this rank's block shard_range(n_total, ...)
    on entry and every rank's block on exit (the needles generated sharded).
    Blocks differ in size by at most one image, so each is sent padded to the largest as raw
    bytes (no int16 type in NCCL/gloo) with one all_gather_into_tensor."""
    world, rank = _world_rank(group)
    if world == 1:
        return images
    per = -(-n_total // world)
    img_bytes = images[0].numel() * images.element_size() if n_total else 0
    lo, hi = shard_range(n_total, world, rank)
    send = torch.zeros(per * img_bytes, dtype=torch.uint8, device=images.device)
    send[: (hi - lo) * img_bytes] = images[lo:hi].reshape(-1).view(torch.uint8)
    recv = torch.empty(world * per * img_bytes, dtype=torch.uint8, device=images.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    flat = images.reshape(-1).view(torch.uint8)
    for r in range(world):
        a, b = shard_range(n_total, world, r)
        if r != rank and b > a:
            flat[a * img_bytes: b * img_bytes] = recv[r * per * img_bytes: (r * per + b - a) * img_bytes]
    return images


def broadcast_images(images: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Broadcast ``images`` (uint16 counts in int16 storage, in place) from global rank ``src``
    (the torch.distributed convention for ``dist.broadcast``).  When every count fits a byte --
    RICI counts of one object rarely exceed a few tens -- the payload goes as uint8, half the
    bytes; otherwise the raw bytes (neither NCCL nor gloo has an int16 type).  Exact either way."""
    dev = images.device
    me = dist.get_rank() == src
    small = torch.zeros(1, dtype=torch.int32, device=dev)
    if me and images.numel():
        small.fill_(int(images.view(torch.int16).to(torch.int32).bitwise_and(0xFFFF).max().item() <= 255))
    dist.broadcast(small, src, group=group)
    if not int(small.item()):
        dist.broadcast(images.view(torch.uint8), src, group=group)   # NCCL/gloo have no int16: bytes
        return images
    packed = images.to(torch.uint8) if me else torch.empty(images.shape, dtype=torch.uint8, device=dev)
    dist.broadcast(packed, src, group=group)
    if not me:
        images.copy_(packed.to(torch.int16))
    return images


def search_sharded(needles: torch.Tensor, haystack_shard: torch.Tensor, shard_lo: int,
                   n_bins: int = 64, group=None, ops: SearchOps | None = None) -> torch.Tensor:
    """Ranks of needle i's correspondence haystack i over the union of all ranks' shards.

    needles         [n_needles, N, N] on every rank (uint16 in int16 storage)
    haystack_shard  this rank's contiguous block of the global haystack, starting at global
                    index ``shard_lo``
    Returns int64 ranks [n_needles] on every rank.
    """
    ops = ops or cuda_ops()
    nn = needles.shape[0]
    dev = needles.device
    n_local = haystack_shard.shape[0]
    # a10 on the owner of h_i: needles whose correspondence lies in [shard_lo, shard_lo + n_local)
    lo = max(0, min(shard_lo, nn))
    hi = max(lo, min(shard_lo + n_local, nn))
    thr = torch.zeros(nn, dtype=torch.int64, device=dev)
    if hi > lo:
        idx = torch.arange(lo, hi, dtype=torch.int64, device=dev)
        pairs = torch.stack([idx, idx - shard_lo], 1).contiguous()
        thr[lo:hi] = ops.pairs(needles, haystack_shard, pairs, n_bins)
    if dist.is_initialized():
        # thresholds are uint64 in int64 storage; CRSS <= 4032 * 131070^2 < 2^63, so MAX is exact
        dist.all_reduce(thr, op=dist.ReduceOp.MAX, group=group)
    counts = ops.count_below(needles, haystack_shard, thr, n_bins).to(torch.int64)
    if dist.is_initialized():
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts
