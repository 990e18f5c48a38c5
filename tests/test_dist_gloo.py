"""Multi-rank host logic of paper_2007_02306_b200.dist on CPU (gloo, world sizes 2 and 3).

The collectives, shard arithmetic and threshold ownership run exactly as on the GPUs; the
two compute primitives are supplied by the oracle here (test-only injection), so the result
must equal the oracle's single-process ranks bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_02306_b200.dist import (SearchOps, all_gather_images, broadcast_images, generate_sharded,
                                        search_sharded, shard_range)


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 34848):
        for w in (1, 2, 3, 8):
            blocks = [shard_range(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_ops():
    import oracle

    def pairs(needles, hay, pr, n_bins):
        n = needles.numpy().view(np.uint16)
        h = hay.numpy().view(np.uint16)
        out = [oracle.crss(n[i], h[j]) for i, j in pr.numpy()]
        return torch.tensor(np.array(out, np.uint64).view(np.int64))

    def count_below(needles, hay, thr, n_bins):
        n = needles.numpy().view(np.uint16)
        h = hay.numpy().view(np.uint16).reshape(-1, n_bins, n_bins)
        return torch.from_numpy(oracle.count_below(n, h, thr.numpy().view(np.uint64)).astype(np.int32))

    return SearchOps(pairs=pairs, count_below=count_below)


def _worker(rank, world, port, needles, haystack, origins, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        # construction: each rank its block of origins, no collective
        import synth
        m = synth.bumpy_torus(40, 20, key=(21,))

        def gen(mesh, o, R, N):
            return torch.from_numpy(oracle.rici_generate(m.vertices, m.indices, o.numpy(), R, N)["images"].view(np.int16))
        imgs, (lo, hi) = generate_sharded(None, torch.from_numpy(origins), 0.3, 64, generate=gen)
        gathered = [None] * world
        dist.all_gather_object(gathered, (lo, hi, imgs.numpy()))
        # the same blocks generated into a full-size buffer and all-gathered in place (the
        # bench's needle path); blocks of unequal size (n % world != 0) are padded on the wire
        full_buf = torch.full((origins.shape[0], 64, 64), -7, dtype=torch.int16)
        generate_sharded(None, torch.from_numpy(origins), 0.3, 64,
                         generate=lambda mesh, o, R, N, out: out.copy_(gen(mesh, o, R, N)), out=full_buf[lo:hi])
        all_gather_images(full_buf, origins.shape[0])
        # search: haystack split in contiguous blocks
        nh = haystack.shape[0]
        slo, shi = shard_range(nh, world, rank)
        shard = torch.from_numpy(haystack[slo:shi].view(np.int16))
        # needles from rank 0 only (the bench's layout): small counts go as uint8, large as is
        nd = torch.from_numpy(needles.view(np.int16).copy()) if rank == 0 else torch.zeros(needles.shape, dtype=torch.int16)
        broadcast_images(nd, 0)
        big = torch.from_numpy(needles.view(np.int16).copy()) if rank == 0 else torch.zeros(needles.shape, dtype=torch.int16)
        if rank == 0:
            big[0, 0, 5] = -2                                        # 65534 as uint16: full width
        broadcast_images(big, 0)
        bcast_ok = bool(torch.equal(nd, torch.from_numpy(needles.view(np.int16)))) and int(big[0, 0, 5]) == -2
        ranks = search_sharded(nd, shard, slo, 64, ops=_oracle_ops())
        q.put((rank, ranks.numpy(), gathered if rank == 0 else None, bcast_ok, full_buf.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_and_generate_equal_single_process(oracle_mod, world):
    import synth
    m = synth.bumpy_torus(40, 20, key=(21,))
    origins = m.origins[::7].copy()
    full = oracle_mod.rici_generate(m.vertices, m.indices, origins, 0.3, 64)["images"]
    rng = np.random.default_rng(world)
    needles = full[:20].copy()
    clutter = full[rng.permutation(full.shape[0])][:37]
    haystack = np.concatenate([full[:20], clutter, full[3:5]])          # ties via duplicates
    want = oracle_mod.ranks(needles, haystack)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, needles, haystack, origins, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ranks, gathered, bcast_ok, full_buf in res:
        assert bcast_ok, rank
        assert np.array_equal(full_buf.view(np.uint16), full), rank         # all_gather_images
        assert np.array_equal(ranks.astype(np.uint32), want), rank
        if gathered is not None:
            parts = sorted(gathered, key=lambda g: g[0])
            cat = np.concatenate([g[2].view(np.uint16) for g in parts])
            assert np.array_equal(cat, full)
