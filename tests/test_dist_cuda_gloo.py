"""The multi-rank search path with the real CUDA library: two processes share cuda:0 and talk
over gloo (functional check of dist.py's collectives and shard arithmetic with the tensor-core
counts; no timing, and no kernel waits on another rank's kernel)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, needles, haystack, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_02306_b200.dist import broadcast_images, search_sharded, shard_range
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        nd = torch.from_numpy(needles.view(np.int16)).to(dev) if rank == 0 else \
            torch.zeros(needles.shape, dtype=torch.int16, device=dev)
        broadcast_images(nd, 0)
        nh = haystack.shape[0]
        lo, hi = shard_range(nh, world, rank)
        shard = torch.from_numpy(haystack[lo:hi].view(np.int16)).to(dev)
        ranks = search_sharded(nd, shard, lo, 64)
        torch.cuda.synchronize()
        q.put((rank, ranks.cpu().numpy(), bool(torch.equal(nd.cpu(), torch.from_numpy(needles.view(np.int16))))))
    finally:
        dist.destroy_process_group()


def test_search_sharded_cuda_two_ranks():
    import torch.multiprocessing as mp

    import paper_2007_02306_b200 as rici
    import synth
    m = synth.bumpy_torus(120, 60, key=(23,))
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    imgs = rici.rici_generate(mesh, torch.from_numpy(m.origins).cuda(), 0.3, 64)
    needles = imgs[:600].cpu().numpy().view(np.uint16).copy()
    rng = np.random.default_rng(5)
    haystack = imgs[torch.from_numpy(np.concatenate([np.arange(600), rng.permutation(imgs.shape[0])[:1500]]))]
    haystack = haystack.cpu().numpy().view(np.uint16).copy()
    want = rici.rici_crss_search(torch.from_numpy(needles.view(np.int16)).cuda(),
                                 torch.from_numpy(haystack.view(np.int16)).cuda()).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, needles, haystack, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ranks, bcast_ok in res:
        assert bcast_ok, rank
        assert np.array_equal(ranks.astype(np.int64), want.astype(np.int64)), rank
