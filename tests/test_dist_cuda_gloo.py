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


def _scene_worker(rank, world, port, ref_v, ref_t, ref_o, sc_v, sc_t, sc_o, q):
    """The bench's N>1 step on one C4-shaped scene: each rank generates its block of the scene's
    oriented points (its haystack shard) and of the reference's (all-gathered into the needle
    set), then search_sharded (owner thresholds + all_reduce MAX, local counts + all_reduce SUM)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2007_02306_b200 as rici
        from paper_2007_02306_b200.dist import all_gather_images, generate_sharded, search_sharded, shard_range
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        rv, rt, ro, sv, st, so = (torch.from_numpy(x).to(dev) for x in (ref_v, ref_t, ref_o, sc_v, sc_t, sc_o))
        needles = torch.full((ro.shape[0], 64, 64), -1, dtype=torch.int16, device=dev)
        lo_r, hi_r = shard_range(ro.shape[0], world, rank)
        m_ref = rici.rici_create_mesh(rv, rt)
        generate_sharded(m_ref, ro, 0.3, 64, out=needles[lo_r:hi_r])
        torch.cuda.synchronize()
        nd_cpu = needles.cpu()                      # gloo moves CPU tensors
        all_gather_images(nd_cpu, ro.shape[0])
        needles.copy_(nd_cpu)
        m_sc = rici.rici_create_mesh(sv, st)
        hay, (lo_h, hi_h) = generate_sharded(m_sc, so, 0.3, 64)
        torch.cuda.synchronize()
        ranks = search_sharded(needles, hay, lo_h, 64)
        torch.cuda.synchronize()
        q.put((rank, lo_h, hay.cpu().numpy(), needles.cpu().numpy(), ranks.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_scene_step_cuda_two_ranks():
    """SURVEY 8(e) on one scene: construction sharded over oriented points (mesh replicated),
    needles all-gathered, haystack sharded -- the images and the ranks must be byte-identical to
    one process doing the whole step."""
    import torch.multiprocessing as mp

    import paper_2007_02306_b200 as rici
    import synth
    objs = [synth.bumpy_torus(70, 35, key=(47, k), minor=0.25 + 0.04 * k, amp=0.08) for k in range(4)]
    sc = synth.clutterbox(objs, key=(47, 1000))
    n_ref = objs[0].n_vertices
    ref = synth.Mesh(sc.vertices[:n_ref].copy(), objs[0].indices.copy(), sc.normals[:n_ref].copy())
    ro, so = ref.origins[:-3].copy(), sc.origins            # ragged blocks: odd counts
    m1 = rici.rici_create_mesh(torch.from_numpy(ref.vertices).cuda(), torch.from_numpy(ref.indices).cuda())
    nd1 = rici.rici_generate(m1, torch.from_numpy(ro).cuda(), 0.3, 64)
    m2 = rici.rici_create_mesh(torch.from_numpy(sc.vertices).cuda(), torch.from_numpy(sc.indices).cuda())
    hay1 = rici.rici_generate(m2, torch.from_numpy(so).cuda(), 0.3, 64)
    want = rici.rici_crss_search(nd1, hay1).cpu().numpy().astype(np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (ref.vertices, ref.indices, ro, sc.vertices, sc.indices, so)
    procs = [ctx.Process(target=_scene_worker, args=(r, 2, port, *args, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    hay = np.concatenate([r[2] for r in res])
    assert np.array_equal(hay, hay1.cpu().numpy())
    for rank, lo, _, needles, ranks in res:
        assert np.array_equal(needles, nd1.cpu().numpy()), rank
        assert np.array_equal(ranks.astype(np.int64), want), rank
