"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

RICI images (north star): at most 1e-4 of the pixels may differ and every differing
pixel must be fragile -- its oracle count changes when the circle moves by up to
tau = 1e-5*R in beta and/or rho.  Closed-form hand cases must match exactly.
CRSS distances and ranks: bit-exact on identical images.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rici():
    import paper_2007_02306_b200 as r
    r._lib.load()
    assert torch.cuda.is_available()
    return r


DEV = "cuda:0"


def _gen(rici, mesh, origins, R, N):
    m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).to(DEV), torch.from_numpy(mesh.indices).to(DEV))
    o = torch.from_numpy(np.ascontiguousarray(origins, dtype=np.float32)).to(DEV)
    out = rici.rici_generate(m, o, R, N)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint16)


def _assert_parity(gpu, ref, max_frac=1e-4):
    """North-star rule on workload-shaped meshes: <= 1e-4 of pixels differ, all attributable.
    Tie-adversarial inputs (grid-snapped soups) keep the attribution rule with a looser count."""
    diff = gpu != ref["images"]
    n_bad = int((diff & ~ref["fragile"]).sum())
    assert n_bad == 0, f"{n_bad} non-attributable differing pixels"
    assert diff.mean() <= max_frac, f"{int(diff.sum())} differing pixels ({diff.mean():.2e})"
    return int(diff.sum())


def _parity_sampled(oracle_mod, g, mesh, origins, R, N, max_frac=1e-4):
    """The parity rule on a sample of images, with the oracle's fragility stencil (9 runs of
    the algorithm per image) evaluated only on the images that differ.  Returns n_diff."""
    ref = oracle_mod.rici_generate(mesh.vertices, mesh.indices, origins, R, N)
    diff = g != ref["images"]
    n_diff = int(diff.sum())
    bad = np.nonzero(diff.reshape(diff.shape[0], -1).any(1))[0]
    if bad.size:
        fr = oracle_mod.rici_generate(mesh.vertices, mesh.indices, origins[bad], R, N, fragile=True)["fragile"]
        n_bad = int((diff[bad] & ~fr).sum())
        assert n_bad == 0, f"{n_bad} non-attributable differing pixels in {bad.size} images"
    assert n_diff <= max_frac * diff.size, f"{n_diff} differing pixels ({n_diff / diff.size:.2e})"
    return n_diff


def test_c1_icosphere(rici, oracle_mod):
    cfg = synth.config_c1()
    g = _gen(rici, cfg["mesh"], cfg["origins"], cfg["R"], cfg["N"])
    ref = oracle_mod.rici_generate(cfg["mesh"].vertices, cfg["mesh"].indices, cfg["origins"],
                                   cfg["R"], cfg["N"], fragile=True)
    _assert_parity(g, ref)


def test_h2_single_triangle_small_N(rici, oracle_mod):
    m = synth.Mesh(np.array([[1, -2, -1], [1, -2, 2], [1, 2, -1]], np.float32),
                   np.array([[0, 1, 2]], np.int32), np.zeros((3, 3), np.float32))
    o = np.array([[0, 0, 0, 0, 0, 1]], np.float32)
    g = _gen(rici, m, o, 4.0, 8)
    assert np.array_equal(g, oracle_mod.rici_generate(m.vertices, m.indices, o, 4.0, 8)["images"])


def test_cube_and_tetra_closed_forms(rici, oracle_mod):
    c = synth.cube()
    corners = np.array([[x, y, z] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)], np.float32)
    o = np.concatenate([corners, corners / np.sqrt(3)], 1).astype(np.float32)
    g = _gen(rici, c, o, 1.0, 64)
    assert np.array_equal(g, oracle_mod.rici_generate(c.vertices, c.indices, o, 1.0, 64)["images"])
    assert (g.reshape(8, -1).sum(1) == 2184).all()
    t = synth.tetrahedron()
    s = 1 / np.sqrt(3)
    o = np.array([[1, 1, 1, s, s, s]], np.float32)
    g = _gen(rici, t, o, 1.0, 64)
    assert g.sum() == 1080


def test_h3_face_diagonal_ties_exact(rici, oracle_mod):
    """H3': the cube corner with S_n = +z puts 32 pixels exactly on a face diagonal shared by
    two triangles.  The count there (2) is locally constant, so the oracle does not flag it and
    the GPU must match every pixel exactly."""
    c = synth.cube()
    o = np.array([[1, 1, 1, 0, 0, 1]], np.float32)
    g = _gen(rici, c, o, 1.0, 64)
    ref = oracle_mod.rici_generate(c.vertices, c.indices, o, 1.0, 64, fragile=True)
    assert not ref["fragile"].any()
    assert np.array_equal(g, ref["images"])


@pytest.mark.parametrize("k", [0.5, -0.5, 2.0, -2.0])
def test_tau_width_cases_exact(rici, oracle_mod, k):
    """The tau-width pins of tests/test_oracle_rici.py (one decision k*tau from a layer edge, a
    |C| edge and a |E| edge): the float32 path resolves even the k = +-0.5 ties exactly."""
    from test_oracle_rici import layer_edge_triangle, double_range_plane, single_range_plane, _O_UP
    for m in (layer_edge_triangle(k), double_range_plane(k), single_range_plane(k)):
        g = _gen(rici, m, _O_UP, 1.0, 64)
        assert np.array_equal(g, oracle_mod.rici_generate(m.vertices, m.indices, _O_UP, 1.0, 64)["images"])


@pytest.mark.parametrize("N", [2, 8, 30, 64, 100, 128])
def test_bin_counts(rici, oracle_mod, N):
    m = synth.bumpy_torus(60, 30, key=(9,))
    o = m.origins[::37]
    g = _gen(rici, m, o, 0.3, N)
    ref = oracle_mod.rici_generate(m.vertices, m.indices, o, 0.3, N, fragile=True)
    _assert_parity(g, ref)


@pytest.mark.parametrize("case", ["soup", "grid_soup", "far_scene"])
def test_adversarial(rici, oracle_mod, case):
    if case == "soup":
        m = synth.triangle_soup(700, (5,), extent=0.5)
        o, R = synth.random_origins(67, (6,), 0.3), 0.5
    elif case == "grid_soup":
        m = synth.triangle_soup(700, (7,), extent=0.5, grid=1 / 32)
        o = synth.random_origins(67, (8,), 0.3)
        o[:, :3] = np.round(o[:, :3] * 32) / 32
        o[::3, 3:] = [0, 0, 1]
        o[1::3, 3:] = [0, 0, -1]
        R = 0.5
    else:
        # scene far from the origin: float cancellation in P - S_v (translate first, Eq. 2)
        m = synth.bumpy_torus(80, 40, key=(13,))
        m = synth.place(m, synth.random_rotation(np.random.default_rng(3)), [2.7, 1.3, 2.2])
        o, R = m.origins[::13], 0.3
    g = _gen(rici, m, o, R, 64)
    ref = oracle_mod.rici_generate(m.vertices, m.indices, o, R, 64, fragile=True)
    # grid_soup snaps every coordinate and half the normals to a 1/32 grid, so ~4% of its
    # pixels sit exactly on a decision, where FP32 and FP64 legitimately resolve the tie
    # differently: attribution stays binding and the differing pixels are bounded by 10% of
    # the fragile ones.  Workload-shaped meshes keep <= 1e-4.
    if case == "grid_soup":
        assert ref["fragile"].mean() > 5e-3
        n_diff = _assert_parity(g, ref, max_frac=1.0)
        # every differing pixel must be an EXACT tie: flagged by the same stencil at
        # tau = 1e-12 R, far below float32 resolution (~6e-8 R), i.e. a decision whose double-
        # precision margin is zero up to rounding -- where FP32 and FP64 may both be right (G16)
        # Exact ties are not errors (G16: both counts are correct); every OTHER differing pixel
        # is a float32-vs-double rounding disagreement and counts against the north star's 1e-4
        # budget, like on the workload meshes.
        tie = oracle_mod.rici_generate(m.vertices, m.indices, o, R, 64, fragile=True, tau_rel=1e-12)["fragile"]
        diff = g != ref["images"]
        n_near = int((diff & ~tie).sum())
        print(f"grid_soup: {n_diff} differing pixels ({n_near} not exact ties), {int(tie.sum())} exact-tie "
              f"pixels, {int(ref['fragile'].sum())} fragile, of {diff.size}")
        assert n_near <= 1e-4 * diff.size, f"{n_near} differing pixels that are not exact ties"
        assert n_diff <= 0.1 * ref["fragile"].sum()
    else:
        _assert_parity(g, ref)


def test_degenerate_inputs(rici):
    c = synth.cube()
    o = np.array([[1, 1, 1, 0, 0, 0], [1, 1, 1, np.nan, 0, 1], [50, 50, 50, 0, 0, 1]], np.float32)
    g = _gen(rici, c, o, 1.0, 64)
    assert not g.any()
    empty = synth.Mesh(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.int32), np.zeros((0, 3), np.float32))
    g = _gen(rici, empty, synth.random_origins(5, (1,)), 1.0, 64)
    assert g.shape == (5, 64, 64) and not g.any()
    # zero images requested
    m = rici.rici_create_mesh(torch.from_numpy(c.vertices).to(DEV), torch.from_numpy(c.indices).to(DEV))
    out = rici.rici_generate(m, torch.zeros((0, 6), device=DEV), 1.0, 64)
    assert out.shape == (0, 64, 64)


def test_bad_index_rejected(rici):
    v = torch.zeros((3, 3), device=DEV)
    t = torch.tensor([[0, 1, 3]], dtype=torch.int32, device=DEV)
    with pytest.raises(rici.RiciError) as e:
        rici.rici_create_mesh(v, t)
    assert e.value.status == 1


def test_c2_sampled(rici, oracle_mod):
    """C2 at full size (34,848 images, the bench launch configuration); oracle on a sample."""
    cfg = synth.config_c2()
    m = cfg["mesh"]
    g = _gen(rici, m, cfg["origins"], cfg["R"], cfg["N"])
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(m.n_vertices, 2000, replace=False))   # >= 2,000
    idx[-1] = m.n_vertices - 1                               # the ragged tail
    _parity_sampled(oracle_mod, g[idx], m, cfg["origins"][idx], cfg["R"], cfg["N"])
    # property at full size: closed surface -> even counts except fragile pixels (sampled above)
    assert (g % 2 == 1).mean() < 1e-4


def test_host_pointer_path_equals_device_path(rici):
    cfg = synth.config_c1()
    m = cfg["mesh"]
    dev = _gen(rici, m, cfg["origins"], cfg["R"], cfg["N"])
    hm = rici.rici_create_mesh(m.vertices, m.indices)                  # numpy -> host pointers
    host = rici.rici_generate(hm, cfg["origins"], cfg["R"], cfg["N"])
    assert np.array_equal(host.numpy().view(np.uint16), dev)
    r_host = rici.rici_crss_search(host, host)
    r_dev = rici.rici_crss_search(torch.from_numpy(dev.view(np.int16)).to(DEV),
                                  torch.from_numpy(dev.view(np.int16)).to(DEV))
    assert np.array_equal(r_host.numpy(), r_dev.cpu().numpy())


# ------------------------------------------------------------------------------- CRSS
def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(DEV)


def _rand_imgs(rng, k, N=64, hi=12, density=0.3):
    a = rng.integers(0, hi, (k, N, N))
    a[rng.random((k, N, N)) > density] = 0
    return a.astype(np.uint16)


def test_crss_distances_c1_bit_exact(rici, oracle_mod):
    cfg = synth.config_c1()
    g = _gen(rici, cfg["mesh"], cfg["origins"], cfg["R"], cfg["N"])
    d = rici.rici_crss_distances(_dev(g), _dev(g)).cpu().numpy().view(np.uint64)
    assert np.array_equal(d, oracle_mod.crss_matrix(g, g))
    assert set(np.unique(d)) <= {0, 8856, 10908}
    r = rici.rici_crss_search(_dev(g), _dev(g)).cpu().numpy()
    assert not r.any()


@pytest.mark.parametrize("hi,nn,nh,N", [(12, 70, 101, 64), (300, 33, 65, 64), (70000, 5, 40, 64),
                                         (12, 1100, 37, 64), (9, 20, 45, 16), (5, 9, 33, 128)])
def test_crss_distances_random_bit_exact(rici, oracle_mod, hi, nn, nh, N):
    """Spans needle chunks (1100 > 1024), ragged haystack tiles, the 64-bit path (values > 127,
    up to uint16 saturation), small and large N."""
    rng = np.random.default_rng(hi + nn)
    A = _rand_imgs(rng, nn, N=N, hi=min(hi, 65536), density=0.3)
    B = _rand_imgs(rng, nh, N=N, hi=min(hi, 65536), density=0.5)
    if hi > 65535:
        A[0, :, 1::2] = 65535
        B[1, :, 0::2] = 65535
    d = rici.rici_crss_distances(_dev(A), _dev(B)).cpu().numpy().view(np.uint64)
    assert np.array_equal(d, oracle_mod.crss_matrix(A, B))


def test_crss_pairs_and_count_below(rici, oracle_mod):
    rng = np.random.default_rng(5)
    A = _rand_imgs(rng, 50, density=0.1)
    B = _rand_imgs(rng, 300, density=0.4)
    pairs = np.stack([rng.integers(0, 50, 200), rng.integers(0, 300, 200)], 1).astype(np.int64)
    pairs[0] = [49, 299]
    got = rici.rici_crss_pairs(_dev(A), _dev(B), torch.from_numpy(pairs).to(DEV)).cpu().numpy().view(np.uint64)
    D = oracle_mod.crss_matrix(A, B)
    assert np.array_equal(got, D[pairs[:, 0], pairs[:, 1]])
    bad = torch.tensor([[0, 300]], dtype=torch.int64, device=DEV)           # device pairs: sentinel
    assert rici.rici_crss_pairs(_dev(A), _dev(B), bad).cpu().numpy().view(np.uint64)[0] == 2**64 - 1
    with pytest.raises(rici.RiciError):                                      # host pairs: error
        rici.rici_crss_pairs(_dev(A), _dev(B), np.array([[0, 300]], np.int64))
    thr = D[np.arange(50), rng.integers(0, 300, 50)]
    cnt = rici.rici_crss_count_below(_dev(A), _dev(B), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), oracle_mod.count_below(A, B, thr))


def test_ranks_c2_sampled_needles_full_haystack(rici, oracle_mod):
    """C2 self-search at full size on the GPU (the bench configuration); the oracle checks a
    sample of needles against the full 34,848-image haystack."""
    cfg = synth.config_c2()
    g = _gen(rici, cfg["mesh"], cfg["origins"], cfg["R"], cfg["N"])
    gd = _dev(g)
    ranks = rici.rici_crss_search(gd, gd).cpu().numpy()
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(g.shape[0], 24, replace=False))
    thr = np.array([oracle_mod.crss(g[i], g[i]) for i in idx], np.uint64)
    want = oracle_mod.count_below(g[idx], g, thr)
    assert np.array_equal(ranks[idx].astype(np.uint32), want)
    assert (ranks >= 0).all() and (ranks < g.shape[0]).all()


def test_ranks_ties_and_duplicates(rici, oracle_mod):
    rng = np.random.default_rng(7)
    A = _rand_imgs(rng, 40, N=64, hi=3, density=0.05)
    H = np.concatenate([A, A[::-1], _rand_imgs(rng, 29, hi=3, density=0.05)])   # duplicates -> ties
    r = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(A, H))


# ------------------------------------------------------------------ tensor-core path (N = 64)
def _mixed_images(rng, k, hi_small, n_big, big):
    a = _rand_imgs(rng, k, hi=hi_small, density=0.3)
    for q in rng.choice(k, n_big, replace=False):             # break the int8 guard
        a[q, rng.integers(0, 64), rng.integers(1, 64)] = big
    return a


@pytest.mark.parametrize("big", [16, 70, 300, 65535])
def test_crss_count_mma_guard_and_fallback(rici, oracle_mod, big):
    """Counts through the tcgen05 path: ragged M/N tiles (300 needles, 777 haystack images),
    images whose |D| breaks the int8 guard (|D_n| > 63 or |D_h| > 15) recounted by the SIMT
    path -- the union must equal the oracle exactly."""
    rng = np.random.default_rng(big)
    A = _mixed_images(rng, 300, 9, 7, big)
    H = np.concatenate([A, _mixed_images(rng, 477, 9, 11, big)])
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(300), rng.integers(0, H.shape[0], 300)].copy()
    rici.rici_crss_guard_stats(reset=True)
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))
    st = rici.rici_crss_guard_stats(reset=True)
    assert st["needles"] == 300 and st["haystack"] == 777
    dn = np.abs(np.diff(A.astype(np.int64), axis=2)).reshape(300, -1).max(1)
    dh = np.abs(np.diff(H.astype(np.int64), axis=2)).reshape(777, -1).max(1)
    assert st["needles_outside_guard"] == int((dn > 63).sum()) and st["haystack_outside_guard"] == int((dh > 15).sum())
    r = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(A, H))


def test_guard_fallback_many_haystack_images(rici, oracle_mod):
    """The haystack-side guard fallback keeps at most 20 guard-breaking haystack images resident
    per pass: 47 of them (three passes) against needles whose change lists overflow the
    512-entry per-warp list several times (density 0.3 -> ~2,000 changes per needle); counts and
    ranks must equal the oracle exactly."""
    rng = np.random.default_rng(2024)
    A = _mixed_images(rng, 260, 9, 3, 300)
    H = np.concatenate([A, _mixed_images(rng, 400, 9, 47, 40)])
    dh = np.abs(np.diff(H.astype(np.int64), axis=2)).reshape(H.shape[0], -1).max(1)
    assert int((dh > 15).sum()) >= 47
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(260), rng.integers(0, H.shape[0], 260)].copy()
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))
    r = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(A, H))


def test_more_needles_than_haystack(rici, oracle_mod):
    """Tensor path with more needle rows than haystack rows (the feature pass is then one
    launch in which every row stages both images): count_below of 700 needles (2:4 and dense
    subsets, one guard break) against 300 haystack images, exact against the oracle."""
    rng = np.random.default_rng(77)
    H = _mixed_images(rng, 300, 6, 2, 40)
    A = np.concatenate([H, _mixed_images(rng, 400, 6, 1, 300)])
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(700), rng.integers(0, 300, 700)].copy()
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))


def test_search_captured_in_cuda_graph(rici, oracle_mod):
    """No host synchronisation anywhere in rici_crss_search / count_below (tensor path with the
    device-sized dense subset and guard fallback): the calls capture into a CUDA graph, and the
    replay -- on new inputs copied into the same buffers -- equals the oracle."""
    rng = np.random.default_rng(91)
    A = _rand_imgs(rng, 600, hi=4, density=0.03)
    A[rng.choice(600, 40, replace=False)] = _rand_imgs(rng, 40, hi=6, density=0.5)   # not 2:4: dense pass
    A[3, 10, 20] = 300                                                          # guard break: fallback
    H = np.concatenate([A + (rng.random(A.shape) < 0.004).astype(np.uint16), _rand_imgs(rng, 500, hi=4, density=0.05)])
    H[700, 5, 9] = 40                                                           # haystack guard break
    nd, hd = _dev(A), _dev(H)
    out = torch.empty(600, dtype=torch.int32, device=DEV)
    rici.rici_crss_search(nd, hd, out=out)                                      # warm-up (caches, smem)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rici.rici_crss_search(nd, hd, out=out)
    A2 = A.copy()
    A2[::5] = H[600:720]                                                        # wrong matches: ranks > 0
    nd.copy_(_dev(A2))
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.uint32), oracle_mod.ranks(A2, H))
    assert out.max() > 0


def test_crss_guard_edges_exact(rici, oracle_mod):
    """The int8 guard at its edges: needle steps of exactly +-63 (largest -2 D_n that is s8; the
    change mask and sum D_n^2 come from those bytes) and +-64 (first outside: SIMT fallback),
    haystack steps of exactly +-15 (D_h^2 = 225, largest u8) and +-16 -- sparse, mixed with
    rows that break 2:4; counts and ranks equal the oracle."""
    rng = np.random.default_rng(63)
    A = _rand_imgs(rng, 520, hi=4, density=0.03)
    H = np.concatenate([A + (rng.random(A.shape) < 0.003).astype(np.uint16), _rand_imgs(rng, 300, hi=4, density=0.05)])
    for q, (r, c, v) in enumerate([(5, 10, 63), (7, 40, 64), (30, 2, 63), (31, 60, 64)]):
        A[q, r, c:] = v                                          # a +v step at c (and -v at 64 if c < 63)
        A[q + 4, r, c] = v                                       # +v then -v: two steps of magnitude v
    for q, (r, c, v) in enumerate([(9, 11, 15), (20, 33, 16), (40, 1, 15), (50, 62, 16)]):
        H[100 + q, r, c] = v
        H[200 + q, r, c:] = v
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(A.shape[0]), rng.integers(0, H.shape[0], A.shape[0])].copy()
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))
    r = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(A, H))
    d = rici.rici_crss_distances(_dev(A[:40]), _dev(H[:260])).cpu().numpy().view(np.uint64)
    assert np.array_equal(d, D[:40, :260])


def _band_copies(rng, A, rows, k):
    """Copies of needle images whose changes differ from the original only in `rows`."""
    out = A[rng.integers(0, A.shape[0], k)].copy()
    for img in out:
        r = rng.choice(rows)
        img[r, rng.integers(1, 64):] += np.uint16(rng.integers(1, 4))
    return out


@pytest.mark.parametrize("seed", [0, 1])
def test_rank_mode_tensor_pruning_exact(rici, oracle_mod, seed):
    """Rank mode on the tensor path: tiles are retired after the K prefixes of rows 24-39 and
    16-47 when every guard-valid pair's partial CRSS is already >= t_i.  The haystack mixes
    pairs that are ruled out by the first prefix, only by the second, only by the full K
    (differences outside rows 16-47), never (duplicates, ranks > 0), and guard-breaking
    images -- the ranks must equal full mode and the oracle exactly."""
    rng = np.random.default_rng(100 + seed)
    A = _mixed_images(rng, 520, 6, 5, 200)                      # ragged: 520 needles (5 M tiles)
    H = np.concatenate([
        A + (rng.random(A.shape) < 0.002).astype(np.uint16),      # true matches, small t_i > 0
        _band_copies(rng, A, list(range(24, 40)), 200),           # differ inside the first band
        _band_copies(rng, A, list(range(16, 24)) + list(range(40, 48)), 200),   # second band only
        _band_copies(rng, A, list(range(0, 16)) + list(range(48, 64)), 200),    # outside both
        A[rng.integers(0, 520, 60)],                              # exact duplicates
        _mixed_images(rng, 333, 6, 4, 40)])
    H = np.ascontiguousarray(H)
    full = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    rank = rici.rici_crss_search(_dev(A), _dev(H), early_exit=True).cpu().numpy()
    simt = rici.rici_crss_search(_dev(A), _dev(H), early_exit=True, simt=True).cpu().numpy()
    ref = oracle_mod.ranks(A, H)
    assert np.array_equal(full.astype(np.uint32), ref)
    assert np.array_equal(rank.astype(np.uint32), ref)
    assert np.array_equal(simt.astype(np.uint32), ref)
    assert ref.max() > 0 and (ref == 0).any()


def test_crss_paths_agree_subprocess(tmp_path):
    """The SIMT path (RICI_CRSS_PATH=simt) and the four tensor-core kernels (RICI_MMA_MODE 0:
    1-CTA, 1: 2-CTA multicast, 2: cta_group::2, 3: cta_group::2 with 2:4-sparse needle rows, one
    or two haystack tiles per staged needle block, RICI_SP_NT, or two needle m tiles per staged
    haystack block, RICI_SP_2M, with and without a haystack slice on the SMs the 4-CTA clusters
    leave free, RICI_SP_SIDE_FRAC) give identical ranks and counts, in
    full mode and in rank mode (early exit: tile pruning on K prefixes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, %r)\n"
        "import synth, paper_2007_02306_b200 as r\n"
        "m = synth.bumpy_torus(120, 60, key=(31,))\n"
        "mesh = r.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())\n"
        "im = r.rici_generate(mesh, torch.from_numpy(m.origins).cuda(), 0.3, 64)\n"
        "nee = im[:2000].clone(); nee[:, ::7, 5::9] += 1   # perturbed needles: thresholds > 0\n"
        "nee[1::2] = im[(torch.arange(1, 2000, 2, device='cuda') * 7 + 3) %% im.shape[0]]   # wrong matches: large ranks\n"
        "ranks = r.rici_crss_search(nee, im).cpu().numpy()\n"
        "pr = torch.stack([torch.arange(2000), (torch.arange(2000) * 7919) %% im.shape[0]], 1).cuda()\n"
        "thr = r.rici_crss_pairs(nee, im, pr)\n"
        "cnt = r.rici_crss_count_below(nee, im, thr).cpu().numpy()\n"
        "early = r.rici_crss_search(nee, im, early_exit=True).cpu().numpy()\n"
        "np.save(sys.argv[1], np.concatenate([ranks.astype(np.int64), cnt.astype(np.int64), early.astype(np.int64)]))\n") % root
    outs = {}
    for path, mode, nt, side, two_m in (("simt", "2", "2", "0", "0"), ("mma", "0", "2", "0", "0"),
                                        ("mma", "1", "2", "0", "0"), ("mma", "2", "2", "0", "0"),
                                        ("mma", "3", "1", "0", "0"), ("mma", "3", "2", "0", "0"),
                                        ("mma", "3", "1", "0.3", "0"), ("mma", "3", "2", "0.3", "0"),
                                        ("mma", "3", "2", "0", "1"), ("mma", "3", "2", "0.3", "1")):
        env = dict(os.environ, RICI_CRSS_PATH=path, RICI_MMA_MODE=mode, RICI_SP_NT=nt, RICI_SP_SIDE_FRAC=side,
                   RICI_SP_2M=two_m)   # RICI_SP_2M: two m tiles per sparse unit (kNM = 2)
        key = f"{path}{mode}_{nt}_{side}_{two_m}"
        f = str(tmp_path / f"{key}.npy")
        subprocess.run([sys.executable, "-c", code, f], env=env, check=True, timeout=600)
        outs[key] = np.load(f)
    ref = outs.pop("simt2_2_0_0")
    assert ref[:2000].max() > 0 and ref[2000:4000].max() > 0  # ranks and counts not trivially zero
    assert np.array_equal(ref[:2000], ref[4000:])            # rank mode (early exit) = full mode
    for k, v in outs.items():
        assert np.array_equal(ref, v), k


def _mini_c4(n_clutter=4, grid=(60, 30)):
    """C4-shaped: needles = a reference object alone, haystack = the cluttered scene with the
    reference placed first (so thresholds t_i > 0 and ranks are informative)."""
    objs = [synth.bumpy_torus(grid[0], grid[1], key=(41, k), minor=0.25 + 0.05 * k, amp=0.08)
            for k in range(1 + n_clutter)]
    sc = synth.clutterbox(objs, key=(41, 1000))
    n_ref = objs[0].n_vertices
    ref = synth.Mesh(sc.vertices[:n_ref].copy(), objs[0].indices.copy(), sc.normals[:n_ref].copy())
    return ref, sc


def test_rank_modes_identical_c4_shaped(rici, oracle_mod):
    """Full mode on the tensor cores, full mode on the SIMT path and rank mode with early exit
     give identical ranks; a sample is checked against the oracle."""
    ref, sc = _mini_c4()
    nd = _dev(_gen(rici, ref, ref.origins, 0.3, 64))
    hd = _dev(_gen(rici, sc, sc.origins, 0.3, 64))
    r_mma = rici.rici_crss_search(nd, hd).cpu().numpy()
    r_simt = rici.rici_crss_search(nd, hd, simt=True).cpu().numpy()
    r_early = rici.rici_crss_search(nd, hd, early_exit=True).cpu().numpy()
    assert np.array_equal(r_mma, r_simt) and np.array_equal(r_mma, r_early)
    assert r_mma.max() > 0                                  # clutter makes some ranks non-zero
    n = nd.cpu().numpy().view(np.uint16)
    h = hd.cpu().numpy().view(np.uint16)
    idx = np.random.default_rng(2).choice(n.shape[0], 48, replace=False)
    thr = np.array([oracle_mod.crss(n[i], h[i]) for i in idx], np.uint64)
    assert np.array_equal(r_mma[idx].astype(np.uint32), oracle_mod.count_below(n[idx], h, thr))


@pytest.mark.slow
def test_c3_clutterbox_full_size_sampled(rici, oracle_mod):
    """C3 (BASELINE configs[2]): 10 objects, 998,560 triangles, RICI at all 499,280 scene
    vertices on the GPU; the oracle checks a sample (incl. the last image) under the parity rule."""
    cfg = synth.config_c3()
    m = cfg["mesh"]
    assert m.n_triangles == 998_560 and m.n_vertices == 499_280
    g = _gen(rici, m, cfg["origins"], cfg["R"], cfg["N"])
    idx = np.sort(np.random.default_rng(3).choice(m.n_vertices, 2000, replace=False))
    idx[-1] = m.n_vertices - 1
    _parity_sampled(oracle_mod, g[idx], m, cfg["origins"][idx], cfg["R"], cfg["N"])


@pytest.mark.slow
def test_c4_full_size_ranks_sampled(rici, oracle_mod):
    """C4 (BASELINE configs[3]): 100,352 needles (reference alone) x 1,003,520 haystack images
    (reference placed first + 9 clutter objects) ranked on the tensor cores; the oracle recounts
    a sample of needles against the full haystack (bit-exact)."""
    cfg = synth.config_c4()
    ref, sc = cfg["reference"], cfg["scene"]
    assert ref.n_vertices == 100_352 and sc.n_vertices == 1_003_520
    nd = _dev(_gen(rici, ref, ref.origins, cfg["R"], cfg["N"]))
    hm = rici.rici_create_mesh(torch.from_numpy(sc.vertices).to(DEV), torch.from_numpy(sc.indices).to(DEV))
    hd = rici.rici_generate(hm, torch.from_numpy(sc.origins).to(DEV), cfg["R"], cfg["N"])
    ranks = rici.rici_crss_search(nd, hd).cpu().numpy()
    assert ranks.shape == (100_352,) and (ranks >= 0).all() and (ranks < 1_003_520).all()
    idx = np.random.default_rng(4).choice(100_352, 64, replace=False)       # 64 needles
    idx[0] = 100_351                                                         # the last needle
    n = nd.cpu().numpy().view(np.uint16)
    h = hd.cpu().numpy().view(np.uint16)
    thr = np.array([oracle_mod.crss(n[i], h[i]) for i in idx], np.uint64)
    assert np.array_equal(ranks[idx].astype(np.uint32), oracle_mod.count_below(n[idx], h, thr))
    # the 2M-triangle construction itself, under the parity rule: 500 haystack images (incl. the
    # last) and 500 needle images (the reference alone)
    hi = np.sort(np.random.default_rng(5).choice(sc.n_vertices, 500, replace=False))
    hi[-1] = sc.n_vertices - 1
    _parity_sampled(oracle_mod, h[hi], sc, sc.origins[hi], cfg["R"], cfg["N"])
    ni = np.sort(np.random.default_rng(6).choice(ref.n_vertices, 500, replace=False))
    _parity_sampled(oracle_mod, n[ni], ref, ref.origins[ni], cfg["R"], cfg["N"])


# ------------------------------------------------------------------ f4: Eq. 8 clutter fraction
def test_clutter_fraction_matches_oracle(rici, oracle_mod):
    ref, sc = _mini_c4(n_clutter=4)
    tag = np.zeros(sc.n_triangles, np.uint8)
    tag[:ref.n_triangles] = 1                                  # the reference object is placed first
    o = sc.origins[: ref.n_vertices]
    m = rici.rici_create_mesh(torch.from_numpy(sc.vertices).to(DEV), torch.from_numpy(sc.indices).to(DEV))
    frac, area = rici.rici_clutter_fraction(m, torch.from_numpy(tag).to(DEV), torch.from_numpy(o).to(DEV),
                                            0.3, 4, with_area=True)
    want, aa, _ = oracle_mod.clutter_fraction(sc.vertices, sc.indices, tag, o, 0.3, q=4)
    g = frac.cpu().numpy().astype(np.float64)
    a = area.cpu().numpy().astype(np.float64)
    assert np.abs(g - want).max() <= 2e-4
    assert np.abs(a - aa).max() <= 1e-4 * aa.max()
    assert (want > 0).any() and (want == 0).any()              # some vertices see clutter, some do not


def test_clutter_fraction_exact_cases(rici):
    m0 = synth.bumpy_torus(40, 20, key=(3,))
    V = np.concatenate([m0.vertices, m0.vertices])
    T = np.concatenate([m0.indices, m0.indices + m0.n_vertices])
    tag = np.concatenate([np.ones(m0.n_triangles, np.uint8), np.zeros(m0.n_triangles, np.uint8)])
    m = rici.rici_create_mesh(V, T)
    f = rici.rici_clutter_fraction(m, tag, m0.origins[::11], 0.3).cpu().numpy()
    assert np.allclose(f, 0.5, atol=1e-6)                     # a coincident duplicate is half the area
    m1 = rici.rici_create_mesh(m0.vertices, m0.indices)
    f1 = rici.rici_clutter_fraction(m1, np.ones(m0.n_triangles, np.uint8), m0.origins[::11], 0.3).cpu().numpy()
    assert (f1 == 0).all()


def test_streams_and_threads(rici):
    """Work enqueued on non-default streams, from two host threads at once, gives the same
    images and ranks as the default stream (stream-ordered workspace, thread-safe ABI state)."""
    import threading
    cfg = synth.config_c1()
    m = synth.bumpy_torus(80, 40, key=(17,))
    ref = _gen(rici, m, m.origins, 0.3, 64)
    ref_r = rici.rici_crss_search(_dev(ref), _dev(ref)).cpu().numpy()
    out = {}

    def work(tag):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).to(DEV), torch.from_numpy(m.indices).to(DEV),
                                         stream=st)
            im = rici.rici_generate(mesh, torch.from_numpy(m.origins).to(DEV), 0.3, 64, stream=st)
            r = rici.rici_crss_search(im, im, stream=st)
            st.synchronize()
            out[tag] = (im.cpu().numpy().view(np.uint16), r.cpu().numpy())
    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for t in range(2):
        assert np.array_equal(out[t][0], ref) and np.array_equal(out[t][1], ref_r)
    assert cfg["N"] == 64


def test_saturation_at_65535(rici, oracle_mod):
    """G9: counts saturate at 65535.  33,000 copies of a vertical quad give 66,000 crossings per
    pixel beyond rho = a; the int32 difference arrays stay exact and the store saturates.  The
    saturated images also exercise CRSS's exact 64-bit path (pixels > 127)."""
    q = synth.quad([[0.2, -5, -5], [0.2, 5, -5], [0.2, 5, 5], [0.2, -5, 5]])
    reps = 33_000
    V = np.tile(q.vertices, (reps, 1))
    T = (q.indices[None, :, :] + 4 * np.arange(reps)[:, None, None]).reshape(-1, 3).astype(np.int32)
    m = synth.Mesh(V, T, np.zeros_like(V))
    o = np.array([[0, 0, 0, 0, 0, 1], [0.01, 0.02, 0.0, 0.1, 0.0, 1.0]], np.float32)
    g = _gen(rici, m, o, 1.0, 64)
    want = oracle_mod.rici_generate(V, T, o, 1.0, 64)["images"]
    assert g.max() == 65535
    assert np.array_equal(g, want)
    d = rici.rici_crss_distances(_dev(g), _dev(g)).cpu().numpy().view(np.uint64)
    assert np.array_equal(d, oracle_mod.crss_matrix(g, g))
    r = rici.rici_crss_search(_dev(g), _dev(g)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(g, g))


def test_unaligned_image_buffers(rici, oracle_mod):
    """Image arrays that start 2 bytes past a 16-byte boundary (legal uint16 pointers) take the
    scalar paths and stay exact."""
    rng = np.random.default_rng(11)
    A = _rand_imgs(rng, 40, density=0.2)
    H = np.concatenate([A, _rand_imgs(rng, 50, density=0.3)])
    nbuf = torch.zeros(A.size + 1, dtype=torch.int16, device=DEV)
    hbuf = torch.zeros(H.size + 1, dtype=torch.int16, device=DEV)
    nbuf[1:] = _dev(A).reshape(-1)
    hbuf[1:] = _dev(H).reshape(-1)
    nv, hv = nbuf[1:].view(40, 64, 64), hbuf[1:].view(90, 64, 64)
    assert nv.data_ptr() % 16 == 2
    assert np.array_equal(rici.rici_crss_search(nv, hv).cpu().numpy().astype(np.uint32), oracle_mod.ranks(A, H))
    d = rici.rici_crss_distances(nv, hv).cpu().numpy().view(np.uint64)
    assert np.array_equal(d, oracle_mod.crss_matrix(A, H))


def test_kernel_timing_api(rici):
    """rici_set_kernel_timing / rici_kernel_time_ms: one event pair per launch of the timed
    kernels, on the launch stream; durations positive; the record clears on read."""
    cfg = synth.config_c1()
    m = cfg["mesh"]
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).to(DEV), torch.from_numpy(m.indices).to(DEV))
    o = torch.from_numpy(cfg["origins"]).to(DEV)
    rici.rici_kernel_time_ms(0), rici.rici_kernel_time_ms(1)
    rici.rici_set_kernel_timing(True)
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            imgs = [rici.rici_generate(mesh, o, cfg["R"], cfg["N"]) for _ in range(3)]
            rici.rici_crss_search(imgs[0], imgs[1])                # N = 64: one GEMM launch
    finally:
        rici.rici_set_kernel_timing(False)
    g_ms, g_n = rici.rici_kernel_time_ms(0)
    c_ms, c_n = rici.rici_kernel_time_ms(1)
    assert g_n == 3 and g_ms > 0 and c_n == 1 and c_ms > 0
    assert rici.rici_kernel_time_ms(0) == (0.0, 0)
    rici.rici_generate(mesh, o, cfg["R"], cfg["N"])                 # timing off: nothing recorded
    assert rici.rici_kernel_time_ms(0) == (0.0, 0)
    mesh.destroy()


def test_destroy_mesh_ordered_after_nonblocking_stream_use(rici):
    """rici_destroy_mesh right after an enqueued rici_generate on a non-blocking stream: the
    frees wait for that use (event recorded by the library), so memory the pool hands to a new
    mesh on another stream cannot be overwritten while the first generate still reads it."""
    cfg = synth.config_c2()
    m = cfg["mesh"]
    o = torch.from_numpy(cfg["origins"]).to(DEV)
    v, t = torch.from_numpy(m.vertices).to(DEV), torch.from_numpy(m.indices).to(DEV)
    ref_mesh = rici.rici_create_mesh(v, t)
    ref = rici.rici_generate(ref_mesh, o, 0.3, 64)
    torch.cuda.synchronize()
    ref_mesh.destroy()
    junk_v = torch.rand_like(v) * 10 - 5                        # a different mesh of the same size
    st = torch.cuda.Stream()                                     # torch streams are non-blocking
    outs = []
    for _ in range(3):
        with torch.cuda.stream(st):
            mesh = rici.rici_create_mesh(v, t, stream=st)
            out = rici.rici_generate(mesh, o, 0.3, 64, stream=st)
            mesh.destroy()                                       # no host wait before the free
        junk = rici.rici_create_mesh(junk_v, t)                  # may reuse the freed blocks
        junk.destroy()
        outs.append(out)
    torch.cuda.synchronize()
    for out in outs:
        assert torch.equal(out, ref)


def test_sparse_needle_path_mixed(rici, oracle_mod):
    """2:4-sparse tensor path (default RICI_MMA_MODE=3): sparse needle rows (D_n density ~2-3%,
    like the RICI workloads) mixed with rows that break the 2:4 structure (counted by the dense
    pass on the side stream) and rows that break the int8 guard (SIMT) -- 700 needles (6 M
    tiles, 4-CTA clusters with a ragged last cluster) against 1,300 haystack images; counts and
    ranks must equal the oracle."""
    rng = np.random.default_rng(77)
    A = _rand_imgs(rng, 700, hi=4, density=0.03)
    dense_rows = rng.choice(700, 60, replace=False)
    A[dense_rows] = _rand_imgs(rng, 60, hi=6, density=0.5)           # many > 2 per group: dense pass
    A[rng.choice(700, 5, replace=False), 10, 20] = 300               # guard break: SIMT
    H = np.concatenate([A + (rng.random(A.shape) < 0.004).astype(np.uint16), _rand_imgs(rng, 600, hi=4, density=0.05)])
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(700), rng.integers(0, H.shape[0], 700)].copy()
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))
    r = rici.rici_crss_search(_dev(A), _dev(H)).cpu().numpy()
    assert np.array_equal(r.astype(np.uint32), oracle_mod.ranks(A, H))


@pytest.mark.parametrize("nn,nh", [(900, 200), (513, 225), (513, 449), (1100, 671), (260, 1)])
def test_count_below_odd_shapes_sparse_path(rici, oracle_mod, nn, nh):
    """count_below through the default (2:4-sparse) tensor path with shapes that stress the
    tilings: more needles than haystack images, a haystack one past a 224 (and a 448) tile, a single
    haystack image; exact against the oracle."""
    rng = np.random.default_rng(nn + nh)
    A = _rand_imgs(rng, nn, hi=4, density=0.03)
    H = _rand_imgs(rng, nh, hi=4, density=0.03)
    D = oracle_mod.crss_matrix(A, H)
    thr = D[np.arange(nn), rng.integers(0, nh, nn)].copy() + rng.integers(0, 3, nn).astype(np.uint64)
    got = rici.rici_crss_count_below(_dev(A), _dev(H), torch.from_numpy(thr.view(np.int64)).to(DEV))
    assert np.array_equal(got.cpu().numpy().astype(np.int64), (D < thr[:, None]).sum(1))
