"""Clutterbox harness: histogram logic on CPU with the oracle injected as
the compute, and the real CUDA path on the GPU."""
import numpy as np
import pytest

from paper_2007_02306_b200.clutterbox import rank_histogram, run_scene


def test_rank_histogram():
    h = rank_histogram(np.array([0, 0, 3, 1, 0]), 10)
    assert h["counts"] == {0: 3, 1: 1, 3: 1} and h["total"] == 5 and h["rank0_fraction"] == 0.6
    with pytest.raises(ValueError):
        rank_histogram(np.array([10]), 10)          # ranks live in [0, |CD|-1]


def test_scene_protocol_with_oracle(oracle_mod):
    """Level 1 = the reference alone: {CD} == {RD}, every self-distance is 0, so every rank is
    exactly 0 (SPEC AC7, exact self-match).  With clutter, histogram totals = |RD|."""
    R, N = 0.3, 64

    def generate(mesh, origins):
        return oracle_mod.rici_generate(mesh.vertices, mesh.indices, origins, R, N)["images"]

    def search(needles, haystack):
        return oracle_mod.ranks(needles, haystack)

    out = run_scene(0, [1, 3], grid=(24, 12), generate=generate, search=search)
    l1, l3 = out["levels"][1], out["levels"][3]
    assert l1["rank0_fraction"] == 1.0 and l1["total"] == out["n_reference_vertices"]
    assert l3["total"] == out["n_reference_vertices"] and l3["n_scene_vertices"] == 3 * 24 * 12
    assert sum(l3["counts"].values()) == l3["total"]


@pytest.mark.gpu
def test_scene_protocol_cuda():
    out = run_scene(1, [1, 4], grid=(64, 32))
    assert out["levels"][1]["rank0_fraction"] == 1.0
    assert 0.0 <= out["levels"][4]["rank0_fraction"] <= 1.0
    assert out["levels"][4]["total"] == 64 * 32


@pytest.mark.gpu
def test_device_resident_scene_path_equals_generic():
    """The device-resident harness path (scene uploaded once, levels as prefixes) gives the same
    histograms, clutter fractions and heatmaps as the generic per-level path on the library."""
    import torch
    import paper_2007_02306_b200 as rici
    R, N = 0.3, 64

    def generate(mesh, origins):
        m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
        out = rici.rici_generate(m, torch.from_numpy(origins).cuda(), R, N)
        m.destroy()
        return out

    def search(a, b):
        return rici.rici_crss_search(a, b, early_exit=True).cpu().numpy()

    def clutter(mesh, tag, origins):
        m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
        f = rici.rici_clutter_fraction(m, torch.from_numpy(tag).cuda(), torch.from_numpy(origins).cuda(), R)
        m.destroy()
        return f.cpu().numpy()

    fast = run_scene(3, [1, 2, 5], grid=(40, 20))
    slow = run_scene(3, [1, 2, 5], grid=(40, 20), generate=generate, search=search, clutter=clutter)
    for lv in (1, 2, 5):
        a, b = fast["levels"][lv], slow["levels"][lv]
        assert a["counts"] == b["counts"] and a["clutter_rank_heatmap"] == b["clutter_rank_heatmap"]
        assert a["mean_clutter_fraction"] == b["mean_clutter_fraction"]


def test_heatmap_counts():
    from paper_2007_02306_b200.clutterbox import clutter_rank_heatmap
    h = clutter_rank_heatmap(np.array([0.0, 0.05, 0.5, 0.99, 1.0]), np.array([0, 1, 3, 2000, 0]), 10)
    H = np.array(h["counts"])
    assert H.sum() == 5 and H[0, 0] == 1 and H[0, 1] == 1 and H[5, 2] == 1 and H[9, -1] == 1 and H[9, 0] == 1


def test_scene_with_clutter_fraction_oracle(oracle_mod):
    R, N = 0.3, 64
    out = run_scene(2, [1, 2], grid=(24, 12),
                    generate=lambda m, o: oracle_mod.rici_generate(m.vertices, m.indices, o, R, N)["images"],
                    search=lambda a, b: oracle_mod.ranks(a, b),
                    clutter=lambda m, tag, o: oracle_mod.clutter_fraction(m.vertices, m.indices, tag, o, R)[0])
    assert out["levels"][1]["mean_clutter_fraction"] == 0.0
    assert np.array(out["levels"][2]["clutter_rank_heatmap"]["counts"]).sum() == out["n_reference_vertices"]


@pytest.mark.gpu
def test_scene_cuda_against_oracle(oracle_mod):
    """f2 against the oracle: the harness runs on CUDA; at every clutter level the
    oracle recounts every rank from the GPU-made {RD} and {CD} (bit-exact), so the
    level's histogram is the oracle's; a sample of {RD} and {CD} images is checked against the
    oracle's construction under the parity rule; the Eq. 8 fractions against the oracle's."""
    import torch
    import paper_2007_02306_b200 as rici
    R, N = 0.3, 64
    made, searched = [], []

    def generate(mesh, origins):
        m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
        out = rici.rici_generate(m, torch.from_numpy(origins).cuda(), R, N)
        m.destroy()
        made.append((mesh, origins, out.cpu().numpy().view(np.uint16)))
        return out

    def search(a, b):
        r = rici.rici_crss_search(a, b, early_exit=True).cpu().numpy()
        searched.append((a.cpu().numpy().view(np.uint16), b.cpu().numpy().view(np.uint16), r))
        return r

    def clutter(mesh, tag, origins):
        m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
        f = rici.rici_clutter_fraction(m, torch.from_numpy(tag).cuda(), torch.from_numpy(origins).cuda(), R)
        m.destroy()
        # G17's inside test is a float decision at the cylinder wall, like a RICI bin edge: a
        # sub-triangle centroid within tau = 1e-5 R of the wall may go either way.  The GPU value
        # must lie in the oracle's bracket over R(1 - 1e-5), R, R(1 + 1e-5) (+1e-5 for float
        # accumulation) -- the same attribution width as the RICI parity rule
        w = [oracle_mod.clutter_fraction(mesh.vertices, mesh.indices, tag, origins, R * (1 + k * 1e-5))[0]
             for k in (-1, 0, 1)]
        lo, hi = np.minimum.reduce(w) - 1e-5, np.maximum.reduce(w) + 1e-5
        g = f.cpu().numpy().astype(np.float64)
        assert ((g >= lo) & (g <= hi)).all(), float(np.max(np.maximum(lo - g, g - hi)))
        return f.cpu().numpy()

    levels = [1, 3, 6]
    out = run_scene(4, levels, grid=(48, 24), generate=generate, search=search, clutter=clutter)
    assert len(searched) == len(levels)
    for lv, (rd, cd, ranks) in zip(levels, searched):
        want = oracle_mod.ranks(rd, cd)
        assert np.array_equal(ranks.astype(np.uint32), want)
        assert out["levels"][lv]["counts"] == rank_histogram(want, cd.shape[0])["counts"]
    assert out["levels"][6]["rank0_fraction"] < 1.0 or out["levels"][6]["mean_clutter_fraction"] > 0
    rng = np.random.default_rng(0)
    for mesh, origins, imgs in made:
        k = min(200, imgs.shape[0])
        idx = np.sort(rng.choice(imgs.shape[0], k, replace=False))
        ref = oracle_mod.rici_generate(mesh.vertices, mesh.indices, origins[idx], R, N, fragile=True)
        diff = imgs[idx] != ref["images"]
        assert not (diff & ~ref["fragile"]).any() and diff.mean() <= 1e-4
    # and the device-resident default path gives the same histograms
    fast = run_scene(4, levels, grid=(48, 24))
    for lv in levels:
        assert fast["levels"][lv]["counts"] == out["levels"][lv]["counts"]
