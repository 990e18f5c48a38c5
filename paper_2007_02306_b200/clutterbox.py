"""Clutterbox experiment harness on synthetic objects.

The protocol, step by step:
  1. a clutterbox of side s (default 3);
  2. n objects drawn at random from an object set (here a pool of seeded synthetic bumpy tori
     instead of SHREC2017, which is not available);
  3. each normalised to the unit sphere;
  4. the reference object is object 0;
  5. reference descriptors {RD}: one RICI per unique vertex of the reference object alone;
  6. objects are placed one at a time (reference first), each at a uniform random rotation
     and a centre in [1, s-1]^3 (G15); after each configured clutter level the cluttered
     descriptors {CD} of the combined mesh are generated and every d in {RD} is ranked
     against {CD} -- the correspondence is vertex i <-> scene vertex i because the reference
     is placed first (G11); "lower ranks are better", ties take the best rank;
  7. one rank histogram per clutter level; the paper plots the rank-0 fraction.

All descriptor and rank work runs through the C ABI (rici_create_mesh / rici_generate /
rici_crss_search); this module only assembles scenes and histograms.

    python -m paper_2007_02306_b200.clutterbox --scenes 4 --levels 1,5,10 --grid 120,60
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)


def rank_histogram(ranks: np.ndarray, n_haystack: int) -> dict:
    """Histogram of ranks (bin i = how often the correct vertex was found at rank i),
    sparse: {rank: count}; plus the rank-0 fraction the paper plots."""
    r = np.asarray(ranks, dtype=np.int64)
    if r.size and (r.min() < 0 or r.max() > n_haystack - 1):
        raise ValueError("rank outside [0, |CD|-1] (P:388)")
    vals, cnts = np.unique(r, return_counts=True)
    return {"counts": {int(v): int(c) for v, c in zip(vals, cnts)}, "total": int(r.size),
            "rank0_fraction": float((r == 0).mean()) if r.size else 0.0}


_POOL: dict = {}


def object_pool(grid=(120, 60), size: int = 64):
    """The object set scenes draw from (the paper draws from SHREC2017's 383 objects):
    `size` seeded unit-sphere bumpy tori with varied minor radius, built once per grid."""
    import synth
    key = (tuple(grid), size)
    if key not in _POOL:
        objs = []
        for k in range(size):
            rng = synth.rng_for(5, k, 99)
            objs.append(synth.bumpy_torus(grid[0], grid[1], key=(5, k),
                                          minor=float(rng.uniform(0.2, 0.45)), amp=0.08))
        _POOL[key] = objs
    return _POOL[key]


def build_scene_objects(scene: int, n_objects: int, grid=(120, 60), pool_size: int = 64):
    """n distinct objects drawn at random (seeded per scene) from the object pool."""
    import synth
    pool = object_pool(grid, max(pool_size, n_objects))
    pick = synth.rng_for(5, scene, 77).choice(len(pool), n_objects, replace=False)
    return [pool[int(i)] for i in pick]


def clutter_rank_heatmap(clutter: np.ndarray, ranks: np.ndarray, n_clutter_bins: int = 10,
                         rank_edges=(0, 1, 2, 5, 10, 100, 1000, 10 ** 9)) -> dict:
    """2D histogram of (Eq. 8 clutter fraction bin, rank bin) -- the data behind the paper's
    clutter-vs-rank heatmap (fig:clutterComparison)."""
    c = np.clip(np.asarray(clutter, dtype=np.float64), 0.0, 1.0)
    cb = np.minimum((c * n_clutter_bins).astype(np.int64), n_clutter_bins - 1)
    rb = np.searchsorted(np.asarray(rank_edges[1:]), np.asarray(ranks, dtype=np.int64), side="right")
    H = np.zeros((n_clutter_bins, len(rank_edges) - 1), dtype=np.int64)
    np.add.at(H, (cb, rb), 1)
    return {"clutter_bins": n_clutter_bins, "rank_edges": list(rank_edges), "counts": H.tolist()}


def run_scene(scene: int, levels, grid=(120, 60), box_side: float = 3.0, R: float = 0.3, N: int = 64,
              generate=None, search=None, clutter=None):
    """One clutterbox run: returns {level: histogram} plus timing.  `generate(mesh, origins)` and
    `search(needles, haystack)` default to the CUDA library."""
    import synth
    if generate is None and search is None and clutter is None:
        return _run_scene_device(scene, levels, grid, box_side, R, N)
    if generate is None or search is None:
        import torch

        import paper_2007_02306_b200 as rici

        def generate(mesh, origins):  # noqa: F811
            m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
            out = rici.rici_generate(m, torch.from_numpy(origins).cuda(), R, N)
            m.destroy()
            return out

        def search(needles, haystack):  # noqa: F811
            # rank mode: only the ranks are needed; identical to full mode
            return rici.rici_crss_search(needles, haystack, early_exit=True).cpu().numpy()

        if clutter is None:
            def clutter(mesh, tag, origins):  # noqa: F811
                m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
                f = rici.rici_clutter_fraction(m, torch.from_numpy(tag).cuda(), torch.from_numpy(origins).cuda(), R)
                m.destroy()
                return f.cpu().numpy()
    levels = sorted(set(int(x) for x in levels))
    objs = build_scene_objects(scene, max(levels), grid)
    placed = synth.clutterbox(objs, key=(5, scene, 1000), box_side=box_side)
    n_ref = objs[0].n_vertices
    # {RD}: the reference object alone, in its placed pose (RICI is rigid-invariant)
    ref = synth.Mesh(placed.vertices[:n_ref].copy(), objs[0].indices.copy(), placed.normals[:n_ref].copy())
    t0 = time.perf_counter()
    rd = generate(ref, ref.origins)
    out = {"scene": scene, "n_reference_vertices": n_ref, "levels": {}}
    v_off = np.cumsum([0] + [o.n_vertices for o in objs])
    t_off = np.cumsum([0] + [o.n_triangles for o in objs])
    for lv in levels:
        nv, nt = int(v_off[lv]), int(t_off[lv])
        sc = synth.Mesh(placed.vertices[:nv], placed.indices[:nt], placed.normals[:nv])
        cd = generate(sc, sc.origins)                      # {CD} of the combined mesh
        ranks = search(rd, cd)
        h = rank_histogram(ranks, nv)
        if clutter is not None:                             # f4: Eq. 8 at every reference vertex
            tag = np.zeros(nt, np.uint8)
            tag[: objs[0].n_triangles] = 1
            cf = clutter(sc, tag, sc.origins[:n_ref])
            h["mean_clutter_fraction"] = float(np.mean(cf))
            h["clutter_rank_heatmap"] = clutter_rank_heatmap(cf, ranks)
        h.update({"n_objects": lv, "n_scene_vertices": nv, "n_scene_triangles": nt,
                  "comparisons": int(n_ref) * nv})
        out["levels"][lv] = h
    out["seconds"] = time.perf_counter() - t0
    return out


def _run_scene_device(scene: int, levels, grid, box_side: float, R: float, N: int):
    """run_scene with the CUDA library, device-resident: the placed scene (vertices, indices,
    oriented points) goes to the GPU once, and clutter level n is the prefix of the first n
    objects -- the reference first (G11) -- so each level's mesh, origins and triangle tags are
    slices of those buffers; one mesh per level serves construction and the Eq. 8 clutter
    fraction.  Same outputs as the generic path (tests/test_clutterbox.py)."""
    import synth
    import torch

    import paper_2007_02306_b200 as rici
    levels = sorted(set(int(x) for x in levels))
    objs = build_scene_objects(scene, max(levels), grid)
    placed = synth.clutterbox(objs, key=(5, scene, 1000), box_side=box_side)
    n_ref = objs[0].n_vertices
    V = torch.from_numpy(placed.vertices).cuda()
    T = torch.from_numpy(placed.indices).cuda()
    O = torch.from_numpy(placed.origins).cuda()
    tag_all = torch.zeros(placed.indices.shape[0], dtype=torch.uint8, device="cuda")
    tag_all[: objs[0].n_triangles] = 1
    t0 = time.perf_counter()
    # {RD}: the reference object alone (vertex and triangle prefix of the placed scene)
    m_ref = rici.rici_create_mesh(V[:n_ref], T[: objs[0].n_triangles])
    rd = rici.rici_generate(m_ref, O[:n_ref], R, N)
    m_ref.destroy()
    out = {"scene": scene, "n_reference_vertices": n_ref, "levels": {}}
    v_off = np.cumsum([0] + [o.n_vertices for o in objs])
    t_off = np.cumsum([0] + [o.n_triangles for o in objs])
    for lv in levels:
        nv, nt = int(v_off[lv]), int(t_off[lv])
        m = rici.rici_create_mesh(V[:nv], T[:nt])
        cd = rici.rici_generate(m, O[:nv], R, N)            # {CD} of the combined mesh
        ranks_d = rici.rici_crss_search(rd, cd, early_exit=True)   # rank mode
        cf_d = rici.rici_clutter_fraction(m, tag_all[:nt], O[:n_ref], R)   # f4: Eq. 8
        m.destroy()
        ranks, cf = ranks_d.cpu().numpy(), cf_d.cpu().numpy()
        h = rank_histogram(ranks, nv)
        h["mean_clutter_fraction"] = float(np.mean(cf))
        h["clutter_rank_heatmap"] = clutter_rank_heatmap(cf, ranks)
        h.update({"n_objects": lv, "n_scene_vertices": nv, "n_scene_triangles": nt,
                  "comparisons": int(n_ref) * nv})
        out["levels"][lv] = h
    out["seconds"] = time.perf_counter() - t0
    return out


def parse_levels(text: str):
    """'1,5,10' or '1-20' (inclusive range) or a mix: '1-5,10,20'."""
    out = []
    for part in text.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return sorted(set(out))


def main():
    """C5 (BASELINE configs[4]): S scenes x clutter levels.  Under torchrun the scenes are split
    over the ranks (independent problems, weak scaling); rank 0 gathers the histograms."""
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", type=int, default=2)
    ap.add_argument("--levels", default="1,5,10")
    ap.add_argument("--grid", default="120,60", help="torus grid per object (nu,nv)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    levels = parse_levels(a.levels)
    grid = tuple(int(x) for x in a.grid.split(","))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    from . import rici_crss_guard_stats
    rici_crss_guard_stats(reset=True)
    t0 = time.perf_counter()
    res = [run_scene(sc, levels, grid) for sc in range(rank, a.scenes, world)]
    wall = time.perf_counter() - t0
    gs = rici_crss_guard_stats(reset=True)          # this rank's tensor-path guard coverage
    guard = {"needles": gs["needles"], "haystack": gs["haystack"],
             "haystack_outside_int8_guard": gs["haystack_outside_guard"] / max(gs["haystack"], 1),
             "needles_outside_int8_guard": gs["needles_outside_guard"] / max(gs["needles"], 1),
             "needles_not_2_4": gs["needles_not_2_4"] / max(gs["needles"], 1)}
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (res, wall))
        res = [r for part, _ in gathered for r in part]
        wall = max(w for _, w in gathered)
        dist.destroy_process_group()
    if rank != 0:
        return
    res.sort(key=lambda r: r["scene"])
    summary = {lv: float(np.mean([r["levels"][lv]["rank0_fraction"] for r in res])) for lv in levels}
    clutter = {lv: float(np.mean([r["levels"][lv].get("mean_clutter_fraction", 0.0) for r in res])) for lv in levels}
    n_img = sum(r["levels"][lv]["n_scene_vertices"] for r in res for lv in levels) + sum(r["n_reference_vertices"] for r in res)
    n_cmp = sum(r["levels"][lv]["comparisons"] for r in res for lv in levels)
    doc = {"protocol": "clutterbox (P:379-391), synthetic tori", "levels": levels, "grid": grid,
           "scenes": a.scenes, "world_size": world, "wall_s": wall,
           "images_generated": n_img, "comparisons": n_cmp,
           "mean_rank0_fraction": summary, "mean_clutter_fraction": clutter, "guard_rank0": guard, "runs": res}
    txt = json.dumps(doc, indent=1, default=str)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)
    print(json.dumps({"scenes": a.scenes, "levels": [levels[0], levels[-1]], "world_size": world, "wall_s": wall,
                      "images_per_s": n_img / wall, "comparisons_per_s": n_cmp / wall,
                      "mean_rank0_fraction": summary, "mean_clutter_fraction": clutter, "guard_rank0": guard}))


if __name__ == "__main__":
    main()
