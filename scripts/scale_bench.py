"""C3/C4-shaped measurements beyond the C2 bench line (device-resident, CUDA events):
  * construction of a clutterbox scene (C3-shaped: n objects, all scene vertices),
  * CRSS rank search, needles = the reference object alone, haystack = the scene (C4-shaped),
    in full mode on the tensor cores, full mode on the SIMT kernel, and rank mode with early
    exit on the tensor path (tile pruning by K-prefix bounds) and on the SIMT kernel --
    all four must give identical ranks.
Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2007_02306_b200 as rici  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    out = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return out, float(np.median(ts))


ap = argparse.ArgumentParser()
ap.add_argument("--objects", type=int, default=10)
ap.add_argument("--grid", default="224,112")
ap.add_argument("--c4", action="store_true", help="the exact C4 config (synth.config_c4)")
a = ap.parse_args()
nu, nv = (int(x) for x in a.grid.split(","))
if a.c4:
    c4 = synth.config_c4()
    ref, sc = c4["reference"], c4["scene"]
    nu, nv = 448, 224
else:
    objs = [synth.bumpy_torus(nu, nv, key=(6, k), minor=0.2 + 0.025 * (k % 10), amp=0.08) for k in range(a.objects)]
    sc = synth.clutterbox(objs, key=(6, 1000))
    n_ref = objs[0].n_vertices
    ref = synth.Mesh(sc.vertices[:n_ref].copy(), objs[0].indices.copy(), sc.normals[:n_ref].copy())
dev = "cuda"
v, t, o = (torch.from_numpy(x).to(dev) for x in (sc.vertices, sc.indices, sc.origins))
mesh = rici.rici_create_mesh(v, t)
hay = torch.empty((sc.n_vertices, 64, 64), dtype=torch.int16, device=dev)
_, gen_ms = timed(lambda: rici.rici_generate(mesh, o, 0.3, 64, out=hay))
rm = rici.rici_create_mesh(torch.from_numpy(ref.vertices).to(dev), torch.from_numpy(ref.indices).to(dev))
nee = rici.rici_generate(rm, torch.from_numpy(ref.origins).to(dev), 0.3, 64)
cmp = float(nee.shape[0]) * hay.shape[0]
reps = 1 if a.c4 else 3
r_mma, t_mma = timed(lambda: rici.rici_crss_search(nee, hay), reps)
r_simt, t_simt = timed(lambda: rici.rici_crss_search(nee, hay, simt=True), reps)
r_early, t_early = timed(lambda: rici.rici_crss_search(nee, hay, early_exit=True), reps)
r_es, t_es = timed(lambda: rici.rici_crss_search(nee, hay, early_exit=True, simt=True), reps)
same = bool(torch.equal(r_mma, r_simt) and torch.equal(r_mma, r_early) and torch.equal(r_mma, r_es))
r = r_mma.cpu().numpy()
print(json.dumps({
    "scene": {"config": "C4" if a.c4 else "scaled", "objects": 10 if a.c4 else a.objects, "grid": [nu, nv],
              "triangles": sc.n_triangles, "vertices": sc.n_vertices},
    "construction": {"ms": gen_ms, "images_per_s": sc.n_vertices / gen_ms * 1e3},
    "search": {"needles": int(nee.shape[0]), "haystack": int(hay.shape[0]), "comparisons": cmp,
               "full_tensor": {"ms": t_mma, "comparisons_per_s": cmp / t_mma * 1e3},
               "full_simt": {"ms": t_simt, "comparisons_per_s": cmp / t_simt * 1e3},
               "rank_tensor_pruned": {"ms": t_early, "comparisons_per_s": cmp / t_early * 1e3},
               "rank_simt_early_exit": {"ms": t_es, "comparisons_per_s": cmp / t_es * 1e3},
               "ranks_identical": same, "rank0_fraction": float((r == 0).mean()),
               "median_rank": float(np.median(r))}}))
