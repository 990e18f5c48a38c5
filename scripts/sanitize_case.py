"""Small end-to-end run through every kernel (for compute-sanitizer): mesh staging, spatial
sort and kd chunk refinement, construction, thresholds, SIMT search (full + early exit),
tensor-core search with the guard fallback (2- and 4-CTA clusters, one and two haystack tiles
per unit, rank-mode prefix passes), distances, pairs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2007_02306_b200 as rici  # noqa: E402

m = synth.bumpy_torus(40, 20, key=(7,))
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(m.origins).cuda()
im = rici.rici_generate(mesh, o, 0.3, 64)
im30 = rici.rici_generate(mesh, o[:50], 0.3, 30)
h = im.clone()
h[5, 3, 7] = 200                                        # break the int8 guard on one image
r1 = rici.rici_crss_search(im[:300], h)
r2 = rici.rici_crss_search(im[:300], h, simt=True)
r3 = rici.rici_crss_search(im[:300], h, early_exit=True)
d = rici.rici_crss_distances(im[:40], h[:70])
p = rici.rici_crss_pairs(im, h, torch.tensor([[0, 1], [5, 5]], dtype=torch.int64).cuda())
r30 = rici.rici_crss_search(im30, im30)
tag = torch.zeros(m.n_triangles, dtype=torch.uint8, device="cuda")
tag[: m.n_triangles // 2] = 1
cf = rici.rici_clutter_fraction(mesh, tag, o[:64], 0.3)     # f4 (clutter.cu)
# a larger mesh: kd chunk refinement over several blocks, 4-CTA clusters with two tiles per
# unit (>= 512 needles), and (RICI_SP_SIDE_FRAC) the side slice
m2 = synth.bumpy_torus(80, 40, key=(8,))
mesh2 = rici.rici_create_mesh(torch.from_numpy(m2.vertices).cuda(), torch.from_numpy(m2.indices).cuda())
im2 = rici.rici_generate(mesh2, torch.from_numpy(m2.origins).cuda(), 0.3, 64)
nee = im2[:700].clone()
nee[1::2] = im2[(torch.arange(1, 700, 2, device="cuda") * 7 + 3) % im2.shape[0]]
r4 = rici.rici_crss_search(nee, im2)
r5 = rici.rici_crss_search(nee, im2, early_exit=True)
torch.cuda.synchronize()
assert torch.equal(r1, r2) and torch.equal(r1, r3) and torch.equal(r4, r5)
print("ok", int(r1.sum()), int(d.sum()), int(p.sum()), int(r30.sum()), int(r4.sum()), float(cf.sum()))
