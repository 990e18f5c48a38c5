"""Small tensor-core CRSS count check against the oracle (run on the GPU box under `timeout`)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
import paper_2007_02306_b200 as rici  # noqa: E402


def imgs(rng, k, hi, density):
    a = rng.integers(0, hi, (k, 64, 64))
    a[rng.random((k, 64, 64)) > density] = 0
    return a.astype(np.uint16)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


rng = np.random.default_rng(0)
for (nn, nh, hi, dens) in [(130, 300, 6, 0.3), (300, 700, 9, 0.2), (64, 520, 40, 0.3)]:
    A = imgs(rng, nn, hi, dens)
    H = np.concatenate([A, imgs(rng, nh - nn, hi, dens)])
    D = oracle.crss_matrix(A, H)
    thr = D[np.arange(nn), rng.integers(0, nh, nn)].copy()
    t0 = time.time()
    got = rici.rici_crss_count_below(dev(A), dev(H), torch.from_numpy(thr.view(np.int64)).cuda())
    torch.cuda.synchronize()
    want = (D < thr[:, None]).sum(1)
    g = got.cpu().numpy().astype(np.int64)
    print(nn, nh, hi, "match", np.array_equal(g, want), "max diff", np.abs(g - want).max(), f"{time.time()-t0:.3f}s",
          flush=True)
