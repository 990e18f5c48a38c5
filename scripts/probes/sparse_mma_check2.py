"""Probe 2: four accumulating 2:4 sparse int8 MMAs (K = 256 logical), metadata in TMEM via
tcgen05.st (mode 0) or tcgen05.cp from a core-matrix smem layout (mode 1, several LBO/SBO)."""
import ctypes
import json
import os

import numpy as np

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sparse_mma_check2.so"))
P = ctypes.c_void_p
rng = np.random.default_rng(1)
G = 64                                                    # groups of 4 per row (K = 256)
idx = np.sort(np.stack([rng.choice(4, 2, replace=False) for _ in range(128 * G)]).reshape(128, G, 2), axis=2)
vals = rng.integers(-20, 20, (128, G, 2)).astype(np.int8)
vals[vals == 0] = 3
Afull = np.zeros((128, 4 * G), np.int64)
for r in range(128):
    for g in range(G):
        for j in range(2):
            Afull[r, 4 * g + idx[r, g, j]] = vals[r, g, j]
B = rng.integers(-20, 20, (256, 4 * G)).astype(np.int8)
ref = Afull @ B.astype(np.int64).T
comp = np.ascontiguousarray(vals.reshape(128, 2 * G))     # 128 bytes per row
nib = (idx[:, :, 0] | (idx[:, :, 1] << 2)).astype(np.uint64)
meta = np.zeros((128, 8), np.uint32)
for g in range(G):
    w, sh = g // 8, 4 * (g % 8)
    meta[:, w] |= (nib[:, g] << np.uint64(sh)).astype(np.uint32)
meta = np.ascontiguousarray(meta)
res = {}
for mode, lbo, sbo in [(0, 0, 0), (1, 128, 256), (1, 256, 128), (1, 128, 128), (1, 2048, 128)]:
    C = np.zeros((128, 256), np.int32)
    rc = lib.run(comp.ctypes.data_as(P), np.ascontiguousarray(B).ctypes.data_as(P), meta.ctypes.data_as(P),
                 mode, lbo, sbo, C.ctypes.data_as(P))
    res[f"mode{mode}_lbo{lbo}_sbo{sbo}"] = {"rc": rc, "match": bool(np.array_equal(C, ref)),
                                            "frac_equal": float((C == ref).mean())}
print(json.dumps(res))
