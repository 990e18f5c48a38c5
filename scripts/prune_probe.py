"""How often could a whole 256 x 256 CRSS tile be retired after a K-prefix?  (C4 rank mode.)
The partial CRSS over a row subset S is exactly CRSS(needle with rows outside S zeroed, h), a
lower bound of the full CRSS; a tile is prunable once every pair's partial >= t_i."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici

cfg = synth.config_c4()
R = cfg["R"]

def gen(mesh):
    m = rici.rici_create_mesh(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.indices).cuda())
    out = rici.rici_generate(m, torch.from_numpy(mesh.origins).cuda(), R, 64)
    m.destroy()
    return out

ref, sc = gen(cfg["reference"]), gen(cfg["scene"])
nn, nh = ref.shape[0], sc.shape[0]
tiles = [int(x) for x in np.linspace(0, nn // 256 - 1, 6)]
def pairs(js):
    return [r for j in js for r in (2 * j, 2 * j + 1)]
subsets = {"all": list(range(64)), "mid16": list(range(24, 40)), "mid24": list(range(20, 44)), "mid32": list(range(16, 48)),
           "lo16": list(range(0, 16)),
           "spread16": pairs(range(1, 32, 4)), "spread16b": pairs(range(2, 32, 4)),
           "midspread16": pairs([8, 10, 12, 14, 17, 19, 21, 23]),
           "spread32": pairs(range(0, 32, 2)), "mid8": list(range(28, 36)), "spread8": pairs(range(2, 32, 8))}
res = {"nn": nn, "nh": nh, "tiles": tiles, "frac_prunable": {k: [] for k in subsets}}
for t0 in tiles:
    nd = ref[t0 * 256:(t0 + 1) * 256].contiguous()
    idx = torch.arange(t0 * 256, (t0 + 1) * 256, device="cuda")
    thr = rici.rici_crss_pairs(nd, sc, torch.stack([torch.arange(256, device="cuda"), idx], 1))
    for name, rows in subsets.items():
        mask = torch.zeros(64, dtype=torch.bool, device="cuda"); mask[rows] = True
        nm = nd.clone(); nm[:, ~mask, :] = 0
        d = rici.rici_crss_distances(nm, sc)                       # [256, nh] int64
        below = (d < thr[:, None])                                  # pairs not yet ruled out
        nb = (nh + 255) // 256
        pad = nb * 256 - nh
        b = torch.nn.functional.pad(below, (0, pad)).reshape(256, nb, 256).any(2).any(0)
        res["frac_prunable"][name].append(float(1.0 - b.float().mean()))
        del d, below
    torch.cuda.empty_cache()
res["mean"] = {k: float(np.mean(v)) for k, v in res["frac_prunable"].items()}
print(json.dumps(res))
