"""C4 needles + haystack (generated once) and one full-mode rici_crss_search (for ncu captures of
the search kernels at the bench's size).  EARLY_EXIT=1 runs rank mode instead."""
import os, sys
sys.path.insert(0, os.environ.get("RICI_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c4()
imgs = []
for m in (cfg["reference"], cfg["scene"]):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    imgs.append(rici.rici_generate(mesh, torch.from_numpy(m.origins).cuda(), cfg["R"], cfg["N"]))
    mesh.destroy()
for _ in range(int(os.environ.get("REPS", "1"))):
    ranks = rici.rici_crss_search(imgs[0], imgs[1], early_exit=os.environ.get("EARLY_EXIT") == "1")
torch.cuda.synchronize(); print("ok", int(ranks.max()), rici.rici_crss_guard_stats())
