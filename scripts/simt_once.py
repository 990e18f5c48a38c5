"""C2 images once, then rici_crss_search(simt=True) twice (for ncu captures of crss_tile_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
imgs = rici.rici_generate(mesh, torch.from_numpy(cfg["origins"]).cuda(), 0.3, 64)
for _ in range(2): r = rici.rici_crss_search(imgs, imgs, simt=True)
torch.cuda.synchronize(); print("ok", int(r.sum()))
