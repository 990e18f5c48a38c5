"""C2 generate + two rici_crss_search calls (for ncu captures of the search kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
imgs = rici.rici_generate(mesh, o, 0.3, 64)
for _ in range(2): ranks = rici.rici_crss_search(imgs, imgs)
torch.cuda.synchronize(); print("ok", int(ranks.max()))
