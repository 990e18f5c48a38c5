import sys, torch
sys.path.insert(0, "/root/repo")
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
for _ in range(2): out = rici.rici_generate(mesh, o, 0.3, 64)
torch.cuda.synchronize(); print("ok")
