"""Two rici_generate calls on C2 (for ncu captures).  RICI_PKG_ROOT selects a throwaway build."""
import os, sys
sys.path.insert(0, os.environ.get("RICI_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
for _ in range(2): out = rici.rici_generate(mesh, o, 0.3, 64)
torch.cuda.synchronize(); print("ok", rici.__file__)
