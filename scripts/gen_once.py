"""Two rici_generate calls (for ncu captures): C2 by default, WORKLOAD=c3 (10-object clutterbox)
or WORKLOAD=c4 (the C4 haystack scene).  RICI_PKG_ROOT selects a throwaway build."""
import os, sys
sys.path.insert(0, os.environ.get("RICI_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2007_02306_b200 as rici
w = os.environ.get("WORKLOAD", "c2")
if w == "c4":
    m = synth.config_c4()["scene"]; o_np = m.origins
elif w == "c3":
    cfg = synth.config_c3(); m = cfg["mesh"]; o_np = cfg["origins"]
else:
    cfg = synth.config_c2(); m = cfg["mesh"]; o_np = cfg["origins"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(o_np).cuda()
for _ in range(int(os.environ.get("REPS", "2"))):
    out = rici.rici_generate(mesh, o, 0.3, 64)
torch.cuda.synchronize(); print("ok", w, rici.__file__)
