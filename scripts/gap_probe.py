"""Host/device timing of each C2 step phase (diagnostic)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2007_02306_b200 as rici

cfg = synth.config_c2()
m = cfg["mesh"]
v = torch.from_numpy(m.vertices).cuda(); t = torch.from_numpy(m.indices).cuda(); o = torch.from_numpy(cfg["origins"]).cuda()
imgs = torch.empty((m.n_vertices, 64, 64), dtype=torch.int16, device="cuda")
ranks = torch.empty(m.n_vertices, dtype=torch.int32, device="cuda")
for it in range(4):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h = [time.perf_counter()]
    ev[0].record(); mesh = rici.rici_create_mesh(v, t); h.append(time.perf_counter())
    ev[1].record(); rici.rici_generate(mesh, o, 0.3, 64, out=imgs); h.append(time.perf_counter())
    ev[2].record(); rici.rici_crss_search(imgs, imgs, out=ranks); h.append(time.perf_counter())
    ev[3].record(); torch.cuda.synchronize(); h.append(time.perf_counter())
    print("gpu ms", [round(ev[i].elapsed_time(ev[i+1]), 3) for i in range(3)],
          "host ms", [round((h[i+1]-h[i])*1e3, 3) for i in range(4)], flush=True)
    mesh.destroy()
