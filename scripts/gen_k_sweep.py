import os, sys, subprocess, json
code = r'''
import os, sys, torch, numpy as np
sys.path.insert(0, %r)
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
out = torch.empty((m.n_vertices, 64, 64), dtype=torch.int16, device="cuda")
for _ in range(3): rici.rici_generate(mesh, o, 0.3, 64, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); rici.rici_generate(mesh, o, 0.3, 64, out=out); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(float(np.median(ts)), int(out.view(torch.uint16).sum()))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for kb in (16, 32, 48, 64, 80, 96, 128):
    env = dict(os.environ, RICI_GEN_SMEM_KB=str(kb))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(kb, "KB ->", r.stdout.strip(), r.stderr.strip()[-200:], flush=True)
