"""Generate C2 (WORKLOAD env) images with several builds (scratch/<name>) and count differing
pixels against the first: python scripts/img_compare.py scratch/a scratch/b ..."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(1, sys.argv[2])
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici
w = os.environ.get("WORKLOAD", "c2")
if w == "c3":
    cfg = synth.config_c3(); m = cfg["mesh"]; o = cfg["origins"]
else:
    cfg = synth.config_c2(); m = cfg["mesh"]; o = cfg["origins"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
img = rici.rici_generate(mesh, torch.from_numpy(o).cuda(), 0.3, 64)
np.save(sys.argv[3], img.cpu().numpy().view(np.uint16))
'''
outs = []
for d in sys.argv[1:]:
    f = f"/tmp/img_{os.path.basename(d)}.npy"
    r = subprocess.run([sys.executable, "-c", CODE, os.path.abspath(d), ROOT, f], capture_output=True, text=True)
    if r.returncode:
        print(d, "FAILED", r.stderr[-500:]); continue
    outs.append((d, np.load(f)))
ref = outs[0][1]
for d, a in outs:
    diff = a != ref
    idx = np.argwhere(diff)
    print(d, "differing pixels", int(diff.sum()), "images", len(np.unique(idx[:, 0])) if len(idx) else 0,
          "first", idx[:5].tolist(), "vals", [(int(ref[tuple(i)]), int(a[tuple(i)])) for i in idx[:5]])
