"""CRSS call time on C2 for several RICI_SP_SIDE_FRAC values (one process each, interleaved)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import sys, torch, numpy as np
sys.path.insert(0, %r)
import synth, paper_2007_02306_b200 as rici
import os
def gen(m, o):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    return rici.rici_generate(mesh, torch.from_numpy(o).cuda(), 0.3, 64)
if os.environ.get("WORKLOAD") == "c4":
    c4 = synth.config_c4()
    nee, hay = gen(c4["reference"], c4["reference"].origins), gen(c4["scene"], c4["scene"].origins)
    reps = 3
else:
    cfg = synth.config_c2()
    nee = hay = gen(cfg["mesh"], cfg["origins"])
    reps = 20
ref = rici.rici_crss_search(nee, hay, simt=os.environ.get("WORKLOAD") != "c4")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(2): r = rici.rici_crss_search(nee, hay)
ts = []
for _ in range(reps):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); r = rici.rici_crss_search(nee, hay); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(__import__("json").dumps({"ms": float(np.median(ts)), "same": bool(torch.equal(r, ref))}))
''' % ROOT
fracs = sys.argv[1:] or ["0", "0.03", "0.05", "0.08"]
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for f in fracs:
        r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, RICI_SP_SIDE_FRAC=f),
                           capture_output=True, text=True)
        print(json.dumps({"round": rnd, "frac": f, "res": r.stdout.strip(), "err": r.stderr.strip()[-300:]}), flush=True)
