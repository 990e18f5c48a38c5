"""C4 rank mode on the tensor path: time per choice of prune-check prefixes (bit mask: 1 = rows
28-35, 2 = rows 24-39, 4 = rows 16-47, 8 = rows 20-43) in RICI_RANK_PREFIXES (dense passes)
or, with PREFIX_VAR=RICI_RANK_PREFIXES_SP, in the 2:4-sparse passes (bits 2, 4 and 8)."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, sys, time, torch, numpy as np
sys.path.insert(0, %r)
import synth, paper_2007_02306_b200 as rici
c4 = synth.config_c4(); ref, sc = c4["reference"], c4["scene"]
def gen(m):
    mm = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    return rici.rici_generate(mm, torch.from_numpy(m.origins).cuda(), 0.3, 64)
nee, hay = gen(ref), gen(sc)
full = rici.rici_crss_search(nee, hay)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = rici.rici_crss_search(nee, hay, early_exit=True)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
print(json.dumps({"ms": float(np.median(ts)), "same": bool(torch.equal(r, full))}))
''' % ROOT
var = os.environ.get("PREFIX_VAR", "RICI_RANK_PREFIXES")
for mask in [int(x) for x in (sys.argv[1:] or ["6", "7", "2", "3", "4", "5", "1"])]:
    env = dict(os.environ, **{var: str(mask)})
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(json.dumps({"mask": mask, "res": r.stdout.strip(), "err": r.stderr.strip()[-300:]}), flush=True)
