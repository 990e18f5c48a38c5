"""A/B timing of throwaway builds (scripts/build_variant.py -> scratch/<name>): each variant runs
in its own process, rounds alternate between variants.  MODE=search: the C4 full search (GEMM
launches timed by the library's events) + a rank checksum; MODE=gen: rici_generate on
WORKLOADS (c2,c3,c4) + an image checksum.   python scripts/variant_time.py scratch/a scratch/b ..."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import hashlib, json, os, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(1, sys.argv[2])
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici
assert rici.library_path().startswith(sys.argv[1]), rici.library_path()
mode, reps = os.environ.get("MODE", "search"), int(os.environ.get("REPS", "5"))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def gen(m, o, out=None):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    r = rici.rici_generate(mesh, torch.from_numpy(o).cuda(), 0.3, 64, out=out)
    return r, mesh
res = {}
if mode == "search":
    c4 = synth.config_c4()
    nee, _ = gen(c4["reference"], c4["reference"].origins)
    hay, _ = gen(c4["scene"], c4["scene"].origins)
    early = os.environ.get("RANK_MODE") == "1"
    for _ in range(2): r = rici.rici_crss_search(nee, hay, early_exit=early)
    ts = []
    rici.rici_kernel_time_ms(1); rici.rici_set_kernel_timing(True)
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); r = rici.rici_crss_search(nee, hay, early_exit=early); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rici.rici_set_kernel_timing(False)
    km, kn = rici.rici_kernel_time_ms(1)
    res = {"ms": float(np.median(ts)), "gemm_ms": km, "rank_sha": hashlib.sha1(r.cpu().numpy().tobytes()).hexdigest()[:12]}
else:
    for w in os.environ.get("WORKLOADS", "c2,c3,c4").split(","):
        if w == "c4":
            m = synth.config_c4()["scene"]; o = m.origins
        elif w == "c3":
            cfg = synth.config_c3(); m = cfg["mesh"]; o = cfg["origins"]
        else:
            cfg = synth.config_c2(); m = cfg["mesh"]; o = cfg["origins"]
        out = torch.empty((o.shape[0], 64, 64), dtype=torch.int16, device="cuda")
        for _ in range(2): _, mesh = gen(m, o, out)
        torch.cuda.synchronize()
        rici.rici_kernel_time_ms(0); rici.rici_set_kernel_timing(True)
        for _ in range(reps):
            flush.fill_(1.0)
            _, mesh = gen(m, o, out)
        rici.rici_set_kernel_timing(False)
        km, kn = rici.rici_kernel_time_ms(0)
        res[w] = {"kernel_ms": km, "sha": hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]}
        del out, mesh; torch.cuda.empty_cache()
print(json.dumps(res))
'''
dirs = sys.argv[1:]
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for d in dirs:
        r = subprocess.run([sys.executable, "-c", CODE, os.path.abspath(d), ROOT], capture_output=True, text=True)
        print(json.dumps({"round": rnd, "variant": os.path.basename(d.rstrip("/")), "res": r.stdout.strip(),
                          "err": r.stderr.strip()[-300:]}), flush=True)
