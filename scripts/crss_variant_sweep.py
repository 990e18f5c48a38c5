"""CRSS tuning sweep: throwaway builds with -D defines (RICI_NVCC_DEFINES), each timing
rici_crss_search on the C2 self-search (images generated once per process)."""
import json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, sys, torch, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(1, sys.argv[2])
import os
import synth, paper_2007_02306_b200 as rici
def gen(m, o):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    return rici.rici_generate(mesh, torch.from_numpy(o).cuda(), 0.3, 64)
if os.environ.get("WORKLOAD") == "c4":
    c4 = synth.config_c4()
    nee, hay = gen(c4["reference"], c4["reference"].origins), gen(c4["scene"], c4["scene"].origins)
else:
    cfg = synth.config_c2()
    nee = hay = gen(cfg["mesh"], cfg["origins"])
early = os.environ.get("RANK_MODE") == "1"
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(2): r = rici.rici_crss_search(nee, hay, early_exit=early)
ts = []
rici.rici_kernel_time_ms(1)
rici.rici_set_kernel_timing(True)
for _ in range(int(os.environ.get("REPS", "10"))):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); r = rici.rici_crss_search(nee, hay, early_exit=early); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
rici.rici_set_kernel_timing(False)
km, kn = rici.rici_kernel_time_ms(1)
print(json.dumps({"ms": float(np.median(ts)), "gemm_ms": km, "rank_sum": int(r.sum())}))
'''
variants = sys.argv[1:] or [""]
dirs = {}
for v in variants:
    d = f"/tmp/rici_cvar_{abs(hash(v))}"
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2007_02306_b200"), os.path.join(d, "paper_2007_02306_b200"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
    defines, _, src = v.partition("@")        # "DEFINES@file.cu": file.cu replaces crss_mma.cu
    if src:
        shutil.copy(os.path.join(ROOT, src), os.path.join(d, "paper_2007_02306_b200", "csrc", "crss_mma.cu"))
    r = subprocess.run([sys.executable, os.path.join(d, "paper_2007_02306_b200", "build.py"), "--force"],
                       env=dict(os.environ, RICI_NVCC_DEFINES=defines), capture_output=True, text=True)
    if r.returncode:
        print(v, "BUILD FAILED", r.stderr[-400:]); continue
    dirs[v] = d
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for v, d in dirs.items():
        r = subprocess.run([sys.executable, "-c", CODE, d, ROOT], capture_output=True, text=True)
        print(json.dumps({"round": rnd, "defines": v, "res": r.stdout.strip(), "err": r.stderr.strip()[-200:]}), flush=True)
