"""Construction tuning sweep: builds throwaway copies of the package with different -D defines
(RICI_NVCC_DEFINES) and times rici_generate on C2 for each, at several smem budgets."""
import json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys, torch, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(1, sys.argv[2])
import synth, paper_2007_02306_b200 as rici
cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
out = torch.empty((m.n_vertices, 64, 64), dtype=torch.int16, device="cuda")
for _ in range(3): rici.rici_generate(mesh, o, 0.3, 64, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); rici.rici_generate(mesh, o, 0.3, 64, out=out); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"ms": float(np.median(ts)), "sum": int(out.view(torch.uint16).sum())}))
'''.replace("json.dumps", "__import__('json').dumps")

variants = [v for v in sys.argv[1:]] or ["", "-DRICI_GEN_MIN_BLOCKS=5", "-DRICI_GEN_MIN_BLOCKS=6"]
budgets = [int(x) for x in os.environ.get("KB", "32,64").split(",")]
dirs = {}
for v in variants:
    d = f"/tmp/rici_var_{abs(hash(v))}"
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2007_02306_b200"), os.path.join(d, "paper_2007_02306_b200"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
    defines, _, src = v.partition("@")        # "DEFINES@file.cu": file.cu replaces generate.cu
    if src:
        shutil.copy(os.path.join(ROOT, src), os.path.join(d, "paper_2007_02306_b200", "csrc", "generate.cu"))
    env = dict(os.environ, RICI_NVCC_DEFINES=defines)
    r = subprocess.run([sys.executable, os.path.join(d, "paper_2007_02306_b200", "build.py"), "--force"],
                       env=env, capture_output=True, text=True)
    if r.returncode:
        print(v, "BUILD FAILED", r.stderr[-400:]); continue
    dirs[v] = d
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
  for v, d in dirs.items():
    for kb in budgets:
        env2 = dict(os.environ, RICI_GEN_SMEM_KB=str(kb))
        r = subprocess.run([sys.executable, "-c", CODE, d, ROOT], env=env2, capture_output=True, text=True)
        print(json.dumps({"round": rnd, "defines": v, "kb": kb, "res": r.stdout.strip(), "err": r.stderr.strip()[-200:]}), flush=True)
