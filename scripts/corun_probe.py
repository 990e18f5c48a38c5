"""Feasibility probe: can RICI construction co-run with the tcgen05 CRSS kernel on the same SMs?
Times (a) generate alone (K per RICI_GEN_SMEM_KB), (b) crss_search alone, (c) both, with the
search issued from a second host thread (its call synchronises once) on its own stream."""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici

cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
n = m.n_vertices
imgs = torch.empty((n, 64, 64), dtype=torch.int16, device="cuda")
rici.rici_generate(mesh, o, 0.3, 64, out=imgs)
out2 = torch.empty_like(imgs)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
torch.cuda.synchronize()

def gen(kb, stream):
    os.environ["RICI_GEN_SMEM_KB"] = str(kb)
    with torch.cuda.stream(stream):
        rici.rici_generate(mesh, o, 0.3, 64, out=out2)

def search(stream):
    with torch.cuda.stream(stream):
        return rici.rici_crss_search(imgs, imgs)

def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return float(np.median(ts))

res = {}
for kb in (34, 17):
    res[f"gen_kb{kb}"] = timed(lambda: gen(kb, s1))
res["search"] = timed(lambda: search(s2))
res["seq_kb34"] = timed(lambda: (gen(34, s1), torch.cuda.synchronize(), search(s2)))
for kb in (17, 34):
    for delay_ms in (0.3, 1.0):
        def both():
            th = threading.Thread(target=search, args=(s2,)); th.start()
            time.sleep(delay_ms / 1e3)
            gen(kb, s1)
            th.join()
        res[f"corun_kb{kb}_delay{delay_ms}"] = timed(both)
print(json.dumps(res))
