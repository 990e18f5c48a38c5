"""Co-running probe at C4 size: the full-mode CRSS search (tensor cores) and the C4 scene's RICI
construction (SIMT, issue-bound) on two streams at once, against each alone.  The two are
independent here (the construction writes a second haystack buffer), so the overlap is the
upper bound of what a chunked generate -> search pipeline could hide.
RICI_PKG_ROOT=scratch/<variant> selects a build.  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.environ.get("RICI_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici

cfg = synth.config_c4()
meshes, origins, imgs = [], [], []
for m in (cfg["reference"], cfg["scene"]):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    o = torch.from_numpy(m.origins).cuda()
    meshes.append(mesh); origins.append(o)
    imgs.append(rici.rici_generate(mesh, o, cfg["R"], cfg["N"]))
hay2 = torch.empty_like(imgs[1])
ranks = torch.empty(imgs[0].shape[0], dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sa = torch.cuda.Stream(priority=-1)
sb = torch.cuda.Stream(priority=0)
frac = float(os.environ.get("GEN_FRAC", "1.0"))           # share of the scene's origins generated
n_gen = int(origins[1].shape[0] * frac)


def search():
    with torch.cuda.stream(sa):
        rici.rici_crss_search(imgs[0], imgs[1], out=ranks)


def gen():
    with torch.cuda.stream(sb):
        rici.rici_generate(meshes[1], origins[1][:n_gen], cfg["R"], cfg["N"], out=hay2[:n_gen])


def timed(parts, reps=3):
    ts = []
    for it in range(reps + 1):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in (sa, sb):
            s.wait_event(e0)
        for p in parts:
            p()
        for s in (sa, sb):
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


res = {"lib": rici.library_path(), "gen_frac": frac}
res["search_ms"] = timed([search])
ref = ranks.clone()
res["gen_ms"] = timed([gen])
res["corun_search_first_ms"] = timed([search, gen])
res["ranks_same"] = bool(torch.equal(ranks, ref))
res["images_same"] = bool(torch.equal(hay2[:n_gen], imgs[1][:n_gen]))
res["corun_gen_first_ms"] = timed([gen, search])
res["sum_ms"] = res["search_ms"] + res["gen_ms"]
print(json.dumps(res))
