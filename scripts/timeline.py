"""Kernel timeline of one C2 step (create_mesh + generate + search) from the torch profiler
(CUPTI activity records: start/end of every kernel on every stream) -- finds gaps and overlap.
WORKLOAD=c4: only the C4 search (images generated first, outside the profile); RANK=1 in rank mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import synth, paper_2007_02306_b200 as rici

if os.environ.get("WORKLOAD") == "c4step":          # the whole bench step (bench.py, N = 1)
    c4 = synth.config_c4()
    dev = [[torch.from_numpy(x).cuda() for x in (mm.vertices, mm.indices, mm.origins)] for mm in (c4["reference"], c4["scene"])]
    outs = [torch.empty((d[2].shape[0], 64, 64), dtype=torch.int16, device="cuda") for d in dev]
    ranks = torch.empty(outs[0].shape[0], dtype=torch.int32, device="cuda")

    def step():
        for d, o in zip(dev, outs):
            mesh = rici.rici_create_mesh(d[0], d[1])
            rici.rici_generate(mesh, d[2], 0.3, 64, out=o)
            mesh.destroy()
        rici.rici_crss_search(outs[0], outs[1], out=ranks)
elif os.environ.get("WORKLOAD") == "c4":
    c4 = synth.config_c4()
    gen = []
    for mm in (c4["reference"], c4["scene"]):
        mesh = rici.rici_create_mesh(torch.from_numpy(mm.vertices).cuda(), torch.from_numpy(mm.indices).cuda())
        gen.append(rici.rici_generate(mesh, torch.from_numpy(mm.origins).cuda(), 0.3, 64))
    ranks = torch.empty(gen[0].shape[0], dtype=torch.int32, device="cuda")

    def step():
        rici.rici_crss_search(gen[0], gen[1], out=ranks, early_exit=os.environ.get("RANK") == "1")
else:
    cfg = synth.config_c2(); m = cfg["mesh"]
    v, t, o = (torch.from_numpy(x).cuda() for x in (m.vertices, m.indices, cfg["origins"]))
    imgs = torch.empty((len(cfg["origins"]), 64, 64), dtype=torch.int16, device="cuda")
    ranks = torch.empty(len(cfg["origins"]), dtype=torch.int32, device="cuda")

    def step():
        mesh = rici.rici_create_mesh(v, t)
        rici.rici_generate(mesh, o, 0.3, 64, out=imgs)
        rici.rici_crss_search(imgs, imgs, out=ranks)
        mesh.destroy()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
allev = sorted(prof.events(), key=lambda e: e.time_range.start)
ev = [e for e in allev if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = ev[0].time_range.start
if os.environ.get("HOST"):                    # host-side runtime calls (CUPTI API records)
    for e in allev:
        if e.device_type != torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 3:
            print(f"HOST {e.time_range.start - t0:9.1f} us  +{e.time_range.elapsed_us():8.1f}  {e.name[:80]}")
last_end = t0
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.elapsed_us()
    gap = e.time_range.start - last_end
    print(f"{s:9.1f} us  +{d:8.1f}  gap {gap:7.1f}  {e.name[:90]}")
    last_end = max(last_end, e.time_range.end)
print("span", last_end - t0, "us")
