"""Time rici_generate (kernel, live events) on C2, C3 and the C4 scene with the in-tree build;
prints one JSON line per workload with a checksum of the images.  WORKLOADS=c2,c3,c4."""
import hashlib, json, os, sys
sys.path.insert(0, os.environ.get("RICI_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2007_02306_b200 as rici

for w in os.environ.get("WORKLOADS", "c2,c3,c4").split(","):
    if w == "c4":
        m = synth.config_c4()["scene"]; o_np = m.origins
    elif w == "c3":
        cfg = synth.config_c3(); m = cfg["mesh"]; o_np = cfg["origins"]
    else:
        cfg = synth.config_c2(); m = cfg["mesh"]; o_np = cfg["origins"]
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    o = torch.from_numpy(o_np).cuda()
    out = torch.empty((o.shape[0], 64, 64), dtype=torch.int16, device="cuda")
    for _ in range(2):
        rici.rici_generate(mesh, o, 0.3, 64, out=out)
    torch.cuda.synchronize()
    rici.rici_kernel_time_ms(0)
    rici.rici_set_kernel_timing(True)
    reps = int(os.environ.get("REPS", "5"))
    for _ in range(reps):
        rici.rici_generate(mesh, o, 0.3, 64, out=out)
    rici.rici_set_kernel_timing(False)
    km, kn = rici.rici_kernel_time_ms(0)
    h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"workload": w, "images": int(o.shape[0]), "kernel_ms": km, "launches": kn,
                      "images_per_s": o.shape[0] / (km / 1e3), "sha": h,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("RICI_")}}), flush=True)
    del out, mesh
    torch.cuda.empty_cache()
