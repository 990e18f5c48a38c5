"""Time rici_crss_search on the C2 self-search (WORKLOAD=c4: the C4 search; RANK_MODE=1: early
exit) with the in-tree build; kernel knobs come from the environment (RICI_SP_NT, ...)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
for _ in range(2):
    r = rici.rici_crss_search(nee, hay, early_exit=early)
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
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("RICI_")},
                  "workload": os.environ.get("WORKLOAD", "c2"), "rank_mode": early,
                  "ms": float(np.median(ts)), "gemm_ms": km, "rank_sum": int(r.sum())}))
