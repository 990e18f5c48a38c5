"""MMA-issuer / TMA-producer wait counters of the sparse GEMM on the C4 search (a throwaway
-DRICI_SP_PROF=1 build in scratch/sp_prof): fraction of the MMA issuer's cycles spent waiting
for a full stage, for a drained accumulator, and the producer's waits for an empty stage."""
import ctypes, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = os.path.join(ROOT, "scratch", "sp_prof")
if len(sys.argv) < 2:
    if not os.path.exists(os.path.join(d, "paper_2007_02306_b200", "librici.so")):
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "build_variant.py"), "sp_prof",
                        "-DRICI_SP_PROF=1 " + os.environ.get("EXTRA", "")], check=True)
    sys.exit(subprocess.run([sys.executable, __file__, "run"]).returncode)
sys.path.insert(0, d); sys.path.insert(1, ROOT)
import torch
import synth, paper_2007_02306_b200 as rici
lib = ctypes.CDLL(rici.library_path())
c4 = synth.config_c4()
imgs = []
for m in (c4["reference"], c4["scene"]):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    imgs.append(rici.rici_generate(mesh, torch.from_numpy(m.origins).cuda(), 0.3, 64))
buf = (ctypes.c_ulonglong * 8)()
rici.rici_crss_search(imgs[0], imgs[1]); lib.rici_debug_sp_prof(buf, 1)
rici.rici_crss_search(imgs[0], imgs[1]); torch.cuda.synchronize(); lib.rici_debug_sp_prof(buf, 1)
v = list(buf)
print(json.dumps({"producer_wait_empty": v[0], "mma_wait_full": v[1], "mma_wait_epilogue": v[2],
                  "mma_issuer_total": v[3], "stages": v[4], "drain_cycles_mean": v[5] / max(v[6], 1),
                  "cycles_per_unit": v[3] / max(v[4], 1) * 32 if v[4] else None,
                  "frac_wait_full": v[1] / max(v[3], 1), "frac_wait_epilogue": v[2] / max(v[3], 1)}))
