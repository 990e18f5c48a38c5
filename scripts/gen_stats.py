"""Construction work counters on C2 (a throwaway -DRICI_GEN_STATS=1 build in /tmp):
chunks visited, (image, triangle) pairs tested / queued / alpha-surviving, rows, segments."""
import ctypes, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = "/tmp/rici_stats"
if len(sys.argv) < 2:
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2007_02306_b200"), os.path.join(d, "paper_2007_02306_b200"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
    subprocess.run([sys.executable, os.path.join(d, "paper_2007_02306_b200", "build.py"), "--force"], check=True,
                   env=dict(os.environ, RICI_NVCC_DEFINES="-DRICI_GEN_STATS=1"), capture_output=True)
    sys.exit(subprocess.run([sys.executable, __file__, "run"]).returncode)
sys.path.insert(0, d); sys.path.insert(1, ROOT)
import torch
import synth, paper_2007_02306_b200 as rici
lib = ctypes.CDLL(os.path.join(d, "paper_2007_02306_b200", "librici.so"))
if os.environ.get("WORKLOAD") == "c3":            # the 10-object clutterbox scene
    cfg = synth.config_c3(); m = cfg["mesh"]
elif os.environ.get("WORKLOAD") == "c4":          # the C4 haystack scene
    m = synth.config_c4()["scene"]; cfg = {"origins": m.origins}
else:
    cfg = synth.config_c2(); m = cfg["mesh"]
mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
o = torch.from_numpy(cfg["origins"]).cuda()
buf = (ctypes.c_ulonglong * 13)()
rici.rici_generate(mesh, o, 0.3, 64); lib.rici_debug_gen_stats(buf, 1)
rici.rici_generate(mesh, o, 0.3, 64); lib.rici_debug_gen_stats(buf, 1)
n = m.n_vertices
names = ["chunk_visits", "chunk_image_pairs", "queued_pairs", "alpha_pass_pairs", "rows", "segments",
         "layer_loop_warp_iterations", "drains", "pairs_without_layer", "pairs_without_segment",
         "pairs_subchunk8_sphere_in_cylinder", "pairs_triangle_sphere_in_cylinder",
         "chunk_image_pairs_inside_radius"]
res = {k: buf[i] / n for i, k in enumerate(names)}
res["triangle_pairs_tested"] = res["chunk_image_pairs"] * 32
print(json.dumps({"per_image": res, "images": n}))
