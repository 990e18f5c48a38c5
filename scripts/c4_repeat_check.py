"""Repeat the C4 full-mode search 20 times (and rank mode every 5th) and check the ranks never
change between calls: a race check of the asynchronous stage / accumulator barriers."""
import os, sys, hashlib
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, synth, paper_2007_02306_b200 as rici
cfg = synth.config_c4()
imgs = []
for m in (cfg["reference"], cfg["scene"]):
    mesh = rici.rici_create_mesh(torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.indices).cuda())
    imgs.append(rici.rici_generate(mesh, torch.from_numpy(m.origins).cuda(), 0.3, 64))
ref = rici.rici_crss_search(imgs[0], imgs[1]).clone()
ref_rank = rici.rici_crss_search(imgs[0], imgs[1], early_exit=True).clone()
bad = 0
for it in range(20):
    r = rici.rici_crss_search(imgs[0], imgs[1])
    bad += int(not torch.equal(r, ref))
    if it % 5 == 0:
        bad += int(not torch.equal(rici.rici_crss_search(imgs[0], imgs[1], early_exit=True), ref))
torch.cuda.synchronize()
print("mismatches", bad, "rank_mode_equal", bool(torch.equal(ref, ref_rank)), hashlib.sha1(ref.cpu().numpy().tobytes()).hexdigest()[:12])
