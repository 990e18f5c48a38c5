"""Benchmark of the RICI hot path (arXiv 2007.02306) on B200.

One step = one pass of the whole hot path over the C4 workload (BASELINE.json configs[3],
"CRSS rank search: 100k needle images vs 1M haystack images"):
  a1     rici_create_mesh   the reference object alone (448x224 torus, T=200,704) and the
                            clutterbox scene (reference placed first + 9 clutter objects,
                            T=2,007,040)
  a2-a8  rici_generate      needles: RICI 64x64 at the 100,352 reference vertices;
                            haystack: RICI 64x64 at all 1,003,520 scene vertices (R=0.3)
  a9-a12 rici_crss_search   full mode: every needle against every haystack image,
                            1.007e11 CRSS comparisons, rank of the true correspondence i <-> i
value = images generated (and ranked) per second of the whole step; comparisons_per_s rides
along.  Extra keys: C3 construction (configs[2]), the C2 step (configs[1]).

At N > 1 GPUs the SAME scene is split (strong scaling): rank 0 builds the meshes
and broadcasts them (NCCL), every rank generates its contiguous block of the scene's oriented
points (its haystack shard) and of the reference's (all-gathered into the needle set), then
search_sharded: thresholds by the owner of h_i + all_reduce(MAX), local counts + all_reduce(SUM).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RICI images/s (64x64) and CRSS comparisons/s at 1/2/4/8 B200; % roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SMS = 148
LANES_PER_SM = 128          # FP32/INT32 lanes per SM
CRSS_OPS_PER_TERM = 3       # D_h difference, (D_n - D_h), multiply-accumulate
K_FEAT = 2 * 4096           # int8 feature length per image
WORKLOAD = ("C4 (BASELINE configs[3]): needles = RICI 64x64 at the 100,352 vertices of a 448x224 "
            "bumpy torus (T=200,704) alone; haystack = RICI 64x64 at all 1,003,520 vertices of a "
            "10-object clutterbox (reference placed first, T=2,007,040), R=0.3; full-mode CRSS "
            "search 100,352 x 1,003,520 = 1.007e11 comparisons, ranks of i <-> i")


def ncu_summaries():
    """Committed ncu summaries, the current one (named in profiles/ncu_current.txt) first, then
    the others newest name first."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary*.txt")), reverse=True)
    cur = os.path.join(ROOT, "profiles", "ncu_current.txt")
    if os.path.exists(cur):
        first = os.path.join(ROOT, "profiles", open(cur).read().strip())
        if first in paths:
            paths.remove(first)
            paths.insert(0, first)
    return paths


def ncu_metric(kernel, metric):
    """A metric of `kernel` from the current committed ncu summary (ncu_summaries())."""
    for path in ncu_summaries():
        cur = None
        for line in open(path):
            if line.startswith("== "):
                cur = line[3:].strip()
            elif cur and cur.split("<")[0] == kernel and line.strip().startswith(metric + " ="):
                return float(line.split("=")[1].split()[0]), os.path.relpath(path, ROOT)
    return None, None


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` per launch, from the newest
    committed `ncu --set full` summary under profiles/; None if absent."""
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for path in ncu_summaries():
        cur, tot, seen = None, 0.0, 0
        for line in open(path):
            if line.startswith("== "):
                cur = line[3:].strip()
            elif cur and cur.split("<")[0] == kernel and "dram__bytes_" in line:
                parts = line.split("=")[1].split()
                if len(parts) == 2 and parts[1] in scale:
                    tot += float(parts[0]) * scale[parts[1]]
                    seen += 1
        if seen == 2:
            return tot, os.path.relpath(path, ROOT) + " (cold-cache ncu replay, one launch)"
    return None, None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def host_cpu():
    """nproc and the lscpu model name of this host."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML polled every ~2 ms)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks = {k: getattr(pynvml, v) for k, v in self.REASONS.items()}

            def poll():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, m in masks.items():
                            if r & m:
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(0.002)
            self._nvml = pynvml
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 2 ms polling"}


# ----------------------------------------------------------------------------- oracle legs
def oracle_c4_sample(cfg, k_img: int, nn_cmp: int, haystack=None, nh_cmp: int | None = None,
                     needles=None):
    """Time the oracle as it stands (oracle/, all host cores) on a sample of the C4 step and
    extrapolate the step:  t_step = n_scene*t_scene_image + n_ref*t_ref_image + n_ref*n_scene*t_cmp.
    k_img scene and k_img reference images are generated by the oracle; CRSS runs nn_cmp
    needles against `haystack` (the full GPU-made haystack for the N=1 cpu_baseline, BASELINE.md
    section 3: 64 needles x 1,003,520) or, without one, the oracle's own sample images tiled to
    nh_cmp (the oracle's Eq. 7 loop costs the same for any uint16 input)."""
    import oracle
    ref, sc, R, N = cfg["reference"], cfg["scene"], cfg["R"], cfg["N"]
    rng = np.random.default_rng(0)
    si = np.sort(rng.choice(sc.n_vertices, k_img, replace=False))
    ri = np.sort(rng.choice(ref.n_vertices, k_img, replace=False))
    t0 = time.perf_counter()
    rs = oracle.rici_generate(sc.vertices, sc.indices, sc.origins[si], R, N)
    t_scene = (time.perf_counter() - t0) / k_img
    t0 = time.perf_counter()
    rr = oracle.rici_generate(ref.vertices, ref.indices, ref.origins[ri], R, N)
    t_ref = (time.perf_counter() - t0) / k_img
    if needles is None:
        needles = rr["images"][np.arange(nn_cmp) % k_img]
        thr_src = rs["images"][np.arange(nn_cmp) % k_img]
    else:
        idx = np.sort(rng.choice(needles.shape[0], nn_cmp, replace=False))
        needles = needles[idx]
        thr_src = haystack[idx]
    if haystack is None:
        haystack = rs["images"][np.arange(nh_cmp) % k_img]
    thr = np.array([oracle.crss(needles[i], thr_src[i]) for i in range(nn_cmp)], np.uint64)
    t0 = time.perf_counter()
    oracle.count_below(needles, haystack, thr)
    t_c = time.perf_counter() - t0
    t_cmp = t_c / (nn_cmp * haystack.shape[0])
    n_s, n_r = sc.n_vertices, ref.n_vertices
    t_step = n_s * t_scene + n_r * t_ref + float(n_r) * n_s * t_cmp
    spp = rs["segments"] / float(k_img * sc.n_triangles)
    spp_ref = rr["segments"] / float(k_img * ref.n_triangles)
    cpu = host_cpu()
    return {"value": (n_s + n_r) / t_step, "unit": "images/s", "cores": oracle.num_threads(),
            "kind": "oracle", "cpu_model": cpu["model"], "nproc": cpu["nproc"],
            "sample": (f"oracle rici_generate of {k_img} sampled C4 scene images ({t_scene * k_img:.2f} s) and "
                       f"{k_img} reference images ({t_ref * k_img:.2f} s); oracle count_below of {nn_cmp} needles "
                       f"x {haystack.shape[0]} haystack images ({t_c:.2f} s); step time EXTRAPOLATED as "
                       f"n_scene*t_scene_image + n_ref*t_ref_image + n_ref*n_scene*t_comparison"),
            "extrapolated": True,
            "t_scene_image_s": t_scene, "t_ref_image_s": t_ref, "t_comparison_s": t_cmp, "t_step_s": t_step,
            "comparisons_per_s": 1.0 / t_cmp, "segments_per_pair": spp, "segments_per_pair_ref": spp_ref}


def run_reference(args):
    """--impl reference: the oracle timed as it stands on the host cores (rank 0 only); each step
    is a bounded sample of the C4 step, extrapolated to the whole step (labelled)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    cfg = synth.config_c4()
    n = cfg["scene"].n_vertices + cfg["reference"].n_vertices
    for _ in range(args.warmup):
        oracle_c4_sample(cfg, 8, 16, nh_cmp=4096)
    vals, cb = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cb = oracle_c4_sample(cfg, 16, 64, nh_cmp=16384)
        vals.append(cb["t_step_s"])
    wall = time.perf_counter() - t0
    t_step = float(np.mean(vals))
    value = n / t_step
    cbl = {k: cb[k] for k in ("unit", "cores", "kind", "sample", "cpu_model", "nproc", "extrapolated")}
    cbl["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "ms_per_step_extrapolated": True,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/i64",
            "data": "synthetic",
            "comparisons_per_s": cb["comparisons_per_s"],
            "config": {"workload": WORKLOAD, "bench_wall_s": wall,
                       "note": "each timed step runs a bounded oracle sample; ms_per_step is extrapolated"},
            "cpu_baseline": cbl,
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- GPU arm
def _bcast_mesh_arrays(arrays, dev, world, rank):
    """Rank 0's host arrays -> device tensors on every rank (NCCL broadcast; the mesh is
    replicated)."""
    import torch
    import torch.distributed as dist
    out = []
    for a in arrays:
        if world == 1:
            out.append(torch.from_numpy(a).to(dev))
            continue
        meta = [a.shape if rank == 0 else None, str(a.dtype) if rank == 0 else None]
        dist.broadcast_object_list(meta, 0)
        t = torch.from_numpy(a).to(dev) if rank == 0 else torch.empty(meta[0], dtype=getattr(torch, meta[1]),
                                                                      device=dev)
        dist.broadcast(t, 0)
        out.append(t)
    return out


def extra_c3(rici, torch, dev, stream, flush, reps=3):
    """C3 (BASELINE configs[2]) construction: 10-object clutterbox, 998,560 triangles, RICI at
    all 499,280 vertices.  Mesh staging + rici_generate, device-resident, CUDA events."""
    import synth
    cfg = synth.config_c3()
    m = cfg["mesh"]
    v, t, o = (torch.from_numpy(x).to(dev) for x in (m.vertices, m.indices, cfg["origins"]))
    out = torch.empty((m.n_vertices, 64, 64), dtype=torch.int16, device=dev)
    ts = []
    for it in range(reps + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        mesh = rici.rici_create_mesh(v, t)
        rici.rici_generate(mesh, o, cfg["R"], cfg["N"], out=out)
        b.record(stream)
        mesh.destroy()
        torch.cuda.synchronize()
        if it:
            ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    del out
    return {"workload": "C3: 10 bumpy tori 316x158 in a clutterbox of side 3, T=998,560, RICI at all 499,280 "
                        "vertices", "ms": ms, "images_per_s": m.n_vertices / (ms / 1e3), "reps": reps}


def extra_gen_series(rici, torch, dev, stream, flush, levels=(1, 2, 4, 6, 8), reps=2):
    """Generation rate vs scene triangle count (fig:results_generation_rate): the C3
    clutterbox recipe with k objects (k = 10 is C3 itself, c3_construction), RICI at all
    vertices; mesh staging + rici_generate, device-resident, CUDA events."""
    import synth
    pts = []
    for k in levels:
        cfg = synth.config_c3(n_obj=k)
        m = cfg["mesh"]
        v, t, o = (torch.from_numpy(x).to(dev) for x in (m.vertices, m.indices, cfg["origins"]))
        out = torch.empty((m.n_vertices, 64, 64), dtype=torch.int16, device=dev)
        ts = []
        for it in range(reps + 1):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mesh = rici.rici_create_mesh(v, t)
            rici.rici_generate(mesh, o, cfg["R"], cfg["N"], out=out)
            b.record(stream)
            mesh.destroy()
            torch.cuda.synchronize()
            if it:
                ts.append(a.elapsed_time(b))
        ms = float(np.mean(ts))
        pts.append({"objects": k, "triangles": int(m.n_triangles), "images": int(m.n_vertices), "ms": ms,
                    "images_per_s": m.n_vertices / (ms / 1e3)})
        del out, v, t, o
    return {"workload": "C3 recipe (bumpy tori 316x158, clutterbox side 3) with k objects, RICI at all vertices; "
                        "the k = 10 point is c3_construction, the 2,007,040-triangle point the step's construction",
            "points": pts, "reps": reps}


def extra_c2(rici, torch, dev, stream, flush, reps=5, simt=True):
    """The round-1 C2 step (BASELINE configs[1]): mesh + RICI at all 34,848 vertices of the
    264x132 torus + CRSS self-search (1.21e9 comparisons); and the SIMT CRSS path on it."""
    import synth
    cfg = synth.config_c2()
    m = cfg["mesh"]
    n = m.n_vertices
    v, t, o = (torch.from_numpy(x).to(dev) for x in (m.vertices, m.indices, cfg["origins"]))
    imgs = torch.empty((n, 64, 64), dtype=torch.int16, device=dev)
    rk = torch.empty(n, dtype=torch.int32, device=dev)
    ts = {"step": [], "gen": [], "crss": []}
    for it in range(reps + 1):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        mesh = rici.rici_create_mesh(v, t)
        rici.rici_generate(mesh, o, cfg["R"], cfg["N"], out=imgs)
        e[1].record(stream)
        rici.rici_crss_search(imgs, imgs, out=rk)
        e[2].record(stream)
        mesh.destroy()
        torch.cuda.synchronize()
        if it:
            ts["step"].append(e[0].elapsed_time(e[2]))
            ts["gen"].append(e[0].elapsed_time(e[1]))
            ts["crss"].append(e[1].elapsed_time(e[2]))
    step = float(np.mean(ts["step"]))
    res = {"workload": "C2: bumpy torus 264x132 (T=69,696), RICI at all 34,848 vertices, CRSS self-search "
                       "34,848 x 34,848", "ms_per_step": step, "images_per_s": n / (step / 1e3),
           "construction_ms": float(np.mean(ts["gen"])), "crss_ms": float(np.mean(ts["crss"])),
           "comparisons_per_s": float(n) * n / (float(np.mean(ts["crss"])) / 1e3), "reps": reps}
    if simt:
        tt = []
        for it in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r_simt = rici.rici_crss_search(imgs, imgs, simt=True)
            b.record(stream)
            torch.cuda.synchronize()
            if it:
                tt.append(a.elapsed_time(b))
        d = torch.diff(imgs.to(torch.int32) & 0xFFFF, dim=2)
        terms = float(int((d != 0).sum())) * n
        t_s = float(np.mean(tt)) / 1e3
        pk = SMS * LANES_PER_SM * 1965.0 * 1e6
        res["crss_simt_path"] = {
            "ms": t_s * 1e3, "comparisons_per_s": float(n) * n / t_s,
            "ranks_equal_tensor_path": bool(torch.equal(r_simt, rk)),
            "roofline": {"bound": "alu", "achieved": terms * CRSS_OPS_PER_TERM / t_s / 1e12, "peak": pk / 1e12,
                         "unit": "Tops/s", "frac": terms * CRSS_OPS_PER_TERM / t_s / pk,
                         "algorithmic": f"{CRSS_OPS_PER_TERM} int ops per masked needle term"},
            "note": "the north star's SIMT streaming compare (DESIGN.md 6.3), rici_crss_search(simt=True)"}
    return res


def extra_rank_mode(rici, torch, needles, hay, ranks_full, stream, flush, reps=3):
    """The same C4 search in rank mode (RICI_CRSS_EARLY_EXIT: tiles retired once a K-prefix
    lower bound reaches t_i): identical ranks, fewer MMAs."""
    out = torch.empty_like(ranks_full)
    ts = []
    for it in range(reps + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rici.rici_crss_search(needles, hay, out=out, early_exit=True)
        b.record(stream)
        torch.cuda.synchronize()
        if it:
            ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    cmp = float(needles.shape[0]) * hay.shape[0]
    return {"ms": ms, "comparisons_per_s": cmp / (ms / 1e3), "ranks_equal_full_mode": bool(torch.equal(out, ranks_full)),
            "reps": reps, "note": "rici_crss_search(early_exit=True) on the step's needles and haystack"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2007_02306_b200 as rici
    from paper_2007_02306_b200 import dist as rdist
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rici._lib.load()

    cfg = synth.config_c4() if rank == 0 else None
    ref, sc = (cfg["reference"], cfg["scene"]) if rank == 0 else (None, None)
    R, N = 0.3, 64
    host = [ref.vertices, ref.indices, ref.origins, sc.vertices, sc.indices, sc.origins] if rank == 0 else [None] * 6
    rv, rt, ro, sv, st, so = _bcast_mesh_arrays(host, dev, world, rank)
    n_ref, n_sc = ro.shape[0], so.shape[0]
    lo_r, hi_r = rdist.shard_range(n_ref, world, rank)
    lo_h, hi_h = rdist.shard_range(n_sc, world, rank)
    needles = torch.empty((n_ref, N, N), dtype=torch.int16, device=dev)
    hay = torch.empty((hi_h - lo_h, N, N), dtype=torch.int16, device=dev)
    ranks_d = torch.empty(n_ref, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > L2 (126 MB)
    stream = torch.cuda.current_stream()
    ev = {k: [] for k in ("step", "needles", "hay", "crss")}

    def step(record: bool, src=None, out_ranks=None):
        v = src or (rv, rt, ro, sv, st, so)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(stream)
        m_ref = rici.rici_create_mesh(v[0], v[1])
        rdist.generate_sharded(m_ref, v[2], R, N, out=needles[lo_r:hi_r])
        rdist.all_gather_images(needles, n_ref)
        e[1].record(stream)
        m_sc = rici.rici_create_mesh(v[3], v[4])
        rdist.generate_sharded(m_sc, v[5], R, N, out=hay)
        e[2].record(stream)
        if world == 1:
            rici.rici_crss_search(needles, hay, out=ranks_d if out_ranks is None else out_ranks)
        else:
            r = rdist.search_sharded(needles, hay, lo_h, N)
            (ranks_d if out_ranks is None else out_ranks).copy_(r.to(torch.int32))
        e[3].record(stream)
        m_ref.destroy()
        m_sc.destroy()
        if record:
            ev["step"].append((e[0], e[3]))
            ev["needles"].append((e[0], e[1]))
            ev["hay"].append((e[1], e[2]))
            ev["crss"].append((e[2], e[3]))

    for _ in range(max(args.warmup, 0)):
        step(False)
        flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    rici.rici_crss_guard_stats(reset=True)
    launches0 = rici.rici_launch_count()
    for kid in (0, 1):                         # clear, then time the kernels' own launches live
        rici.rici_kernel_time_ms(kid)
    rici.rici_set_kernel_timing(True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step(True)
            flush.zero_()                      # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - t0
    launches = rici.rici_launch_count() - launches0
    rici.rici_set_kernel_timing(False)
    gs = rici.rici_crss_guard_stats(reset=True)
    guard = {"needles_outside_int8_guard": gs["needles_outside_guard"] / max(gs["needles"], 1),
             "haystack_outside_int8_guard": gs["haystack_outside_guard"] / max(gs["haystack"], 1),
             "needles_not_2_4": gs["needles_not_2_4"] / max(gs["needles"], 1),
             "note": "fractions over the timed searches: outside the guard -> exact SIMT fallback; "
                     "guard-valid but not 2:4 -> dense tcgen05 kernel on the side stream"}
    gen_kernel_ms, n_gen_k = rici.rici_kernel_time_ms(0)       # generate_kernel, per call (2 per step)
    mma_kernel_ms, n_mma_k = rici.rici_kernel_time_ms(1)       # tcgen05 GEMM launches, per search call

    def ms(k):
        return float(np.mean([a.elapsed_time(b) for a, b in ev[k]]))

    step_ms, nd_ms, hay_ms, crss_ms = ms("step"), ms("needles"), ms("hay"), ms("crss")
    local_step = step_ms
    if world > 1:
        t = torch.tensor([step_ms, nd_ms, hay_ms, crss_ms, mma_kernel_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, nd_ms, hay_ms, crss_ms, mma_kernel_ms = [float(x) for x in t.cpu()]

    # ---- end-to-end through the public API with HOST buffers: meshes and oriented points from
    # pinned host memory (H2D inside rici_create_mesh / rici_generate), ranks to pinned host memory
    hv = [torch.from_numpy(x.cpu().numpy()).pin_memory() for x in (rv, rt, ro, sv, st, so)]
    rh = torch.empty(n_ref, dtype=torch.int32).pin_memory()
    for _ in range(2):
        step(False, src=hv, out_ranks=rh)
        flush.zero_()
    torch.cuda.synchronize()
    tt = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step(False, src=hv, out_ranks=rh)
        b.record(stream)
        torch.cuda.synchronize()
        tt.append(a.elapsed_time(b))
        flush.zero_()
    e2e_ms = float(np.mean(tt))
    if world > 1:
        tmax = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        e2e_ms = float(tmax.item())
    h2d = int(sum(x.numel() * x.element_size() for x in (hv[0], hv[1], hv[3], hv[4]))
              + (hi_r - lo_r + hi_h - lo_h) * 24)
    e2e = {"value": (n_ref + n_sc) / (e2e_ms / 1e3), "unit": "images/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": int(rh.numel() * 4), "ms_per_step": e2e_ms,
           "note": ("per rank, max over ranks; " if world > 1 else "") +
                   "meshes + this rank's oriented points H2D inside the library calls, ranks D2H"}

    ranks_ok = None
    if world > 1:                              # ranks identical on every rank (all-reduced counts)
        chk = ranks_d.to(torch.int64).sum().reshape(1)
        allv = [torch.zeros_like(chk) for _ in range(world)]
        dist.all_gather(allv, chk)
        ranks_ok = all(int(x) == int(chk) for x in allv)
    rank0_frac = float((ranks_d == 0).float().mean())

    if rank != 0:
        dist.destroy_process_group()
        return

    pk, src = peaks()
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    comparisons = float(n_ref) * n_sc
    cmp_rank = float(n_ref) * (hi_h - lo_h)
    # ---- roofline of the CRSS GEMM: algorithmic ops = 2 x K int8 per comparison;
    # peak = measured bf16 burst x the guide's nominal ratio for 2:4-sparse int8 (x2 int8, x2 2:4)
    achieved = cmp_rank * 2.0 * K_FEAT / (mma_kernel_ms / 1e3) / 1e12 if n_mma_k else None
    peak = 4.0 * pk.get("bf16_tflops", 1590.0)
    sp_rate = None
    try:
        with open(os.path.join(ROOT, "profiles", "int8_sparse_rate.json")) as f:
            sp_rate = json.load(f)["sparse"]["logical_tops"]
    except Exception:
        pass
    traffic, tsrc = ncu_traffic("crss_mma_sp_kernel")
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic, "traffic_source": tsrc,
            "kernel": "crss_mma_sp_kernel (tcgen05.mma.sp.cta_group::2.kind::i8, 2:4 needle rows, 4-CTA clusters "
                      "with B multicast) + the dense subset and side slice on a side stream",
            "kernel_ms": mma_kernel_ms, "kernel_launches_timed": n_mma_k,
            "timing": "CUDA events recorded by the library on the launch stream around each search call's GEMM "
                      "launches in the timed region (rici_set_kernel_timing / rici_kernel_time_ms)",
            "peak_source": (f"{src} bf16 dense burst {pk.get('bf16_tflops')} TFLOP/s x 4 (int8 = 2x bf16, 2:4 "
                            f"sparsity = 2x dense: the B200_PROFILING.md nominal ratios)"),
            "frac_vs_sustained_derived": (achieved / (4.0 * pk["bf16_tflops_sustained"])
                                          if achieved and pk.get("bf16_tflops_sustained") else None),
            "frac_vs_nominal_9pops": achieved / 9000.0 if achieved else None,
            "frac_vs_probed_sparse_rate": (achieved / sp_rate) if (achieved and sp_rate) else None,
            "frac_of_whole_search_call": cmp_rank * 2.0 * K_FEAT / (crss_ms / 1e3) / 1e12 / peak,
            "dtype": "int8 (2:4-sparse needle rows) x int8 -> int32",
            "algorithmic": f"2 x {K_FEAT} int8 MACs per comparison x {cmp_rank:.0f} comparisons per rank",
            "hbm_equivalent_frac": cmp_rank * 8192 / (crss_ms / 1e3) / 1e9 / pk.get("hbm_gbs", 6548.8),
            "hbm_equivalent_note": "comparisons/s x 8192 B (the north star's streaming bytes) / measured HBM: "
                                   "the GEMM reuses each staged haystack row across 512 needles"}

    cb = None
    if world == 1 and not args.no_cpu_baseline:
        h_host = hay.cpu().numpy().view(np.uint16)
        n_host = needles.cpu().numpy().view(np.uint16)
        cfg_h = cfg
        cb = oracle_c4_sample(cfg_h, 64, 64, haystack=h_host, needles=n_host)
        del h_host, n_host

    alu_peak = SMS * LANES_PER_SM * sm_mhz * 1e6
    T_sc, T_ref = sc.n_triangles, ref.n_triangles
    P_pairs = float(n_sc) * T_sc + float(n_ref) * T_ref
    construction = {"ms": nd_ms + hay_ms, "needles_ms": nd_ms, "haystack_ms": hay_ms,
                    "images_per_s": (n_ref + n_sc) / ((nd_ms + hay_ms) / 1e3),
                    "haystack_images_per_s": n_sc / (hay_ms / 1e3),
                    "generate_kernel_ms_mean_per_call": gen_kernel_ms, "generate_calls_timed": n_gen_k,
                    "note": "events around mesh staging + generate (+ the needles' all-gather at N>1)"}
    if cb is not None:
        W = (43.0 * P_pairs + 40.0 * (cb["segments_per_pair"] * n_sc * T_sc + cb["segments_per_pair_ref"] * n_ref * T_ref)
             + 3.0 * N * N * (n_sc + n_ref))
        construction.update({"paper_literal_ops": W, "segments_per_pair": cb["segments_per_pair"],
                             "paper_literal_frac": W / ((nd_ms + hay_ms) / 1e3) / alu_peak,
                             "paper_literal_note": "W = 43 P + 40 S + 3 N^2 n over brute-force pairs P (P:123); "
                                                   "the exact cull skips provably-zero pairs, so this can exceed 1"})
    issue, isrc = ncu_metric("generate_kernel", "smsp__issue_active.avg.pct_of_peak_sustained_active")
    if issue is not None:
        construction["issue_slot_utilisation"] = issue / 100.0
        construction["issue_source"] = isrc + " (ncu --set full; the kernel is issue-bound)"

    extras = {}
    if world == 1 and not args.no_extras:
        extras["c4_rank_mode_search"] = extra_rank_mode(rici, torch, needles, hay, ranks_d, stream, flush)
        del hay
        torch.cuda.empty_cache()
        extras["c3_construction"] = extra_c3(rici, torch, dev, stream, flush)
        extras["generation_rate_series"] = extra_gen_series(rici, torch, dev, stream, flush)
        extras["c2_step"] = extra_c2(rici, torch, dev, stream, flush)
    images = n_ref + n_sc
    line = {"metric": METRIC, "value": images / (step_ms / 1e3), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/i8",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "images_per_step": images, "comparisons_per_step": comparisons,
                       "l2": "inputs > L2 (haystack 8.2 GB) and a 256 MB L2 flush between timed steps",
                       "parallelism": f"dp{world}: scene and reference vertices sharded, haystack sharded, "
                                      "needles all-gathered" if world > 1 else "single GPU"},
            "comparisons_per_s": comparisons / (step_ms / 1e3),
            "construction": construction,
            "crss": {"ms": crss_ms, "comparisons_per_s": comparisons / (crss_ms / 1e3), "mode": "full",
                     "rank0_fraction": rank0_frac, "ranks_identical_on_all_ranks": ranks_ok,
                     "guard": guard},
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(), "bench_wall_s": wall, "rank0_local_step_ms": local_step}
    line.update(extras)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rici", choices=["rici", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C3 / C2 extra keys")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
