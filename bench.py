"""Benchmark of the RICI hot path (arXiv 2007.02306) on B200.

One step = one pass of the whole hot path over the C2 workload (BASELINE.json configs[1]):
  a1     rici_create_mesh   bumpy torus 264x132, T=69,696 triangles
  a2-a8  rici_generate      RICI 64x64 at all V=34,848 vertices, R=0.3
  a9-a12 rici_crss_search   every image as a needle against all images (self-search,
                            correspondence i <-> i): 34,848^2 = 1.21e9 CRSS comparisons
value = images (generated and ranked) per second for the whole job.  At N>1 GPUs (weak
scaling) each rank adds its own C2-sized object: rank r generates object r's images (its
haystack shard); the needles are rank 0's images (broadcast); thresholds and counts are
all-reduced over NCCL (paper_2007_02306_b200.dist).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
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


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` per launch, from the newest
    committed `ncu --set full` summary under profiles/ (r1*_ncu_summary.txt); None if absent."""
    import glob
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.txt")), reverse=True):
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


def ncu_metric(kernel, metric):
    """A metric of `kernel` from the newest committed ncu summary (profiles/r*_ncu_summary.txt)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.txt")), reverse=True):
        cur = None
        for line in open(path):
            if line.startswith("== "):
                cur = line[3:].strip()
            elif cur and cur.split("<")[0] == kernel and line.strip().startswith(metric + " ="):
                return float(line.split("=")[1].split()[0]), os.path.relpath(path, ROOT)
    return None, None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled every ~2 ms from
    a thread (the timed region is only tens of ms), nvidia-smi as a fallback."""

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


# ----------------------------------------------------------------------------- workload
def workload(rank: int):
    import synth
    cfg = synth.config_c2() if rank == 0 else {
        **synth.config_c2(), "mesh": synth.bumpy_torus(264, 132, key=(2, rank, 0))}
    if rank != 0:
        cfg["origins"] = cfg["mesh"].origins
    return cfg


def cpu_baseline(cfg, budget_s: float = 20.0):
    """The oracle as it stands on a bounded sample of the C2 step: generate a sample of the
    images and run CRSS of sampled needles against a sample of the haystack; extrapolate the
    step's time (n * t_image + n^2 * t_comparison) and report images/s of the step."""
    import oracle
    m = cfg["mesh"]
    n = m.n_vertices
    rng = np.random.default_rng(0)
    k_img = 512
    idx = np.sort(rng.choice(n, k_img, replace=False))
    t0 = time.perf_counter()
    imgs = oracle.rici_generate(m.vertices, m.indices, cfg["origins"][idx], cfg["R"], cfg["N"])["images"]
    t_gen = time.perf_counter() - t0
    per_img = t_gen / k_img
    # CRSS: needles x haystack from the generated sample (the oracle's dense loop cost is
    # data independent); scale the pair count to ~budget/2 seconds
    nn_s, nh_s = 32, k_img
    t0 = time.perf_counter()
    oracle.crss_matrix(imgs[:nn_s], imgs[:nh_s])
    t_c = time.perf_counter() - t0
    reps = max(1, int((budget_s / 2) / max(t_c, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.crss_matrix(imgs[:nn_s], imgs[:nh_s])
    t_c = (time.perf_counter() - t0) / reps
    per_cmp = t_c / (nn_s * nh_s)
    t_step = n * per_img + float(n) * n * per_cmp
    return {"value": n / t_step, "unit": "images/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": (f"oracle rici_generate of {k_img} sampled C2 images ({t_gen:.2f} s) + "
                       f"{reps}x oracle CRSS {nn_s}x{nh_s} ({t_c:.3f} s each); step time "
                       f"extrapolated as n*t_image + n^2*t_comparison for n={n}"),
            "t_image_s": per_img, "t_comparison_s": per_cmp, "t_step_s": t_step}


def segments_per_pair(cfg, k: int = 96) -> float:
    """S/P for the paper-literal construction work W = 43 P + 40 S + 3 N^2 n,
    from the oracle's segment counter on a fixed sample of images."""
    import oracle
    m = cfg["mesh"]
    idx = np.linspace(0, m.n_vertices - 1, k).astype(np.int64)
    r = oracle.rici_generate(m.vertices, m.indices, cfg["origins"][idx], cfg["R"], cfg["N"])
    return r["segments"] / float(k * m.n_triangles)


def run_reference(args):
    """--impl reference: the oracle timed as it stands on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workload(0)
    n = cfg["mesh"].n_vertices
    for _ in range(args.warmup):
        cpu_baseline(cfg, budget_s=2.0)
    vals = []
    cb = None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cb = cpu_baseline(cfg, budget_s=6.0)
        vals.append(cb["t_step_s"])
    wall = time.perf_counter() - t0
    t_step = float(np.mean(vals))
    value = n / t_step
    cbl = {k: cb[k] for k in ("unit", "cores", "kind", "sample")}
    cbl["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64/i64", "data": "synthetic",
            "config": {"workload": "C2: bumpy torus 264x132 (T=69,696), RICI 64x64 at all 34,848 "
                                   "vertices, R=0.3, CRSS self-search 34,848 x 34,848",
                       "bench_wall_s": wall},
            "cpu_baseline": cbl,
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2007_02306_b200 as rici
    from paper_2007_02306_b200 import dist as rdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rici._lib.load()

    cfg = workload(rank)
    m = cfg["mesh"]
    R, N = cfg["R"], cfg["N"]
    n = m.n_vertices
    v_d = torch.from_numpy(m.vertices).to(dev)
    t_d = torch.from_numpy(m.indices).to(dev)
    o_d = torch.from_numpy(cfg["origins"]).to(dev)
    imgs = torch.empty((n, N, N), dtype=torch.int16, device=dev)
    needles = torch.empty((workload(0)["mesh"].n_vertices if world > 1 else n, N, N), dtype=torch.int16, device=dev)
    ranks_d = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > L2 (126 MB)
    stream = torch.cuda.current_stream()

    ev = {k: [] for k in ("step", "mesh", "gen", "crss")}

    def step(record: bool):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(stream)
        mesh = rici.rici_create_mesh(v_d, t_d)
        e[1].record(stream)
        rici.rici_generate(mesh, o_d, R, N, out=imgs)
        e[2].record(stream)
        if world == 1:
            rici.rici_crss_search(imgs, imgs, out=ranks_d)
        else:
            if rank == 0:
                needles.copy_(imgs)
            rdist.broadcast_images(needles, 0)
            rdist.search_sharded(needles, imgs, rank * n, N)
        e[3].record(stream)
        mesh.destroy()
        if record:
            ev["step"].append((e[0], e[3]))
            ev["mesh"].append((e[0], e[1]))
            ev["gen"].append((e[1], e[2]))
            ev["crss"].append((e[2], e[3]))

    for _ in range(max(args.warmup, 0)):
        step(False)
        flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
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
    gen_kernel_ms, n_gen_k = rici.rici_kernel_time_ms(0)       # generate_kernel, per launch
    mma_kernel_ms, n_mma_k = rici.rici_kernel_time_ms(1)       # tcgen05 GEMM, per search call

    def ms(k):
        return float(np.mean([a.elapsed_time(b) for a, b in ev[k]]))

    step_ms, gen_ms, crss_ms, mesh_ms = ms("step"), ms("gen"), ms("crss"), ms("mesh")
    step_ms_max = step_ms
    if world > 1:
        t = torch.tensor([step_ms, gen_ms, crss_ms, gen_kernel_ms, mma_kernel_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms_max, gen_ms, crss_ms, gen_kernel_ms, mma_kernel_ms = [float(x) for x in t.cpu()]

    # ---- end-to-end through the public API with HOST buffers (every rank): mesh and origins
    # from pinned host memory (H2D inside the library), ranks back to host memory (D2H)
    vh = torch.from_numpy(m.vertices).pin_memory()
    th = torch.from_numpy(m.indices).pin_memory()
    oh = torch.from_numpy(cfg["origins"]).pin_memory()
    rh = torch.empty(needles.shape[0] if world > 1 else n, dtype=torch.int32).pin_memory()

    def e2e_step():
        mesh = rici.rici_create_mesh(vh, th)                     # H2D inside the library
        rici.rici_generate(mesh, oh, R, N, out=imgs)             # origins H2D inside
        if world == 1:
            rici.rici_crss_search(imgs, imgs, out=rh)            # ranks D2H + sync inside
        else:
            if rank == 0:
                needles.copy_(imgs)
            rdist.broadcast_images(needles, 0)
            rh.copy_(rdist.search_sharded(needles, imgs, rank * n, N).to(torch.int32))   # D2H
        mesh.destroy()
    for _ in range(2):
        e2e_step()
        flush.zero_()
    torch.cuda.synchronize()
    tt = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)                                          # device clock, like the step
        e2e_step()
        b.record(stream)                                          # after the ranks' D2H completed
        torch.cuda.synchronize()
        tt.append(a.elapsed_time(b) / 1e3)
        flush.zero_()
    e2e_ms = float(np.mean(tt)) * 1e3
    if world > 1:
        tmax = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        e2e_ms = float(tmax.item())
    e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "images/s",
           "h2d_bytes_per_step": int(vh.numel() * 4 + th.numel() * 4 + oh.numel() * 4),
           "d2h_bytes_per_step": int(rh.numel() * 4), "ms_per_step": e2e_ms,
           "note": "per rank; max over ranks" if world > 1 else "single GPU"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel: the tcgen05 int8 GEMM that ranks all pairs
    # (DESIGN.md 6.2).  Algorithmic ops per comparison = 2 x K with K = 2 x 4096 int8 features;
    # peak = the nominal dense int8 4.5 POPS (the measured-derived figures ride along).
    pk, src = peaks()
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    imgs_np = imgs.cpu().numpy().view(np.uint16)
    comparisons = float(imgs_np.shape[0]) * n                # per rank
    n_total_hay = n * world
    crss_s = crss_ms / 1e3
    mma = os.environ.get("RICI_CRSS_PATH", "") != "simt"
    sparse = mma and os.environ.get("RICI_MMA_MODE", "3") == "3"
    if mma and n_mma_k > 0:
        K = 2 * 4096
        kern_s = mma_kernel_ms / 1e3                               # the GEMM launches, live events
        achieved = comparisons * 2.0 * K / kern_s / 1e12          # logical int8 ops/s (Tops/s)
        # measured bf16 x the guide's nominal ratio for this dtype (dense int8 2x, 2:4 int8 4x)
        derived = (4.0 if sparse else 2.0) * pk.get("bf16_tflops", 1587.6)
        arch = SMS * 8192 * 2 * sm_mhz * 1e6 / 1e12                # 8192 int8 MAC/clk/SM at sm_max
        sp_rate = None
        try:
            with open(os.path.join(ROOT, "profiles", "int8_sparse_rate.json")) as f:
                sp_rate = json.load(f)["sparse"]["logical_tops"]
        except Exception:
            pass
        if sparse:   # 2:4-sparse needle operand: NVIDIA's doubled (sparse) figure is the ceiling
            peak = 9000.0
            kname = ("crss_mma_sp_kernel (tcgen05.mma.sp.cta_group::2.kind::i8, 2:4 needle rows, 4-CTA clusters "
                     "with B multicast) + the dense subset pass on a side stream")
        else:
            peak = 4500.0                                          # nominal dense int8 (guide table)
            kname = "crss_mma2_kernel (tcgen05.mma.cta_group::2.kind::i8, TMA, TMEM)"
        traffic, tsrc = ncu_traffic("crss_mma_sp_kernel" if sparse else "crss_mma2_kernel")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": tsrc,
                "kernel": kname,
                "kernel_ms": mma_kernel_ms, "kernel_launches_timed": n_mma_k,
                "timing": "CUDA events recorded by the library on the launch stream around each GEMM launch "
                          "in the timed region (rici_set_kernel_timing / rici_kernel_time_ms)",
                "frac_of_whole_search_call": comparisons * 2.0 * K / crss_s / 1e12 / peak,
                "dtype": "int8 (2:4-sparse needle rows) x int8 -> int32" if sparse else "int8 x int8 -> int32",
                "peak_source": ("nominal 2:4-sparse int8 9 POPS (2 x the dense 4.5 POPS of B200_PROFILING.md, whose "
                                "doubled vendor figures are the 2:4 ones); the measured sparse issue rate is "
                                "profiles/int8_sparse_rate.json" if sparse else
                                "nominal dense int8 4.5 POPS (B200_PROFILING.md table)") +
                               f".  The measured-derived figure (bf16 dense burst {pk.get('bf16_tflops', 1587.6)}"
                               f" x {4 if sparse else 2} = {derived:.0f}) and cuBLAS int8 (profiles/int8_peak.json) "
                               "are power-limited on random operands",
                "frac_vs_measured_sparse_rate": (achieved / sp_rate) if (sparse and sp_rate) else None,
                "dense_equivalent_frac_of_dense_peak": achieved / 4500.0,
                "frac_vs_measured_derived": achieved / derived,
                "frac_vs_arch_at_sm_max": achieved / arch,
                "algorithmic": f"2 x {K} int8 MACs per comparison x {comparisons:.0f} comparisons"}
        try:
            with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as f:
                roof["int8_cublas_measured_tops"] = json.load(f)["int8_tops_burst"]
        except Exception:
            pass
    else:
        d = np.diff(imgs_np.astype(np.int32), axis=2)
        nnz = int((d != 0).sum())
        terms = float(nnz) * n
        achieved = terms * CRSS_OPS_PER_TERM / crss_s / 1e12
        peak = SMS * LANES_PER_SM * sm_mhz * 1e6 / 1e12
        traffic, tsrc = ncu_traffic("crss_tile_kernel")
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
                "kernel": "crss_tile_kernel (SIMT; timed as the rici_crss_search call)",
                "peak_source": f"{SMS} SMs x {LANES_PER_SM} INT32 lanes x sm_max {sm_mhz} MHz ({src} clock)",
                "algorithmic": f"{CRSS_OPS_PER_TERM} int ops per masked term; {nnz} masked needle terms "
                               f"x {n} haystack images per rank"}
    roof["hbm_equivalent_frac"] = comparisons * 8192 / crss_s / 1e9 / pk.get("hbm_gbs", 6548.8)
    # the north star's own CRSS design (warp-cooperative integer streaming compare over the
    # needle change lists, ballot/popc rank) on the same images, outside the step
    simt_line = None
    if world == 1 and mma and not args.no_cpu_baseline:
        ts = []
        for it in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            a.record(stream)
            r_simt = rici.rici_crss_search(imgs, imgs, simt=True)
            b.record(stream)
            torch.cuda.synchronize()
            if it:
                ts.append(a.elapsed_time(b))
        d = np.diff(imgs_np.astype(np.int32), axis=2)
        terms = float(int((d != 0).sum())) * n
        t_s = float(np.mean(ts)) / 1e3
        simt_line = {"ms": t_s * 1e3, "comparisons_per_s": comparisons / t_s,
                     "ranks_equal_tensor_path": bool(torch.equal(r_simt.cpu(), ranks_d.cpu())),
                     "roofline": {"bound": "alu", "achieved": terms * CRSS_OPS_PER_TERM / t_s / 1e12,
                                  "peak": SMS * LANES_PER_SM * sm_mhz * 1e6 / 1e12, "unit": "Tops/s",
                                  "frac": terms * CRSS_OPS_PER_TERM / t_s / (SMS * LANES_PER_SM * sm_mhz * 1e6),
                                  "algorithmic": f"{CRSS_OPS_PER_TERM} int ops per masked needle term"},
                     "note": "rici_crss_search(simt=True), whole call, not part of the timed step"}
    images_per_s = n_total_hay / (step_ms_max / 1e3)
    spp = segments_per_pair(cfg)
    alu_peak = SMS * LANES_PER_SM * sm_mhz * 1e6 / 1e12
    P_pairs = float(n) * m.n_triangles
    W = 43.0 * P_pairs + 40.0 * spp * P_pairs + 3.0 * N * N * n
    construction = {"ms": gen_ms, "kernel_ms": gen_kernel_ms, "images_per_s": n / (gen_ms / 1e3),
                    "paper_literal_ops": W, "segments_per_pair": spp,
                    "paper_literal_frac": W / (gen_ms / 1e3) / (alu_peak * 1e12),
                    "note": "W = 43 P + 40 S + 3 N^2 n (brute-force pairs); the exact cull skips "
                            "provably-zero pairs, so this fraction can exceed 1"}
    issue, isrc = ncu_metric("generate_kernel", "smsp__issue_active.avg.pct_of_peak_sustained_active")
    if issue is not None:
        construction["issue_slot_utilisation"] = issue / 100.0
        construction["issue_source"] = isrc + " (ncu --set full; the kernel is issue-bound)"
    cb = cpu_baseline(cfg) if world == 1 and not args.no_cpu_baseline else None
    line = {"metric": METRIC, "value": images_per_s, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/i8",
            "data": "synthetic",
            "config": {"workload": "C2: bumpy torus 264x132 (T=69,696), RICI 64x64 at all 34,848 "
                                   "vertices, R=0.3, CRSS self-search 34,848 x 34,848"
                                   + ("" if world == 1 else f"; weak: {world} objects, haystack sharded"),
                       "images_per_rank": n, "comparisons_per_step": comparisons * world,
                       "l2": "flushed between timed steps (256 MB write); haystack 285 MB > L2",
                       "parallelism": f"dp{world}"},
            "comparisons_per_s": comparisons * world / (step_ms_max / 1e3),
            "construction": construction,
            "crss": {"ms": crss_ms, "comparisons_per_s": comparisons / crss_s},
            "mesh_staging_ms": mesh_ms,
            "crss_simt_path": simt_line,
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(), "bench_wall_s": wall}
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
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
