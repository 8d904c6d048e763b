"""Benchmark: frames/s of the textured-2DGS render path (BASELINE configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "cfg2"): make_shell_scene(100000, T=8,
seed=3) with lobe_environment(default_rng(0), 64, 6), 800x800 views from the
bench_cameras orbit (256 views, each rank takes views r, r+N, ...). One step =
one frame: binning (preprocess, 32-bit depth-key one-sweep sort with the
fp64 run fix, duplication fused with the tile sort, ranges), K5 per-tile
textured compositor (atlas fetched by the texture units), K6 deferred
split-sum shading — one CUDA-graph replay per view. Scene, atlas and
environment are resident in HBM. `value`: K frames back to back between a
barrier + synchronize on both sides, CUDA events on the launch stream, max
over ranks (inputs larger than L2: the 205 MB atlas alone exceeds the 126 MB
L2). `breakdown_ms` / the roofline use a second pass with the L2 flushed
(256 MB write) before every frame. --batch-views B (cfg3: 256): one step =
the whole B-view orbit batch split over the ranks (strong scaling).

--impl reference times the reference's CPU implementation of the same path:
the C oracle port of texsplat's render_forward + shade_gbuffer (oracle/) on
all host threads, K steps after W warm-up frames. The numpy reference
itself (baseline/_ref) is timed inside the cpu_baseline leg on crop windows,
single-process and one process per core (`cpu_baseline.numpy_reference`).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec at 800×800 (100k textured 2DGS) 1–8 B200; % TEX/HBM peak"
WORKLOAD = ("cfg2 (BASELINE configs[1]): 100k textured 2D Gaussians, 8x8 texel atlas, 800x800, "
            "forward + deferred envmap shading")
CPU_BASELINE_NOTE = ("C oracle port of texsplat render_forward+shade_gbuffer (fp32, OpenMP over "
                     "tiles), the faster of the two CPU figures; the numpy reference itself is "
                     "timed on the same host in numpy_reference (single process and one "
                     "process per core)")


# BASELINE.json configs; cfg2 is the headline workload.
CONFIGS = {
    "cfg2": dict(splats=100_000, texture_res=8, width=800, height=800, env_height=64),
    "cfg3": dict(splats=500_000, texture_res=8, width=1920, height=1080, env_height=64,
                 batch_views=256),
    "cfg5": dict(splats=2_000_000, texture_res=16, width=1920, height=1080, env_height=128),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--splats", type=int, default=100_000)
    ap.add_argument("--texture-res", type=int, default=8)
    ap.add_argument("--width", type=int, default=800)
    ap.add_argument("--height", type=int, default=800)
    ap.add_argument("--sampler", default="hw", choices=["hw", "verify", "flat"])
    ap.add_argument("--texel-format", default="rgba32f", choices=["rgba32f", "rgba16f"])
    ap.add_argument("--tile", type=int, default=16)
    ap.add_argument("--env-height", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS),
                    help="BASELINE.json config preset (sets splats/texture/size/env)")
    ap.add_argument("--workload", default="render", choices=["render", "train"])
    ap.add_argument("--batch-views", type=int, default=0,
                    help="one step = a batch of this many orbit views over all ranks")
    ap.add_argument("--no-numpy-reference", action="store_true")
    ap.add_argument("--pipeline", type=int, default=6,
                    help="views in flight: independent workspaces on separate streams "
                         "(1 = one view at a time)")
    a = ap.parse_args()
    preset = CONFIGS[a.config]
    for k, v in preset.items():
        if getattr(a, k) == ap.get_default(k):
            setattr(a, k, v)
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10.0:
                time.sleep(0.05)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline_run(args, frames: int):
    """Oracle port render+shade on host cores; returns (fps, cores, sample)."""
    import numpy as np
    from oracle import oracle
    from paper_2506_13348_b200 import synth
    from paper_2506_13348_b200.environment import BrdfLut

    scene = synth.make_shell_scene(args.splats, args.texture_res, seed=3, with_environment=True,
                                   env_height=args.env_height)
    cams = synth.bench_cameras(256, args.width, args.height)
    lut = BrdfLut.build()
    atlas = oracle.pack(scene.texels)
    cores = oracle.cpu_threads()
    mode = "flat" if args.sampler == "flat" else "verify"
    # one untimed frame (page-in, thread-pool start)
    r = oracle.render(scene, cams[0], mode=mode, threads=cores, atlas=atlas)
    times = []
    for i in range(frames):
        cam = cams[i % len(cams)]
        t0 = time.perf_counter()
        r = oracle.render(scene, cam, mode=mode, threads=cores, atlas=atlas)
        oracle.shade(r["gbuf"], cam, scene.environment, lut.table, scene.background,
                     threads=cores)
        times.append(time.perf_counter() - t0)
    fps = len(times) / sum(times)
    sample = (f"{len(times)} full {args.width}x{args.height} frames of the same workload "
              f"(render_forward+shade_gbuffer), views 0..{len(times) - 1}")
    return fps, cores, sample, float(np.median(times))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle
    from paper_2506_13348_b200 import synth
    from paper_2506_13348_b200.environment import BrdfLut

    scene = synth.make_shell_scene(args.splats, args.texture_res, seed=3, with_environment=True,
                                   env_height=args.env_height)
    cams = synth.bench_cameras(256, args.width, args.height)
    lut = BrdfLut.build()
    atlas = oracle.pack(scene.texels)
    cores = oracle.cpu_threads()
    mode = "flat" if args.sampler == "flat" else "verify"

    def frame(cam):
        r = oracle.render(scene, cam, mode=mode, threads=cores, atlas=atlas)
        oracle.shade(r["gbuf"], cam, scene.environment, lut.table, scene.background,
                     threads=cores)

    for i in range(args.warmup):
        frame(cams[i % len(cams)])
    t0 = time.perf_counter()
    for i in range(args.steps):
        frame(cams[i % len(cams)])
    dt = time.perf_counter() - t0
    fps = args.steps / dt
    sample = (f"{args.steps} full {args.width}x{args.height} frames (render_forward+"
              f"shade_gbuffer), views 0..{args.steps - 1} after {args.warmup} warm-up frames")
    line = {
        "metric": METRIC, "value": round(fps, 6), "unit": "frames/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD if args.config == "cfg2" else
                   f"{args.config}: {args.splats} textured 2D Gaussians, {args.texture_res}x"
                   f"{args.texture_res} atlas, {args.width}x{args.height}",
                   "splats": args.splats, "texture_res": args.texture_res,
                   "width": args.width, "height": args.height,
                   "sampler": "fp32 bilinear (the reference's lerp_corners arithmetic)",
                   "texel_format": "rgba32f", "tile": args.tile,
                   "views": "bench_cameras(256) orbit, views 0.. in order",
                   "parallelism": f"{cores} host threads (OpenMP over tiles), rank 0 only"},
        "cpu_baseline": {"value": round(fps, 6), "unit": "frames/s", "cores": cores,
                         "kind": "port", "sample": sample, "note": CPU_BASELINE_NOTE},
        "e2e": {"value": round(fps, 6), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    del np
    print(json.dumps(line), flush=True)


def numpy_reference_timing(args, frags_frame: float, procs: int):
    """The numpy reference (baseline/_ref, texsplat itself) on crop windows
    of view 0: single process (3 windows) and `procs` processes at once (2
    windows each, one process per host core). A full frame is estimated per
    window as prepare + render x F_frame / F_window + shade x pixels ratio
    (crop windows are pixel-identical to the full frame)."""
    if not (ROOT / "baseline" / "_ref" / "texsplat").exists():
        return {"unavailable": "baseline/_ref/texsplat not installed"}
    W, H = args.width, args.height
    w = h = 96
    xs = [int(W * f) - w // 2 for f in (0.35, 0.5, 0.65)]
    ys = [int(H * f) - h // 2 for f in (0.35, 0.5, 0.65)]
    windows = [(x, y, w, h) for y in ys for x in xs]

    def launch(crops):
        cmd = [sys.executable, str(ROOT / "scripts" / "numpy_ref_worker.py"), str(args.splats),
               str(args.texture_res), str(W), str(H), str(args.env_height), "0"]
        cmd += [",".join(str(v) for v in c) for c in crops]
        return subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                text=True, env=dict(os.environ, OMP_NUM_THREADS="1",
                                                    OPENBLAS_NUM_THREADS="1"))

    def frame_s(rec):
        f = max(rec["fragments"], 1)
        return (rec["prepare_s"] + rec["render_s"] * frags_frame / f
                + rec["shade_s"] * (W * H) / (rec["crop"][2] * rec["crop"][3]))

    try:
        p = launch(windows[3:6])
        single = json.loads(p.communicate(timeout=600)[0].strip().splitlines()[-1])
        t_single = statistics.median(frame_s(r) for r in single)
        ps = [launch([windows[(2 * i) % 9], windows[(2 * i + 1) % 9]]) for i in range(procs)]
        par = []
        for q in ps:
            par += json.loads(q.communicate(timeout=900)[0].strip().splitlines()[-1])
        t_par = statistics.median(frame_s(r) for r in par)
    except Exception as e:  # noqa: BLE001 — report, do not fail the bench
        return {"unavailable": f"numpy reference run failed: {e!r}"[:200]}
    return {"fps_single_process": round(1.0 / t_single, 5),
            "fps_process_parallel": round(procs / t_par, 5), "cores": procs,
            "frame_s_single": round(t_single, 3), "frame_s_parallel_each": round(t_par, 3),
            "sample": f"texsplat (numpy, baseline/_ref) atlas-mode prepare + render_forward + "
                      f"shade_gbuffer of 96x96 windows of view 0, extrapolated to the "
                      f"{W}x{H} frame by fragment count ({frags_frame:.0f}); 3 windows single-"
                      f"process, {procs} processes x 2 windows at once"}


def run_train(args, scene, cams, lut, rank, world, dev):
    """cfg4: data-parallel training steps (forward + shade + loss + backward +
    bucketed all-reduce + Adam), each rank on its own views."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2506_13348_b200 import _lib, render_forward, shade_gbuffer
    from paper_2506_13348_b200.backward import splat_backward
    from paper_2506_13348_b200.rasterize import render_prepared
    from paper_2506_13348_b200.shading import shade_planar
    from paper_2506_13348_b200.training import (DataParallelTrainer, linear_to_display,
                                                partition_views)
    views = [cams[i] for i in partition_views(len(cams), rank, world)]
    nt = min(len(views), max(1, args.warmup + args.steps))
    targets = []
    for cam in views[:nt]:
        gb = render_forward(scene, cam, "perprim")
        targets.append(linear_to_display(shade_gbuffer(gb, cam, scene.environment, lut,
                                                       background=scene.background).color))
    init = scene.copy()
    init.positions = init.positions + 0.003
    tr = DataParallelTrainer(init, lut)
    for i in range(args.warmup):
        tr.step(views[i % nt], targets[i % nt])
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        terms, _ = tr.step(views[i % nt], targets[i % nt])
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    n_adam = (len(tr._single_launches()) if world == 1
              else sum(1 for _, _, n, _ in tr._launches if n))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # ---- e2e: the public step with host data every step --------------------
    # target image copied from pinned host memory, loss read back, per step
    host_tgts = [tg.cpu().pin_memory() for tg in targets]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss_sum = 0.0
    for i in range(args.steps):
        tgt = host_tgts[i % nt].to(dev, non_blocking=True)
        terms_i, _ = tr.step(views[i % nt], tgt)
        loss_sum += terms_i["loss"]  # D2H of the step's loss terms
    e2e_s = time.perf_counter() - t0
    clk = clocks.stop()
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = world * args.steps / float(te.item())

    # ---- roofline of the dominant kernel: K8 (k_raster_bwd) ---------------
    # K8 alone on view 0 (events around splat_backward), the global atomic
    # adds it issues (device counter), and the RED throughput peak measured
    # live with tsb_red_probe (scattered float adds, L2-resident buffer)
    L = _lib.lib()
    cam0, tgt0 = views[0], targets[0]
    H, W = int(cam0.height), int(cam0.width)
    tr.grads_and_loss(cam0, tgt0)
    gbuf, tape = render_prepared(tr.prep, cam0, tr.tile, check=True)
    dg = torch.randn((13, H, W), dtype=torch.float32, device=dev) * 1e-3
    for _ in range(2):
        splat_backward(None, cam0, tr.prep, tape, dg, grads=tr.grads, scratch=tr.bwd_scratch)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kr = 5
    torch.cuda.synchronize()
    k0.record()
    for _ in range(kr):
        splat_backward(None, cam0, tr.prep, tape, dg, grads=tr.grads, scratch=tr.bwd_scratch)
    k1.record()
    torch.cuda.synchronize()
    k8_ms = k0.elapsed_time(k1) / kr
    cnt = C.c_ulonglong()
    _lib.check(L.tsb_debug_red_count(1, None), "red count")
    splat_backward(None, cam0, tr.prep, tape, dg, grads=tr.grads, scratch=tr.bwd_scratch)
    torch.cuda.synchronize()
    _lib.check(L.tsb_debug_red_count(0, C.byref(cnt)), "red count")
    reds = int(cnt.value)
    fragments = int(gbuf.pixels.n_contrib.sum(dtype=torch.int64).item())
    pbuf = torch.zeros(1 << 23, dtype=torch.float32, device=dev)  # 32 MB, L2-resident
    blocks, threads, iters = 148 * 16, 256, 256
    for _ in range(2):
        L.tsb_red_probe(_lib.ptr(pbuf), 23, iters, blocks, threads, _lib.stream_handle())
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(5):
        L.tsb_red_probe(_lib.ptr(pbuf), 23, iters, blocks, threads, _lib.stream_handle())
    p1.record()
    torch.cuda.synchronize()
    red_peak = 5 * blocks * threads * iters / (p0.elapsed_time(p1) * 1e-3) / 1e9  # G adds/s
    red_rate = reds / (k8_ms * 1e-3) / 1e9
    k8_traffic = None
    tjp = ROOT / "profiles" / "traffic.json"
    if tjp.exists():
        k8_traffic = json.loads(tjp.read_text()).get("cfg4/k_raster_bwd")

    if rank == 0:
        line = {
            "metric": "training steps/s (cfg4: 100k textured 2DGS, 800x800, DP over views)",
            "value": round(world * args.steps / (ms * 1e-3), 3), "unit": "view-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg4 training step (BASELINE configs[3]): forward + shade + "
                       "loss + backward into atlas and Gaussian params + all-reduce + Adam",
                       "splats": args.splats, "texture_res": args.texture_res,
                       "width": args.width, "height": args.height,
                       "allreduce": "bucketed async all-reduce of the flat fp32 gradient buffer "
                                    "(geometry + env, then 4 texel buckets of 7-channel "
                                    "gradients), Adam per bucket",
                       "parallelism": f"data parallel over views, {world} GPU(s)"},
            "last_loss": terms["loss"],
            "roofline": {"bound": "l2_atomics", "kernel": "k_raster_bwd",
                         "achieved": round(red_rate, 3), "peak": round(red_peak, 3),
                         "unit": "G float atomic adds/s", "frac": round(red_rate / red_peak, 4),
                         "traffic": k8_traffic, "k8_ms": round(k8_ms, 4),
                         "traffic_source": "profiles/traffic.json (ncu --set full DRAM bytes "
                                           "read + written by one k_raster_bwd launch)",
                         "atomic_adds_per_launch": reds, "fragments": fragments,
                         "algorithmic_adds_before_warp_reduction": 28 * fragments,
                         "peak_source": "measured live: tsb_red_probe, scattered float adds "
                                        "into a 32 MB L2-resident buffer",
                         "note": "adds issued counted on the device (tsb_debug_red_count); K8 "
                                 "reduces each live splat's 22 terms and each bilinear cell's "
                                 "28 texel values over the warp before one add"},
            "clocks": clk,
            "e2e": {"value": round(e2e, 3), "unit": "view-steps/s",
                    "h2d_bytes_per_step": H * W * 3 * 4, "d2h_bytes_per_step": 8 * 8,
                    "note": "DataParallelTrainer.step with the view's display target copied "
                            "from pinned host memory and the step's loss terms read back "
                            "every step"},
            "gpu_launches": args.steps * (24 + n_adam),
            "gpu_launches_note": "ours per step: the 13 forward kernels (K1-K6 as in the render "
                                 "line), 3 K10 SSIM passes, k_shade_bwd, k_env_shard_reduce, "
                                 "k_reg_count, k_reg_grad, k_raster_bwd, k_finish_grads, "
                                 "k_guard_finite, k_orthonormalize and k_adam (one launch on one "
                                 "GPU, one per all-reduce bucket with DP); plus one torch copy "
                                 "of the fp64 geometry gradients into the flat buffer",
        }
        if world == 1 and not args.no_cpu_baseline and not args.no_numpy_reference:
            line["cpu_baseline"] = numpy_train_timing(args, fragments)
        if world > 1 and "TSB_BENCH_DEVICE" in os.environ:  # ranks share one GPU
            line["shared_device"] = True  # a code-path check, not a measurement
            line["value"] = None
            line["e2e"]["value"] = None
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def numpy_train_timing(args, frags_frame: float):
    """The reference's compute_step (numpy, baseline/_ref) on 64x64 windows
    of view 0, extrapolated to the full frame by fragment count: one process
    (2 windows) and one process per core (1 window each)."""
    from oracle import oracle
    if not (ROOT / "baseline" / "_ref" / "texsplat").exists():
        return {"unavailable": "baseline/_ref/texsplat not installed"}
    W, H = args.width, args.height
    procs = oracle.cpu_threads()
    windows = [(int(W * fx) - 32, int(H * fy) - 32, 64, 64)
               for fy in (0.4, 0.5, 0.6) for fx in (0.4, 0.5, 0.6)]

    def launch(crops):
        cmd = [sys.executable, str(ROOT / "scripts" / "numpy_ref_worker.py"), "--train",
               str(args.splats), str(args.texture_res), str(W), str(H), str(args.env_height),
               "0"] + [",".join(str(v) for v in c) for c in crops]
        return subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                text=True, env=dict(os.environ, OMP_NUM_THREADS="1",
                                                    OPENBLAS_NUM_THREADS="1"))

    def step_s(r):
        return r["prepare_s"] + (r["step_s"] - r["prepare_s"]) * frags_frame / max(r["fragments"], 1)

    try:
        one = json.loads(launch(windows[3:5]).communicate(timeout=900)[0].strip().splitlines()[-1])
        t1 = statistics.median(step_s(r) for r in one)
        ps = [launch([windows[i % 9]]) for i in range(procs)]
        par = []
        for q in ps:
            par += json.loads(q.communicate(timeout=900)[0].strip().splitlines()[-1])
        tp = statistics.median(step_s(r) for r in par)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"numpy reference run failed: {e!r}"[:200]}
    return {"value": round(1.0 / t1, 6), "unit": "view-steps/s", "cores": 1, "kind": "reference",
            "process_parallel": {"value": round(procs / tp, 6), "cores": procs},
            "sample": f"texsplat compute_step (numpy, baseline/_ref) on 64x64 windows of view 0 "
                      f"(2 single-process, {procs} concurrent processes x 1), extrapolated to "
                      f"the {W}x{H} frame by fragment count ({frags_frame:.0f})"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_13348_b200 import Renderer, pack_atlases, synth
    from paper_2506_13348_b200 import _lib
    from paper_2506_13348_b200.environment import BrdfLut
    from paper_2506_13348_b200.rasterize import render_prepared
    from paper_2506_13348_b200.shading import shade_planar

    rank, world, local = dist_env()
    # (TSB_BENCH_DEVICE / TSB_BENCH_BACKEND: test hooks that run every rank on
    # one GPU over gloo to exercise the multi-rank code path on a 1-GPU box)
    gpu = int(os.environ.get("TSB_BENCH_DEVICE", local))
    shared_device = world > 1 and "TSB_BENCH_DEVICE" in os.environ
    if shared_device and os.environ.get("TSB_BENCH_BACKEND", "nccl") == "nccl":
        raise SystemExit("TSB_BENCH_DEVICE puts every rank on one GPU: set "
                         "TSB_BENCH_BACKEND=gloo (NCCL cannot share a device)")
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("TSB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    scene = synth.make_shell_scene(args.splats, args.texture_res, seed=3, with_environment=True,
                                   env_height=args.env_height)
    cams = synth.bench_cameras(256, args.width, args.height)
    lut = BrdfLut.build()
    if args.workload == "train":
        run_train(args, scene, cams, lut, rank, world, dev)
        return
    texture_mode = "flat" if args.sampler == "flat" else "atlas"
    atlas = pack_atlases(scene) if texture_mode == "atlas" else None
    r = Renderer(scene, atlas, scene.environment, lut, texture_mode=texture_mode,
                 sampler=None if args.sampler == "flat" else args.sampler,
                 texel_format=args.texel_format, tile=args.tile)
    if args.batch_views > 0:  # one step = the first batch_views orbit views over all ranks
        my_views = [cams[i] for i in range(rank, min(args.batch_views, len(cams)), world)]
    else:
        my_views = [cams[i] for i in range(rank, len(cams), world)]

    # size the workspace from every view of this rank once (no per-frame host
    # sync later); the device-side running maximum of the entry counts
    # (k_ranges) then guards every timed / phased / e2e frame
    need = 0
    for cam in my_views:
        r.render(cam, check=True)
        need = max(need, r.entries_needed())
    r.reserve(my_views[0], int(need * 1.25) + 4096)
    r.prep.workspace.reset_max()

    W, H = args.width, args.height
    gb, px, col, _, _ = r._buffers(W, H)
    prep = r.prep
    L = _lib.lib()
    stream = torch.cuda.current_stream()
    sh = _lib.stream_handle(stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ws = prep.workspace
    mode = {"hw": _lib.MODE_HW, "verify": _lib.MODE_VERIFY, "flat": _lib.MODE_FLAT}[prep.sampler]
    sc, at = prep.scene.struct(), prep.atlas.struct()
    import ctypes as C

    def step(cam, evs=None):
        cs = _lib.camera_struct(cam)
        pst = px.struct()
        if evs:
            evs[0].record(stream)
        _lib.check(L.tsb_render_binning(C.byref(sc), C.byref(cs), C.byref(at), mode, args.tile,
                                        _lib.ptr(ws.buf), ws.nbytes, ws.capacity,
                                        _lib.ptr(ws.needed), sh), "binning")
        if evs:
            evs[1].record(stream)
        _lib.check(L.tsb_render_composite(C.byref(sc), C.byref(cs), C.byref(at), mode, args.tile,
                                          _lib.ptr(ws.buf), ws.nbytes, ws.capacity,
                                          _lib.ptr(gb), C.byref(pst), sh), "composite")
        if evs:
            evs[2].record(stream)
        shade_planar(gb, cam, r.env, r.background, color=col, want_split=False, stream=stream)
        if evs:
            evs[3].record(stream)

    for i in range(args.warmup):
        step(my_views[i % len(my_views)])
    torch.cuda.synchronize()

    K = args.steps
    # per-phase breakdown (binning / raster / shade events around each
    # library call): diagnostics and the raster kernel's roofline timing
    KB = min(K, 30)
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(KB)]
    frag_total = torch.zeros((), dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    for i in range(KB):
        flush.zero_()  # L2 flush (outside the timed events)
        step(my_views[i % len(my_views)], events[i])
        frag_total += px.n_contrib.sum(dtype=torch.int64)
    torch.cuda.synchronize()
    bin_ms = [e[0].elapsed_time(e[1]) for e in events]
    rast_ms = [e[1].elapsed_time(e[2]) for e in events]
    shade_ms = [e[2].elapsed_time(e[3]) for e in events]
    phased_ms = [e[0].elapsed_time(e[3]) for e in events]

    # timed steps: K steps back to back, one CUDA-graph replay per frame,
    # between a barrier + synchronize on both sides (inputs larger than L2)
    graph, _ = r._graph(my_views[0], W, H)
    cams_c = [_lib.camera_struct(c) for c in my_views]
    batch = args.batch_views > 0
    per_step = len(cams_c) if batch else 1
    npipe = max(1, args.pipeline)
    pipes = [(graph, col, stream)] + [
        (*r._graph(my_views[0], W, H, slot=j), torch.cuda.Stream(dev)) for j in range(1, npipe)]

    def launch(i):
        g_, c_, s_ = pipes[i % npipe]
        _lib.check(L.tsb_frame_graph_launch(g_, C.byref(cams_c[i % len(cams_c)]),
                                            _lib.ptr(c_), _lib.stream_handle(s_)), "graph")

    for i in range(args.warmup * per_step):
        launch(i)
    # diagnostic: the same frames with the L2 flushed before each one
    KF = min(K, 30)
    gevents = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(KF)]
    for i in range(KF):
        flush.zero_()
        gevents[i][0].record(stream)
        launch(i * npipe)  # (slot 0, the timing stream)
        gevents[i][1].record(stream)
    torch.cuda.synchronize()
    frame_ms = [e[0].elapsed_time(e[1]) for e in gevents]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(gpu)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _, _, s_ in pipes[1:]:
        s_.wait_event(ev0)
    for i in range(K * per_step):
        launch(i)
    for _, _, s_ in pipes[1:]:  # join the other frame streams
        ej = torch.cuda.Event()
        ej.record(s_)
        stream.wait_event(ej)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    overflow = r.max_entries_needed() > ws.capacity  # any phased or timed frame
    fragments = int(frag_total.item()) / KB

    # ---- e2e: public API, host result every step ---------------------------
    # Renderer.stream_views: each frame's colour image lands in pinned host
    # memory; frame i's device->host copy overlaps frame i+1's render.
    cam_bytes = C.sizeof(_lib.Camera_t)
    e2e_views = (list(my_views) if batch else
                 [my_views[i % len(my_views)] for i in range(args.e2e_steps)])
    for _ in r.stream_views(e2e_views[:4], pipeline=npipe):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    checksum = 0.0
    for _, host_img in r.stream_views(e2e_views, pipeline=npipe):
        checksum += float(host_img[H // 2, W // 2, 0])
    e2e_s = time.perf_counter() - t0
    clk = clocks.stop()
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_fps = (args.batch_views if batch else world * args.e2e_steps) / float(te.item())

    # ---- e2e through texsplat's own per-view loop (cli.py:63-68) ----------
    # render_forward(scene, cam, "atlas", atlas) + shade_gbuffer(...) per view
    # with the reference's objects, colour to a numpy array each view: the
    # one-shot API (device copies cached per host object, resident.py)
    loop_fps = None
    if world == 1 and not batch and args.sampler == "hw":
        from paper_2506_13348_b200 import render_forward, shade_gbuffer
        nl = min(args.e2e_steps, 50)
        for cam in my_views[:3]:
            gbl = render_forward(scene, cam, "atlas", atlas, texel_format=args.texel_format)
            shade_gbuffer(gbl, cam, scene.environment, lut, background=scene.background)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(nl):
            cam = my_views[i % len(my_views)]
            gbl = render_forward(scene, cam, "atlas", atlas, texel_format=args.texel_format)
            srl = shade_gbuffer(gbl, cam, scene.environment, lut, background=scene.background)
            img = srl.color.cpu().numpy()
        loop_fps = nl / (time.perf_counter() - t0)
        del img

    # ---- TEX peak probe (same texture, L1-resident window) ------------------
    tex_peak = None
    if prep.atlas.tex is not None:
        blocks, threads, iters = 148 * 8, 256, 512
        sink = torch.empty(blocks * threads, dtype=torch.float32, device=dev)
        for _ in range(2):
            _lib.check(L.tsb_tex_probe(prep.atlas.tex, 32, iters, _lib.ptr(sink), blocks, threads,
                                       sh), "tex probe")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = 5
        for _ in range(reps):
            L.tsb_tex_probe(prep.atlas.tex, 32, iters, _lib.ptr(sink), blocks, threads, sh)
        e1.record(stream)
        torch.cuda.synchronize()
        tex_peak = reps * blocks * threads * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9  # Gfetch/s

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return

    import json as _json
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = _json.loads(pk.read_text())
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"

    rast_avg_s = statistics.mean(rast_ms) * 1e-3
    T = args.texture_res
    P = args.splats
    texel_b = 16 if args.texel_format == "rgba32f" else 8
    # compulsory HBM bytes of one K5 launch: G-buffer
    # + pixel state out, entry list + per-splat records in, and the atlas
    # charts (both families) of every splat that composites, read once.
    # The touched-splat count comes from one extra, untimed diagnostic frame.
    entries = r.entries_needed()
    touched = torch.zeros(P, dtype=torch.uint8, device=dev)
    cam_d = _lib.camera_struct(my_views[0])
    pst_d = px.struct(touched)
    _lib.check(L.tsb_render_binning(C.byref(sc), C.byref(cam_d), C.byref(at), mode, args.tile,
                                    _lib.ptr(ws.buf), ws.nbytes, ws.capacity,
                                    _lib.ptr(ws.needed), sh), "binning")
    _lib.check(L.tsb_render_composite(C.byref(sc), C.byref(cam_d), C.byref(at), mode, args.tile,
                                      _lib.ptr(ws.buf), ws.nbytes, ws.capacity, _lib.ptr(gb),
                                      C.byref(pst_d), sh), "composite")
    n_touched = int(touched.sum(dtype=torch.int64).item())
    entries = r.entries_needed()
    alg_bytes = 68 * W * H + 4 * entries + 128 * P + 2 * n_touched * T * T * texel_b
    traffic, ncu_l1 = None, None
    tj = ROOT / "profiles" / "traffic.json"
    if tj.exists():
        tjd = _json.loads(tj.read_text())
        traffic = tjd.get(f"{args.config}/{args.sampler}/{args.texel_format}")
        if f"{args.config}/{args.sampler}/{args.texel_format}" == "cfg2/hw/rgba32f":
            ncu_l1 = tjd.get("ncu")
    hbm_achieved = alg_bytes / rast_avg_s / 1e9
    fetch_rate = 2 * fragments / rast_avg_s / 1e9 if args.sampler != "flat" else 0.0

    value = (K * args.batch_views if batch else world * K) / (max_ms * 1e-3)
    verify_fps = None
    if args.sampler == "hw" and world == 1 and not batch:
        # like-for-like with the CPU arms (fp32 software bilinear = verify mode)
        rv = Renderer(scene, atlas, scene.environment, lut, texture_mode="atlas",
                      sampler="verify", tile=args.tile)
        rv.reserve(my_views[0], ws.capacity)
        for i in range(3):
            rv.render(my_views[i], check=False)
        gv, _ = rv._graph(my_views[0], W, H)
        gcol = rv._buffers(W, H)[2]
        torch.cuda.synchronize()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        for i in range(K):
            _lib.check(L.tsb_frame_graph_launch(gv, C.byref(cams_c[i % len(cams_c)]),
                                                _lib.ptr(gcol), sh), "graph")
        v1.record(stream)
        torch.cuda.synchronize()
        verify_fps = K / (v0.elapsed_time(v1) * 1e-3)
        rv.check_capacity()
        rv.close()
        del rv
    # the texel pages both families occupy in HBM (the texture arrays / linear copies)
    _a = prep.atlas
    atlas_mb = (2 * getattr(_a, "pages", 0) * getattr(_a, "page_h", 0) * getattr(_a, "page_w", 0)
                * 4 * (2 if args.texel_format == "rgba16f" else 4) / 1e6)
    view0_frags = None
    if world == 1 and not args.no_cpu_baseline:  # fragments of view 0 (numpy extrapolation)
        r.render(cams[0], check=True)
        view0_frags = float(px.n_contrib.sum(dtype=torch.int64).item())
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(max_ms / K, 4),
        "higher_is_better": True, "scaling": "strong" if batch else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD if args.config == "cfg2" else
                   f"{args.config}: {P} textured 2D Gaussians, {T}x{T} atlas, {W}x{H}",
                   "splats": P, "texture_res": T, "width": W,
                   "height": H, "sampler": args.sampler, "texel_format": args.texel_format,
                   "tile": args.tile,
                   "views": (f"one step = the {args.batch_views}-view bench_cameras orbit batch, "
                             f"rank r renders views r::N" if batch else
                             "bench_cameras(256) orbit, rank r takes r::N, one view per step"),
                   "l2": ((f"inputs larger than L2 (atlas pages {atlas_mb:.0f} MB > 126 MB "
                           "L2): frames back to back, no flush; ") if atlas_mb > 126 else
                          ("no atlas larger than L2 in this mode: frames back to back without a "
                           "flush (a diagnostic line, not the headline); ")) +
                         "breakdown_ms.frame_median_l2_flushed repeats frames with a 256 MB "
                         "L2 flush before each",
                   "parallelism": f"views partitioned over {world} GPU(s), scene replicated",
                   "frames_in_flight": npipe},
        "breakdown_ms": {"binning": round(statistics.mean(bin_ms), 4),
                         "raster": round(statistics.mean(rast_ms), 4),
                         "shade": round(statistics.mean(shade_ms), 4),
                         "frame_median_l2_flushed": round(statistics.median(frame_ms), 4),
                         "frame_median_launches": round(statistics.median(phased_ms), 4)},
        "verify_sampler_fps": None if verify_fps is None else round(verify_fps, 3),
        "verify_sampler_note": "the same frames with the fp32 software-bilinear sampler "
                               "(verify mode), the arithmetic the CPU reference arm runs: "
                               "the like-for-like ratio is verify_sampler_fps / reference",
        "fragments_per_frame": fragments, "entries_per_frame": entries,
        "capacity_overflow": bool(overflow),
        "roofline": {"bound": "hbm", "kernel": "k_raster_fwd", "achieved": round(hbm_achieved, 2),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(hbm_achieved / hbm_peak, 4),
                     "traffic": traffic, "peak_source": hbm_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "splats_composited": n_touched,
                     "traffic_source": "profiles/traffic.json (ncu --set full dram__bytes_read.sum"
                                       " + dram__bytes_write.sum of one k_raster_fwd launch)"},
        "roofline_tex": {"bound": "tex", "kernel": "k_raster_fwd",
                         "achieved": round(fetch_rate, 3), "unit": "Gfetch/s",
                         "peak": round(tex_peak, 3) if tex_peak else None,
                         "frac": round(fetch_rate / tex_peak, 4) if tex_peak else None,
                         "peak_source": "measured live: tsb_tex_probe bilinear RGBA fetches, "
                                        "L1-resident 32x32 window of the same texture",
                         "fetches_per_launch": 2 * fragments,
                         "ncu_l1tex": ncu_l1},
        "clocks": clk,
        "e2e": {"value": round(e2e_fps, 3), "unit": "frames/s",
                "h2d_bytes_per_step": cam_bytes, "d2h_bytes_per_step": H * W * 3 * 4,
                "note": "Renderer.stream_views: render + D2H of every frame's (H,W,3) float32 "
                        "colour into pinned host memory, host consumes each image in order; "
                        "frames_in_flight views in independent workspaces on their own "
                        "streams, each colour copied out on a copy stream as its view "
                        "completes; camera passed by value in the launch; scene, atlas, "
                        "environment resident (uploaded once)"},
        "e2e_reference_loop": None if loop_fps is None else {
            "value": round(loop_fps, 3), "unit": "frames/s",
            "h2d_bytes_per_step": cam_bytes, "d2h_bytes_per_step": H * W * 3 * 4,
            "note": "texsplat's cmd_render per-view body (cli.py:63-68) through the drop-in "
                    "API: render_forward + shade_gbuffer with the same host scene / atlas / "
                    "environment objects, colour copied to numpy every view, synchronously "
                    "(no overlap of the copy with the next view, a host sync per view for "
                    "the capacity check)"},
        "gpu_launches": 13 * K * per_step,
        "gpu_launches_note": "ours per frame (one CUDA graph replay per view, no library "
                             "kernels): k_preprocess, 4 x k_onesweep (depth), k_fix_runs, "
                             "k_sort_long_runs, k_dup_tx, k_onesweep (tile rows), k_ranges, "
                             "k_tile_schedule, k_raster_fwd, k_shade (+ 2 memset nodes)",
    }
    if world == 1 and not args.no_cpu_baseline:
        fps, cores, sample, _ = cpu_baseline_run(args, args.cpu_frames)
        line["cpu_baseline"] = {"value": round(fps, 6), "unit": "frames/s", "cores": cores,
                                "kind": "port", "sample": sample, "note": CPU_BASELINE_NOTE}
        if not args.no_numpy_reference and view0_frags:
            npr = numpy_reference_timing(args, view0_frags, cores)
            line["cpu_baseline"]["numpy_reference"] = npr
            if "fps_single_process" in npr:
                line["vs_numpy_reference"] = {
                    "e2e_over_single_process": round(e2e_fps / npr["fps_single_process"], 1),
                    "e2e_over_process_parallel": round(e2e_fps / npr["fps_process_parallel"], 1)}
    if shared_device:  # every rank on one GPU: a code-path check, not a measurement
        line["shared_device"] = True
        line["value"] = None
        line["e2e"]["value"] = None
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
