#!/usr/bin/env python
"""Benchmark of the Schwarzschild ray-tracing hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step = one full frame of BASELINE.json configs[C] (default C=2: 3840x2160,
4 jittered spp, disk + 64 spheres, RKF45 tol 1e-9) rendered by all ranks
(cyclic row tiles). With N > 1 every rank's kernel stores its rows straight
into rank 0's image over CUDA-IPC peer memory (NVLink/NVSwitch), completion
by a stream-ordered NCCL all-reduce (an NCCL gather + unshuffle if the image
cannot be mapped). Prints ONE JSON line on rank 0. Metric: Mrays/s (rays =
pixels x spp), whole job.

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU); it exits non-zero, without
timing anything, when fewer than N GPUs are visible.

--impl reference times the CPU implementation of the same workload on the
host cores (rank 0 only): the oracle port of the full scene on the same full
frame (the reference itself cannot render disk/spheres/RKF45 —
SPEC.md:14,171), kind "port"; beside it the compiled reference's own code on
the sky-only projection through its own harness (run_strong_scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    0: "config0: 256x256x1spp disk+checker, RK4 dphi=1e-3",
    1: "config1: 1920x1080x1spp disk+checker, RKF45 tol 1e-9",
    2: "config2: 3840x2160x4spp jittered, disk r6-30 + 64 Lambertian spheres, RKF45 tol 1e-9",
    3: "config3: 7680x4320x1spp approximate mode (100k-entry b-table by RKF45), disk+checker",
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                m = float(f[1])
                mx = float(f[2])
            except ValueError:
                continue
            mhz.append(m)
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [m for m in mhz if m > 500] or mhz
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(mhz)}


def hbm_peak() -> float:
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the
    B200_PROFILING.md fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 7000.0


# ---------------------------------------------------------------- CPU legs
def cpu_port_rows(scene, rows_sel, threads):
    """Render the selected rows with the oracle's pthread row queue."""
    import ctypes as C
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import oracle
    from paper_2507_16165_b200.abi import StatusInfo
    L = oracle()
    # contiguous block of rows keeps the oracle's dynamic row queue busy
    r0, r1 = rows_sel
    out = np.zeros((r1 - r0) * scene.s.width * 3, np.uint8)
    info = StatusInfo()
    t0 = time.perf_counter()
    rc = L.orc_render_rows(C.byref(scene.s), r0, r1, threads,
                           out.ctypes.data_as(C.POINTER(C.c_uint8)), None, C.byref(info))
    dt = time.perf_counter() - t0
    if rc:
        raise RuntimeError(f"oracle failed: {info.message}")
    return (r1 - r0) * scene.s.width * scene.s.spp, dt


def centre_band(height: int, rows: int):
    r0 = max(0, height // 2 - rows // 2)
    return r0, min(height, r0 + rows)


def lattice(width: int, height: int, nx: int = 96, ny: int = 64):
    """A cyclic lattice over the whole frame: ny rows x nx columns, evenly
    spaced (pixel centres of an ny x nx grid laid over the image)."""
    xs = [int((i + 0.5) * width / nx) for i in range(min(nx, width))]
    ys = [int((j + 0.5) * height / ny) for j in range(min(ny, height))]
    return [(x, y) for y in ys for x in xs]


def reference_sky_only(scene, threads: int, repeats: int = 5, nx: int = 96, ny: int = 64):
    """The compiled reference (oracle/_ref) on the sky-only projection of the
    workload, timed by its own harness: run_strong_scaling(scene, {threads},
    repeats) (bench.cpp:59-73, mean of 5 as PAPER.md:265) with a RenderRunner
    that shades a 64-row x 96-column lattice of the frame's pixels through
    the reference's shade_pixel on `threads` threads."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import have_ref, ref
    from paper_2507_16165_b200 import scenes
    if not have_ref():
        return None
    proj = scenes.sky_only_projection(scene)
    pts = lattice(proj.s.width, proj.s.height, nx, ny)
    px = (C.c_int * len(pts))(*[p[0] for p in pts])
    py = (C.c_int * len(pts))(*[p[1] for p in pts])
    mean = ref().ref_strong_scaling_pixels_mean(C.byref(proj.s), threads, repeats, px, py, len(pts))
    if not mean > 0:
        return None
    rays = len(pts) * proj.s.spp
    return {"value": rays / mean / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "reference",
            "sample": f"oracle/_ref (the reference's own code) on the sky-only projection of the "
                      f"workload (DOPRI5 eps=0.05 windows, checker baked into a 2048x1024 PPM): "
                      f"run_strong_scaling(scene, {{{threads}}}, {repeats}) mean wall time, its "
                      f"RenderRunner shading a {ny}-row x {nx}-column pixel lattice of the "
                      f"{proj.s.width}x{proj.s.height} frame ({rays} rays/run) with shade_pixel",
            "seconds_per_run": mean}


def measure_secondary(device: int, peak: float, reps: int = 3, rank: int = 0, world: int = 1) -> dict:
    """Device-timed Mrays/s of configs 0, 1, 3 (scene resident, best of
    `reps` after one warm-up) and config 4's whole 120-frame orbit (frames/s,
    wall clock, per-frame scene upload + cull table included; with N ranks
    the frames are sharded f mod N and the whole-box rate uses the slowest
    rank). Everything but config 4 runs on rank 0 only."""
    import torch
    import torch.distributed as dist

    from paper_2507_16165_b200 import render, roofline, scenes
    out = {}
    ctx = render.Context(device)
    ctx.set_timing(True)
    st = torch.cuda.current_stream()
    for idx in (0, 1, 3) if rank == 0 else ():
        sb = scenes.config(idx)
        t0 = time.perf_counter()
        ctx.set_scene(sb)
        setup_s = time.perf_counter() - t0
        buf = torch.empty(sb.s.width * sb.s.height * 3, dtype=torch.uint8, device="cuda")
        best = None
        kern = None
        for r in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
            e1.record(st)
            ctx.finish()
            e1.synchronize()  # finish() waits for the render only; the end event may trail it
            ms = e0.elapsed_time(e1)
            if r > 0 and (best is None or ms < best):
                best = ms
                kern = ctx.kernel_ms()[0]
        rays = sb.s.width * sb.s.height * sb.s.spp
        stats = ctx.stats()
        line = {"ms": best, "kernel_ms": kern, "Mrays/s": rays / best / 1e3,
                "steps_per_ray": stats["steps"] / rays,
                "set_scene_s": setup_s, "size": [sb.s.width, sb.s.height, sb.s.spp]}
        if idx == 3:
            # table mode: no integration; bound by the latency of its table
            # gathers (L1/L2). Algorithmic bytes = roofline.table_bytes
            # (per-sample lookups + per-event orbit evaluations + RGB8 out)
            nbytes = roofline.table_bytes(sb, stats)
            line["steps_per_ray"] = None
            line["orbit_evals_per_ray"] = stats["steps"] / rays
            line["roofline"] = {"bound": "latency (table gathers)", "algorithmic_bytes": nbytes,
                                "achieved_GBps": nbytes / (kern * 1e-3) / 1e9, "unit": "GB/s",
                                "hbm_peak_GBps": hbm_peak(),
                                "frac_of_hbm": nbytes / (kern * 1e-3) / 1e9 / hbm_peak()}
        else:
            fl = roofline.launch_flops(sb, stats)
            line["roofline"] = {"bound": "fp64", "flops_per_launch": fl,
                                "achieved": fl / (kern * 1e-3) / 1e12, "peak": peak,
                                "unit": "TFLOP/s", "frac": fl / (kern * 1e-3) / 1e12 / peak}
        out[f"config{idx}"] = line
    frames = 120
    sb0 = scenes.config(4, frame=0)
    buf = torch.empty(sb0.s.width * sb0.s.height * 3, dtype=torch.uint8, device="cuda")
    for f in range(2):  # warm-up
        ctx.set_scene(scenes.config(4, frame=f))
        ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
        ctx.finish()
    scs = [scenes.config(4, frame=f) for f in range(frames)]
    # six contexts on six streams in turn: frame f+1's scene upload (cull
    # lists built on the device, async copies) proceeds while frame f
    # renders, and later frames' kernels fill the SMs while the close-camera
    # frames' longest rays drain (3/4/6/8 streams: 533/548/556/559 frames/s,
    # tools/orbit_time.py); each finish() waits for its own frame only
    NC = 6
    ctxs = [ctx] + [render.Context(device) for _ in range(NC - 1)]
    bufs = [buf] + [torch.empty_like(buf) for _ in range(NC - 1)]
    strs = [st] + [torch.cuda.Stream(device) for _ in range(NC - 1)]
    mine = scs[rank::world]  # frame sharding f mod N (BASELINE.json config 4)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    flops4 = 0.0
    for f, sb in enumerate(mine):
        c = ctxs[f % NC]
        c.set_scene(sb)
        c.render_async(bufs[f % NC].data_ptr(), stream=strs[f % NC].cuda_stream)
        if f >= NC - 1:
            g = f - NC + 1
            ctxs[g % NC].finish()
            flops4 += roofline.launch_flops(mine[g], ctxs[g % NC].stats())
    for g in range(max(0, len(mine) - NC + 1), len(mine)):
        ctxs[g % NC].finish()
        flops4 += roofline.launch_flops(mine[g], ctxs[g % NC].stats())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tdt = torch.tensor([dt, flops4], device="cuda", dtype=torch.float64)
    if world > 1:
        tmax = tdt[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tdt, op=dist.ReduceOp.SUM)
        dt, flops4 = float(tmax.item()), float(tdt[1].item())
    for c in ctxs[1:]:
        c.close()
    out["config4"] = {"frames": frames, "seconds": dt, "frames/s": frames / dt,
                      "Mrays/s": frames * sb0.s.width * sb0.s.height * sb0.s.spp / dt / 1e6,
                      "size": [sb0.s.width, sb0.s.height, sb0.s.spp], "n_gpus": world,
                      "roofline": {"bound": "fp64", "flops": flops4,
                                   "achieved": flops4 / dt / 1e12 / world, "peak": peak,
                                   "unit": "TFLOP/s per GPU", "frac": flops4 / dt / 1e12 / world / peak,
                                   "note": "whole orbit incl. per-frame host setup (wall clock)"},
                      "note": "frames sharded f mod N; whole-box rate = frames / slowest rank"}
    if rank != 0:
        ctx.close()
        return out
    # strong-scaling projection on this one GPU: each rank's cyclic-row share
    # of the config-2 frame rendered alone (device time), max over ranks, vs
    # the whole frame / N. Communication is not included (the multi-GPU run
    # writes rows into rank 0's image over NVLink while they are shaded).
    sb2 = scenes.config(2)
    ctx.set_scene(sb2)
    buf = torch.empty(sb2.s.width * sb2.s.height * 3, dtype=torch.uint8, device="cuda")

    def share_ms(world, rank):
        best = None
        for r in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.render_async(buf.data_ptr(), 0, sb2.s.height, 1, world, rank, stream=st.cuda_stream)
            e1.record(st)
            ctx.finish()
            e1.synchronize()  # finish() waits for the render only; the end event may trail it
            ms = e0.elapsed_time(e1)
            if r > 0 and (best is None or ms < best):
                best = ms
        return best

    full = share_ms(1, 0)
    proj = {"full_frame_ms": full}
    for world in (2, 4, 8):
        per = [share_ms(world, r) for r in range(world)]
        proj[f"n{world}"] = {"max_rank_ms": max(per), "min_rank_ms": min(per),
                             "efficiency": full / (world * max(per))}
    proj["note"] = ("device time of each rank's cyclic-row share rendered alone on this GPU; "
                    "efficiency = T1 / (N * max_rank T_N); excludes the completion collective")
    out["strong_scaling_projection"] = proj
    # the same orbit written out as PPM files (the host output pipeline,
    # sequence.SequenceRenderer: kernel of frame f overlaps writing f-1)
    import tempfile

    from paper_2507_16165_b200.sequence import SequenceRenderer
    with tempfile.TemporaryDirectory() as tmp:
        paths = [os.path.join(tmp, f"frame_{f:04d}.ppm") for f in range(frames)]
        sr = SequenceRenderer(device)
        sr.render(scs[:2], paths[:2])  # warm-up
        res = sr.render(scs, paths)
        sr.close()
    out["config4_ppm"] = {"frames": frames, "seconds": res["seconds"], "frames/s": res["frames/s"],
                          "note": "render + D2H + PPM encode/write of every frame (save_ppm "
                                  "layout), writer thread overlapped with the next frame's kernel"}
    # the reference's own algorithm (mode R: DOPRI5 in eps-windows, its
    # arithmetic) on the GPU, on the same sky-only projection of config 2 that
    # `reference_sky_only` times on the CPU: same algorithm, same bytes
    proj = scenes.sky_only_projection(scenes.config(2))
    ctx.set_scene(proj)
    buf = torch.empty(proj.s.width * proj.s.height * 3, dtype=torch.uint8, device="cuda")
    ctx.render_async(buf.data_ptr(), 1000, 1016, stream=st.cuda_stream)  # warm-up band
    ctx.finish()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    ctx.finish()
    e1.synchronize()  # finish() waits for the render only; the end event may trail it
    ms = e0.elapsed_time(e1)
    rays = proj.s.width * proj.s.height * proj.s.spp
    stR = ctx.stats()
    flR = roofline.launch_flops(proj, stR)
    kR = ctx.kernel_ms()[0]
    out["modeR_sky_only"] = {"ms": ms, "kernel_ms": kR, "Mrays/s": rays / ms / 1e3,
                             "windows_per_ray": stR["steps"] / rays,
                             "roofline": {"bound": "fp64", "flops_per_launch": flR,
                                          "achieved": flR / (kR * 1e-3) / 1e12, "peak": peak,
                                          "unit": "TFLOP/s", "frac": flR / (kR * 1e-3) / 1e12 / peak},
                             "size": [proj.s.width, proj.s.height, proj.s.spp],
                             "note": "trace_reference_kernel (reference algorithm, bit-identical "
                                     "window arithmetic) on the full sky-only projection; compare "
                                     "reference_sky_only (the reference on the host cores)"}
    ctx.close()
    return out


# ---------------------------------------------------------------- arms
def run_reference_arm(args):
    """The CPU implementation of the path on this box's host cores (rank 0
    only): the oracle port (C, pthreads) renders the same full frame as our
    arm each step. The scene is built with the oracle's own sphere generator,
    so no product library is loaded in this process."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import oracle
    from paper_2507_16165_b200 import scenes
    scene = scenes.config(args.config, sphere_lib=oracle())
    threads = os.cpu_count() or 1
    H = scene.s.height
    band = (0, H) if args.ref_rows is None else centre_band(H, args.ref_rows)
    for _ in range(args.warmup):  # untimed: thread pool + caches, one centre row
        cpu_port_rows(scene, centre_band(H, 1), threads)
    tot_rays, tot_s = 0, 0.0
    for _ in range(args.steps):
        rays, dt = cpu_port_rows(scene, band, threads)
        tot_rays += rays
        tot_s += dt
    value = tot_rays / tot_s / 1e6
    full = band == (0, H)
    sample = (f"oracle port (C, pthreads) of the full workload, "
              + (f"the whole {scene.s.width}x{H}x{scene.s.spp} frame" if full
                 else f"rows [{band[0]},{band[1]})")
              + f" = {tot_rays // args.steps} rays per step")
    ref_sky = None if args.no_ref_sky else reference_sky_only(scene, threads)
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": value, "unit": "Mrays/s",
        "n_gpus": world if "WORLD_SIZE" in os.environ else args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "width": scene.s.width,
                   "height": scene.s.height, "spp": scene.s.spp, "parallelism": f"cpu x{threads}"},
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_sky_only": ref_sky,
    }
    print(json.dumps(line), flush=True)
    return 0


def dropin_e2e(scene, device: int, iters: int, flush) -> dict:
    """The reference-facing drop-in: bhrt_cuda_render_rows (include/bhrt_cuda.h,
    the C ABI render_shim.cpp's render_rows calls) with HOST buffers — scene
    from host memory, pixels into a caller-owned host buffer — timed end to
    end per call (wall clock, synchronous API)."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2507_16165_b200 import native
    from paper_2507_16165_b200.abi import StatusInfo
    L = native.lib()
    W, H = scene.s.width, scene.s.height
    out = np.zeros(W * H * 3, np.uint8)  # caller-owned, pages touched once
    devs = (C.c_int32 * 1)(device)
    info = StatusInfo()

    def call():
        rc = L.bhrt_cuda_render_rows(scene.ptr(), 0, H, devs, 1,
                                     out.ctypes.data_as(C.POINTER(C.c_uint8)), out.nbytes, None,
                                     C.byref(info))
        native.check(rc, info)

    call()
    call()
    ms = []
    for _ in range(iters):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        ms.append((time.perf_counter() - t0) * 1e3)
    return {"ms": ms, "image": out}


def gpu_reference_harness(scene, device: int, repeats: int = 5) -> dict | None:
    """The GPU timed by the reference's OWN harness: dropin/bhrt_bench_b200
    (csrc/bench_main.cpp) runs bench.cpp's run_strong_scaling(scene, {1},
    repeats) and emit_csv unchanged, its default RenderRunner render_image
    resolving to render_shim.cpp (mode R, byte-identical to the reference).
    Scene: the sky-only projection of the workload at full size — the same
    scene reference_sky_only times on the CPU through the same harness. One
    untimed warm-up frame first (CUDA context); mean of the run = -1 row."""
    import subprocess
    import tempfile

    from paper_2507_16165_b200 import scenes
    exe = os.path.join(ROOT, "paper_2507_16165_b200", "dropin", "bhrt_bench_b200")
    if not os.path.exists(exe):
        return None
    proj = scenes.sky_only_projection(scene)
    sky = proj.sky
    with tempfile.TemporaryDirectory() as d:
        cfg, bg, out = (os.path.join(d, n) for n in ("scene.txt", "sky.ppm", "bench.csv"))
        open(cfg, "w").write(proj.to_text())
        with open(bg, "wb") as f:
            f.write(f"P6\n{sky.shape[1]} {sky.shape[0]}\n255\n".encode() + sky.tobytes())
        r = subprocess.run([exe, "bench", "--config", cfg, "--background", bg, "--output", out,
                            "--worker-counts", "1", "--repeats", str(repeats), "--warmup", "1"],
                           capture_output=True, text=True, timeout=900,
                           env=dict(os.environ, BHRT_DEVICES=str(device)))
        if r.returncode != 0:
            return {"error": r.stderr.strip()[-300:]}
        rows = [ln.split(",") for ln in open(out).read().splitlines()[1:]]
    mean = [float(x[8]) for x in rows if x[7] == "-1"][0]
    rays = proj.s.width * proj.s.height * proj.s.spp
    return {"value": rays / mean / 1e6, "unit": "Mrays/s", "seconds_per_run": mean,
            "runs": [float(x[8]) for x in rows if x[7] != "-1"],
            "harness": "reference bench.cpp run_strong_scaling(scene, {1}, %d) + emit_csv, "
                       "RenderRunner = render_image (render_shim.cpp -> C ABI, mode R)" % repeats,
            "scene": f"sky-only projection of the workload, {proj.s.width}x{proj.s.height}x"
                     f"{proj.s.spp}, DOPRI5 eps={proj.s.epsilon} windows, 2048x1024 PPM sky, "
                     f"host image out (wall clock per frame)"}


def self_launch(args) -> int:
    """--gpus N outside torchrun: re-launch under torch.distributed.run with N
    ranks, or refuse (non-zero, nothing timed) when fewer GPUs are visible."""
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA device(s) are visible; "
              f"refusing to time fewer GPUs than requested", file=sys.stderr, flush=True)
        return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2507_16165_b200 import native, roofline, scenes
    from paper_2507_16165_b200.parallel import FrameRenderer

    rank, world, local = env_rank()
    # BHRT_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 over gloo, to
    # exercise the N > 1 control flow (collective order, no deadlock) on a
    # one-GPU lease; never a timing configuration
    shared = os.environ.get("BHRT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    scene = scenes.config(args.config)
    W, H, spp = scene.s.width, scene.s.height, scene.s.spp
    total_rays = W * H * spp

    fr = FrameRenderer(rank, world, local)
    fr.set_scene(scene)
    fr.ctx.set_timing(True)
    st = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        return fr.render_device(st)

    for _ in range(args.warmup):
        step()
        fr.finish()
    torch.cuda.synchronize()
    barrier()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ms, trace_ms, shade_ms, flops = [], [], [], []
    stats = None
    for _ in range(args.steps):
        flush.zero_()  # L2 flush (256 MiB > 126 MB L2) outside the timed window
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        fr.finish()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        t_ms, s_ms = fr.ctx.kernel_ms()
        trace_ms.append(t_ms)
        shade_ms.append(s_ms)
        stats = fr.ctx.stats()
        flops.append(roofline.launch_flops(scene, stats))
    clocks = sampler.stop()
    step_ms = sum(ms) / len(ms)
    t = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms_max = float(t.item())
    value = total_rays / (step_ms_max * 1e-3) / 1e6

    # ---- e2e through the public API: H2D scene, render, gather, D2H image
    e2e_ms = []
    for i in range(max(2, args.steps) + 1):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        fr.render(scene)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:
            e2e_ms.append(dt)
    te = torch.tensor([sum(e2e_ms) / len(e2e_ms)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = total_rays / (float(te.item()) * 1e-3) / 1e6
    staged, params, counters = fr.ctx.upload_bytes()
    e2e_launches = fr.ctx.stats()["launches"]
    # scene uploads + kernel parameter blocks + the counter slots' reset
    h2d = staged + e2e_launches * params + counters
    d2h = (W * H * 3 if rank == 0 else 0) + counters  # the image + the counter slots
    peer = fr.peer is not None

    # ---- the reference-facing drop-in (C ABI, host buffers), N = 1
    dropin = None
    if world == 1:
        dr = dropin_e2e(scene, local, max(3, args.steps), flush)
        dms = sum(dr["ms"]) / len(dr["ms"])
        same = bool((dr["image"].reshape(H, W, 3) == fr.host.numpy()).all())
        dropin = {"value": total_rays / (dms * 1e-3) / 1e6, "unit": "Mrays/s", "ms": dms,
                  "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                  "api": "bhrt_cuda_render_rows (C ABI; render_shim.cpp render_rows), host buffers",
                  "image_equals_frame_renderer": same}

    # ---- roofline denominator (every rank measures its own GPU)
    peak = native.lib().bhrt_b200_fp64_peak_tflops(200000, 3, None)

    # ---- the other BASELINE.json configs (secondary lines). Called on EVERY
    # rank: config 4's frames are sharded over the ranks (its barrier and
    # max-over-ranks reduction are collectives); the rest runs on rank 0.
    secondary = None
    if not args.no_secondary:
        secondary = measure_secondary(local, peak, rank=rank, world=world)

    if rank != 0:
        dist.barrier() if world > 1 else None
        dist.destroy_process_group() if world > 1 else None
        return 0

    # ---- roofline of the dominant kernel (trace), FP64 pipe
    avg_trace_ms = sum(trace_ms) / len(trace_ms)
    achieved = (sum(flops) / len(flops)) / (avg_trace_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    pipe_busy = None
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = tj.get(f"config{args.config}")
            pipe_busy = tj.get(f"config{args.config}_fp64_pipe_active")
        except Exception:
            traffic = None

    # ---- CPU baseline on this box's host cores (rank 0, N=1 only)
    cpu = None
    ref_sky = None
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        band = centre_band(H, args.cpu_rows)
        rays, dt = cpu_port_rows(scene, band, threads)
        cpu = {"value": rays / dt / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "port",
               "sample": f"oracle port (C, pthreads) of the full workload, rows "
                         f"[{band[0]},{band[1]}) = {rays} rays, {dt:.1f} s"}
        if not args.no_ref_sky:
            ref_sky = reference_sky_only(scene, threads)
    harness = None
    if world == 1 and not args.no_ref_sky:
        harness = gpu_reference_harness(scene, local)

    if world > 1:
        par = (f"cyclic rows x{world}: each rank's kernel stores its rows into rank 0's image "
               f"over CUDA-IPC peer memory (NVLink), completion by a stream-ordered NCCL "
               f"all-reduce" if peer else
               f"cyclic rows x{world} + NCCL gather + unshuffle on rank 0")
    else:
        par = "1 GPU"
    line = {
        "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "width": W, "height": H, "spp": spp,
                   "rays_per_step": total_rays,
                   "l2": "flushed between steps (256 MiB write, outside the timed window)",
                   "parallelism": par},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "fp64_pipe_active_ncu": pipe_busy,
                     "kernel": "trace_scene_kernel" if scene.s.integrator else "trace_reference_kernel",
                     "kernel_ms": avg_trace_ms, "shade_ms": sum(shade_ms) / len(shade_ms),
                     "peak_source": "K0 fp64 FMA microbenchmark measured in this run "
                                    "(MEASURED_PEAKS.json has no FP64 entry)",
                     "flops_per_launch": sum(flops) / len(flops)},
        "cpu_baseline": cpu,
        "reference_sky_only": ref_sky,
        "reference_harness_gpu": harness,
        "e2e": {"value": e2e_value, "unit": "Mrays/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "FrameRenderer.render (python; pinned host image)"},
        "e2e_dropin": dropin,
        "mpixels_per_s": value / spp,  # BASELINE metric also quotes pixels/s
        "gpu_launches": stats["launches"] * args.steps if stats else None,
        "gpu_launches_per_step": stats["launches"] if stats else None,
        "steps_per_ray": stats["steps"] / stats["rays"] if stats else None,
        "rejected_per_ray": stats["rejected"] / stats["rays"] if stats else None,
        "clocks": clocks,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # CPU samples: the oracle port renders the whole frame (~2 s on 16 cores
    # for config 2); --ref-rows N restricts the reference arm to N centre rows
    ap.add_argument("--cpu-rows", type=int, default=2160)
    ap.add_argument("--ref-rows", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ref-sky", action="store_true",
                    help="skip the reference-harness timings: the compiled reference's sky-only "
                         "lattice (CPU, ~10 s) and the GPU through bhrt_bench_b200 (~10 s)")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference_arm(args)
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus > 1:
            return self_launch(args)
    elif int(env_world) != args.gpus:
        print(f"bench.py: launched with WORLD_SIZE={env_world} but --gpus {args.gpus}; "
              f"they must agree", file=sys.stderr, flush=True)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
