#!/usr/bin/env python
"""Benchmark of the Schwarzschild ray-tracing hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step = one full frame of BASELINE.json configs[C] (default C=2: 3840x2160,
4 jittered spp, disk + 64 spheres, RKF45 tol 1e-9) rendered by all ranks
(cyclic row tiles) and gathered to rank 0 over NCCL. Prints ONE JSON line on
rank 0. Metric: Mrays/s (rays = pixels x spp), whole job.

--impl reference times the CPU implementation of the same workload on the
host cores (rank 0 only): the oracle port of the full scene (the reference
itself cannot render disk/spheres/RKF45 — SPEC.md:14,171), kind "port".
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


def reference_sky_only(scene, rows: int, threads: int):
    """The compiled reference (oracle/_ref) on the sky-only projection of the
    workload (its own render_rows)."""
    import ctypes as C
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import have_ref, ref
    from paper_2507_16165_b200 import scenes
    from paper_2507_16165_b200.abi import StatusInfo
    if not have_ref():
        return None
    proj = scenes.sky_only_projection(scene)
    r0, r1 = centre_band(proj.s.height, rows)
    out = np.zeros((r1 - r0) * proj.s.width * 3, np.uint8)
    info = StatusInfo()
    t0 = time.perf_counter()
    rc = ref().ref_render_rows(C.byref(proj.s), r0, r1, threads,
                               out.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(info))
    dt = time.perf_counter() - t0
    if rc:
        return None
    rays = (r1 - r0) * proj.s.width * proj.s.spp
    return {"value": rays / dt / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "reference",
            "sample": f"oracle/_ref render_rows (the reference's own code), sky-only projection "
                      f"of the workload (DOPRI5 eps=0.05 windows, checker baked into a 2048x1024 "
                      f"PPM), rows [{r0},{r1}) = {rays} rays, {dt:.1f} s"}


def measure_secondary(device: int, reps: int = 3, rank: int = 0, world: int = 1) -> dict:
    """Device-timed Mrays/s of configs 0, 1, 3 (scene resident, best of
    `reps` after one warm-up) and config 4's whole 120-frame orbit (frames/s,
    wall clock, per-frame scene upload + cull table included; with N ranks
    the frames are sharded f mod N and the whole-box rate uses the slowest
    rank). Everything but config 4 runs on rank 0 only."""
    import torch
    import torch.distributed as dist

    from paper_2507_16165_b200 import render, scenes
    out = {}
    ctx = render.Context(device)
    st = torch.cuda.current_stream()
    for idx in (0, 1, 3) if rank == 0 else ():
        sb = scenes.config(idx)
        t0 = time.perf_counter()
        ctx.set_scene(sb)
        setup_s = time.perf_counter() - t0
        buf = torch.empty(sb.s.width * sb.s.height * 3, dtype=torch.uint8, device="cuda")
        best = None
        for r in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
            e1.record(st)
            ctx.finish()
            ms = e0.elapsed_time(e1)
            if r > 0 and (best is None or ms < best):
                best = ms
        rays = sb.s.width * sb.s.height * sb.s.spp
        out[f"config{idx}"] = {"ms": best, "Mrays/s": rays / best / 1e3,
                               "steps_per_ray": ctx.stats()["steps"] / rays,
                               "set_scene_s": setup_s, "size": [sb.s.width, sb.s.height, sb.s.spp]}
    frames = 120
    sb0 = scenes.config(4, frame=0)
    buf = torch.empty(sb0.s.width * sb0.s.height * 3, dtype=torch.uint8, device="cuda")
    for f in range(2):  # warm-up
        ctx.set_scene(scenes.config(4, frame=f))
        ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
        ctx.finish()
    scs = [scenes.config(4, frame=f) for f in range(frames)]
    # two contexts in turn: frame f+1's scene upload (cull table on the host,
    # async copies) proceeds while frame f renders; frames stay in order on
    # one stream and each finish() waits for its own frame only
    ctx2 = render.Context(device)
    bufs = [buf, torch.empty_like(buf)]
    ctxs = [ctx, ctx2]
    mine = scs[rank::world]  # frame sharding f mod N (BASELINE.json config 4)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for f, sb in enumerate(mine):
        c = ctxs[f % 2]
        c.set_scene(sb)
        c.render_async(bufs[f % 2].data_ptr(), stream=st.cuda_stream)
        if f > 0:
            ctxs[(f - 1) % 2].finish()
    if mine:
        ctxs[(len(mine) - 1) % 2].finish()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        tdt = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(tdt, op=dist.ReduceOp.MAX)
        dt = float(tdt.item())
    ctx2.close()
    out["config4"] = {"frames": frames, "seconds": dt, "frames/s": frames / dt,
                      "Mrays/s": frames * sb0.s.width * sb0.s.height * sb0.s.spp / dt / 1e6,
                      "size": [sb0.s.width, sb0.s.height, sb0.s.spp], "n_gpus": world,
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
    ms = e0.elapsed_time(e1)
    rays = proj.s.width * proj.s.height * proj.s.spp
    out["modeR_sky_only"] = {"ms": ms, "Mrays/s": rays / ms / 1e3,
                             "windows_per_ray": ctx.stats()["steps"] / rays,
                             "size": [proj.s.width, proj.s.height, proj.s.spp],
                             "note": "trace_reference_kernel (reference algorithm, bit-identical "
                                     "window arithmetic) on the full sky-only projection; compare "
                                     "reference_sky_only (the reference on the host cores)"}
    ctx.close()
    return out


# ---------------------------------------------------------------- arms
def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_2507_16165_b200 import scenes
    scene = scenes.config(args.config)
    threads = os.cpu_count() or 1
    rows = args.ref_rows
    band = centre_band(scene.s.height, rows)
    for _ in range(args.warmup):
        cpu_port_rows(scene, (band[0], band[0] + 1), threads)
    tot_rays, tot_s = 0, 0.0
    per = []
    for _ in range(args.steps):
        rays, dt = cpu_port_rows(scene, band, threads)
        tot_rays += rays
        tot_s += dt
        per.append(dt)
    value = tot_rays / tot_s / 1e6
    sample = (f"oracle port (C, pthreads) of the full workload, centre rows [{band[0]},{band[1]}) "
              f"= {tot_rays // args.steps} rays per step")
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": value, "unit": "Mrays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "width": scene.s.width,
                   "height": scene.s.height, "spp": scene.s.spp, "parallelism": f"cpu x{threads}"},
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2507_16165_b200 import native, roofline, scenes
    from paper_2507_16165_b200.abi import Scene, Sphere
    from paper_2507_16165_b200.parallel import FrameRenderer

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
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
    h2d = C.sizeof(Scene) + C.sizeof(Sphere) * scene.s.n_spheres
    if scene.s.sky_kind == 0 and scene.sky is not None:
        h2d += scene.sky.nbytes
    d2h = W * H * 3 if rank == 0 else 0

    if rank != 0:
        dist.barrier() if world > 1 else None
        dist.destroy_process_group() if world > 1 else None
        return 0

    # ---- roofline of the dominant kernel (trace), FP64 pipe
    peak = native.lib().bhrt_b200_fp64_peak_tflops(200000, 3, None)
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

    # ---- the other BASELINE.json configs (secondary lines, rank 0, this GPU)
    secondary = None
    if not args.no_secondary:
        secondary = measure_secondary(local, rank=rank, world=world)

    # ---- CPU baseline on this box's host cores (rank 0, N=1 only)
    cpu = None
    ref_sky = None
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        band = centre_band(H, args.cpu_rows)
        rays, dt = cpu_port_rows(scene, band, threads)
        cpu = {"value": rays / dt / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "port",
               "sample": f"oracle port (C, pthreads) of the full workload, centre rows "
                         f"[{band[0]},{band[1]}) = {rays} rays, {dt:.1f} s"}
        ref_sky = reference_sky_only(scene, args.ref_sky_rows, threads)

    line = {
        "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "width": W, "height": H, "spp": spp,
                   "rays_per_step": total_rays,
                   "l2": "flushed between steps (256 MiB write, outside the timed window)",
                   "parallelism": f"cyclic rows x{world} + NCCL gather" if world > 1 else "1 GPU"},
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
        "e2e": {"value": e2e_value, "unit": "Mrays/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
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
    # CPU samples: rows of the workload around the frame centre (the whole
    # 2160-row frame is ~3 s on 16 cores for the port; the reference's own
    # epsilon-window path is ~1e5x slower, so it gets 2 rows)
    ap.add_argument("--cpu-rows", type=int, default=2160)
    ap.add_argument("--ref-rows", type=int, default=540)
    ap.add_argument("--ref-sky-rows", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
