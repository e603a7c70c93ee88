"""Ablation timing of the config-2 frame (developer tool): full scene, no
spheres, no disk, sky only, and spp=1 — to split time between integration,
events and per-ray setup."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402


def timeit(sb, reps=3):
    ctx = render.Context(0)
    ctx.set_scene(sb)
    out = torch.empty(sb.s.height * sb.s.width * 3, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    best = 1e30
    for r in range(reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.render_async(out.data_ptr(), stream=st.cuda_stream)
        e1.record(st)
        ctx.finish()
        if r:
            e1.synchronize()  # finish() waits for the render only; the end event may trail it
            best = min(best, e0.elapsed_time(e1))
    s = ctx.stats()
    ctx.close()
    return best, s["steps"] / s["rays"]


def main():
    base = scenes.config(2)
    variants = {"full": base}
    v = base.clone()
    v.set_spheres([])
    variants["no_spheres"] = v
    v = base.clone()
    v.s.disk_enabled = 0
    variants["no_disk"] = v
    v = base.clone()
    v.set_spheres([])
    v.s.disk_enabled = 0
    variants["sky_only"] = v
    for n in (1, 8, 32):
        v = base.clone()
        v.set_spheres(base.spheres[:n])
        variants[f"spheres_{n}"] = v
    v = base.clone()  # one sphere far outside every ray's plane pencil
    far = scenes.Sphere()
    for i, x in enumerate((0.0, 90.0, 0.0)):
        far.center[i] = x
    far.radius = 0.5
    v.set_spheres([far])
    variants["sphere_far"] = v
    for name, sb in variants.items():
        ms, spr = timeit(sb)
        rays = sb.s.width * sb.s.height * sb.s.spp
        print(f"{name:12s} {ms:7.2f} ms  {rays / ms / 1e3:8.1f} Mrays/s  steps/ray {spr:6.2f}  "
              f"ns/step/ray {ms * 1e6 / rays / max(spr, 1e-9):.3f}", flush=True)


if __name__ == "__main__":
    main()
