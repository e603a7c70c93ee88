"""Diagnostic counters of the config-2 frame (needs a -DBHRT_COUNTERS build)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

sb = scenes.config(2)
ctx = render.Context(0)
ctx.set_scene(sb)
out = torch.empty(sb.s.height * sb.s.width * 3, dtype=torch.uint8, device="cuda")
ctx.render_async(out.data_ptr())
ctx.finish()
c = ctx.counters()
rays = c[2]
print(f"rays {rays}  steps/ray {c[0] / rays:.2f}  sphere-event steps/ray {c[4] / rays:.3f}  "
      f"active candidate-steps/ray {c[5] / rays:.3f}  candidates/ray {c[6] / rays:.3f} "
      f"(overflow counted as 100)")
print(f"step_events calls/ray {c[7] / rays:.3f}")
import time
for variant in ("full", "no_spheres"):
    s2 = sb.clone()
    if variant == "no_spheres":
        s2.set_spheres([])
    ctx.set_scene(s2)
    ctx.render_async(out.data_ptr())
    ctx.finish()
    c = ctx.counters()
    print(variant, f"step_events calls/ray {c[7] / rays:.3f} candidates/ray {c[6] / rays:.3f}")
