"""Render config 2 with all 64 spheres, then with none (one launch each), for
an ncu metrics comparison of the two launches (developer tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

base = scenes.config(2)
nosph = base.clone()
nosph.set_spheres([])
ctx = render.Context(0)
out = torch.empty(base.s.height * base.s.width * 3, dtype=torch.uint8, device="cuda")
for sb in (base, nosph):
    ctx.set_scene(sb)
    ctx.render_async(out.data_ptr())
    ctx.finish()
print("ok")
