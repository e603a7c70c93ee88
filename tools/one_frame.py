"""Render config C once after one warm-up frame (for ncu captures; developer tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sb = scenes.config(idx)
ctx = render.Context(0)
ctx.set_scene(sb)
out = torch.empty(sb.s.height * sb.s.width * 3, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ctx.render_async(out.data_ptr())
    ctx.finish()
print("ok", ctx.stats())
