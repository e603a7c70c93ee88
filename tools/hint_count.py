"""How often mode R forms the exact step hint (developer check; needs a
-DBHRT_HINT_COUNT build via BHRT_B200_LIB)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_16165_b200 import native, render, scenes  # noqa: E402
proj = scenes.sky_only_projection(scenes.config(2, 480, 270))
proj.set(spp=1)
ctx = render.Context(0)
ctx.set_scene(proj)
buf = torch.empty(480 * 270 * 3, dtype=torch.uint8, device="cuda")
ctx.render_async(buf.data_ptr())
ctx.finish()
out = (C.c_ulonglong * 4)()
native.lib().bhrt_debug_hint_counts(out)
s = ctx.stats()
print("windows", s["steps"], "exact hints", out[0], "binding", out[1], "in-window re-steps", out[2])
