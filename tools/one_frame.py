"""Render config C once after one warm-up frame (for ncu captures; developer tool).

    python tools/one_frame.py C             # BASELINE config C
    python tools/one_frame.py R W H         # mode R: sky-only projection of config 2 at W x H
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

if sys.argv[1] == "R":
    sb = scenes.sky_only_projection(scenes.config(2, int(sys.argv[2]), int(sys.argv[3])))
else:
    sb = scenes.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
ctx = render.Context(0)
ctx.set_scene(sb)
out = torch.empty(sb.s.height * sb.s.width * 3, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for i in range(2):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.render_async(out.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    ctx.finish()
    e1.synchronize()  # finish() waits for the render only; the end event may trail it
    print(f"frame {i}: {e0.elapsed_time(e1):.3f} ms", ctx.stats())
