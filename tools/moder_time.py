"""Device timing of mode R (the reference algorithm) on the sky-only
projection of config 2 at a reduced size (developer tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

w, h, spp = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (960, 540, 1)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
proj = scenes.sky_only_projection(scenes.config(2, w, h))
proj.set(spp=spp)
ctx = render.Context(0)
ctx.set_scene(proj)
buf = torch.empty(w * h * 3, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for r in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    ctx.finish()
    e1.synchronize()  # finish() waits for the render only; the end event may trail it
    ms = e0.elapsed_time(e1)
    s = ctx.stats()
    print(f"modeR {w}x{h}x{spp} rep {r}: {ms:.2f} ms  {s['rays'] / ms / 1e3:.2f} Mrays/s  "
          f"windows/ray {s['steps'] / s['rays']:.1f} rej/ray {s['rejected'] / s['rays']:.2f}", flush=True)
