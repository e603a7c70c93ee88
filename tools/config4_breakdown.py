"""Config 4 (120-frame orbit) timing breakdown: host set_scene time per
frame, device kernel time per frame, and the pipelined frames/s
(developer tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

frames = 120
scs = [scenes.config(4, frame=f) for f in range(frames)]
ctx = render.Context(0)
ctx.set_timing(True)
buf = torch.empty(scs[0].s.width * scs[0].s.height * 3, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for f in range(3):
    ctx.set_scene(scs[f])
    ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
    ctx.finish()
hs, ks = [], []
for f in range(frames):
    t0 = time.perf_counter()
    ctx.set_scene(scs[f])
    hs.append(time.perf_counter() - t0)
    ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
    ctx.finish()
    ks.append(ctx.kernel_ms()[0])
print(f"set_scene host: mean {1e3 * sum(hs) / frames:.3f} ms, max {1e3 * max(hs):.3f} ms")
print(f"trace kernel:   mean {sum(ks) / frames:.3f} ms, min {min(ks):.3f}, max {max(ks):.3f} ms")
print(f"serial sum:     {1e3 * sum(hs) + sum(ks):.1f} ms for {frames} frames")
