"""Config-4 orbit (120 frames of 1080p x 4 spp) frames/s under different
pipelining choices (developer tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402

frames = 120
scs = [scenes.config(4, frame=f) for f in range(frames)]
W, H = scs[0].s.width, scs[0].s.height


def run(nctx, nstreams):
    ctxs = [render.Context(0) for _ in range(nctx)]
    bufs = [torch.empty(W * H * 3, dtype=torch.uint8, device="cuda") for _ in range(nctx)]
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for f in range(2 * nctx):  # warm-up
        c = ctxs[f % nctx]
        c.set_scene(scs[f])
        c.render_async(bufs[f % nctx].data_ptr(), stream=streams[f % nstreams].cuda_stream)
        c.finish()
    torch.cuda.synchronize()
    t_set = 0.0
    t0 = time.perf_counter()
    for f, sb in enumerate(scs):
        c = ctxs[f % nctx]
        ta = time.perf_counter()
        c.set_scene(sb)
        t_set += time.perf_counter() - ta
        c.render_async(bufs[f % nctx].data_ptr(), stream=streams[f % nstreams].cuda_stream)
        if f >= nctx - 1:
            ctxs[(f - nctx + 1) % nctx].finish()
    for f in range(max(0, frames - nctx + 1), frames):
        ctxs[f % nctx].finish()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for c in ctxs:
        c.close()
    print(f"contexts {nctx} streams {nstreams}: {frames / dt:.1f} frames/s ({dt * 1e3 / frames:.3f} ms/frame, "
          f"set_scene {t_set * 1e3 / frames:.3f} ms/frame)", flush=True)


st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx = render.Context(0)
buf = torch.empty(W * H * 3, dtype=torch.uint8, device="cuda")
tot = 0.0
for sb in scs:
    ctx.set_scene(sb)
    e0.record(st)
    ctx.render_async(buf.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    ctx.finish()
    e1.synchronize()
    tot += e0.elapsed_time(e1)
ctx.close()
print(f"kernel-only sum: {tot / frames:.3f} ms/frame ({frames * 1e3 / tot:.1f} frames/s)")
for nctx, nst in ((3, 3), (4, 4), (6, 6), (8, 8)):
    run(nctx, nst)
