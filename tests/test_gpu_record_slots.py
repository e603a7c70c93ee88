"""Unfused shading (spp not dividing the warp: the trace kernel writes
per-sample records, shade_kernel reads them) with several renders of one
context in flight on different streams: each render takes its own record
slot (bhrt_ctx_render_async, RecSlot), so concurrent bands cannot overwrite
each other's records. Images must equal the one-shot render."""
import math

import numpy as np
import pytest

from paper_2507_16165_b200 import render, scenes
from paper_2507_16165_b200.abi import INTEGRATOR_REFERENCE

pytestmark = pytest.mark.gpu


def _scenes():
    sb = scenes.config(2, 40, 32)
    sb.set(spp=3)
    bg = scenes.gradient_background(64, 32)
    mr = scenes.small_scene(bg, 40, 1.0)
    mr.set(height=32, spp=3, cam_pos=scenes.inclined_camera(20.0, 80.0, 0.3),
           vertical_fov=math.radians(60.0), epsilon=0.2, integrator=INTEGRATOR_REFERENCE)
    return [sb, mr]


@pytest.mark.parametrize("which", [0, 1])
def test_concurrent_unfused_bands_on_two_streams(which):
    import torch
    sb = _scenes()[which]
    ref = render.render_image(sb).reshape(-1)
    W, H = sb.s.width, sb.s.height
    ctx = render.Context(0)
    ctx.set_scene(sb)
    ctx.set_output_layout(1)  # whole-image buffer, bands land at their rows
    out = torch.zeros(W * H * 3, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    ctx.frame_begin(s2.cuda_stream)
    s1.wait_stream(s2)
    bands = [(y, min(y + 4, H)) for y in range(0, H, 4)]
    for k, (y0, y1) in enumerate(bands):
        ctx.render_async(out.data_ptr(), y0, y1, stream=(s1 if k % 2 else s2).cuda_stream)
    ctx.finish()
    st = ctx.stats()
    ctx.close()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    assert st["rays"] == W * H * 3


def test_back_to_back_unfused_renders():
    import torch
    sb = _scenes()[0]
    ref = render.render_image(sb).reshape(-1)
    ctx = render.Context(0)
    ctx.set_scene(sb)
    for _ in range(6):
        out = torch.zeros(ref.size, dtype=torch.uint8, device="cuda")
        ctx.render_async(out.data_ptr())
        ctx.finish()
        assert np.array_equal(out.cpu().numpy(), ref)
    ctx.close()


@pytest.mark.parametrize("kind", ["rk4", "rkf45", "table", "modeR"])
def test_counter_slots_fold_to_frame_totals(kind):
    """The render counters are spread over line-separated slots (one per
    block mod kStatSlots) and folded on the host: rays = every sample of the
    frame, steps = the sum of the per-sample step counts of the records path
    (integration kernels), over a frame of many blocks and across renders."""
    import torch
    sb = {"rk4": lambda: scenes.config(0, 160, 90), "rkf45": lambda: scenes.config(2, 320, 180),
          "table": lambda: scenes.config(3, 320, 180),
          "modeR": lambda: scenes.sky_only_projection(scenes.config(2, 96, 54))}[kind]()
    W, H, spp = sb.s.width, sb.s.height, sb.s.spp
    ctx = render.Context(0)
    ctx.set_scene(sb)
    out = torch.zeros(W * H * 3, dtype=torch.uint8, device="cuda")
    for _ in range(2):  # the second render starts from reset slots
        ctx.render_async(out.data_ptr())
        ctx.finish()
        st = ctx.stats()
        assert st["rays"] == W * H * spp
    ctx.close()
    if kind != "table":  # table mode records carry no step counts
        _, rec = render.render_rows(sb, 0, H, 1, records=True)
        assert st["steps"] == int(rec["steps"].astype(np.int64).sum())
    assert st["steps"] > 0
