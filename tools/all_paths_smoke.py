"""Small renders of every kernel path (developer smoke; compute-sanitizer is
not available on the GPU pool): scene kernels (RK4, RKF45 with disk+spheres, overflow), table mode,
mode R, the ray-batch trace, unfused shading and the banded frame path."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2507_16165_b200 import geodesic as G  # noqa: E402
from paper_2507_16165_b200 import parallel, render, scenes  # noqa: E402

for idx, w, h in ((0, 24, 24), (1, 32, 18), (2, 32, 18), (3, 64, 36)):
    sb = scenes.config(idx, w, h)
    if idx == 3:
        sb.set(table_entries=2000, table_samples=256)
    render.render_rows(sb, 0, h)
    render.render_rows(sb, 0, h, records=True)
sb = scenes.config(2, 20, 12)
sb.set(spp=3)
render.render_rows(sb, 0, 12)
bg = scenes.gradient_background()
render.render_rows(scenes.small_scene(bg, 12), 0, 12)
o = np.random.default_rng(1).normal(size=(64, 3)) * 20
d = np.random.default_rng(2).normal(size=(64, 3))
d /= np.linalg.norm(d, axis=1)[:, None]
G.trace_batch(o, d, G.BlackHole(1.0), G.TraceConfig(epsilon=0.2, escape_radius=100.0), deflection=True)
fr = parallel.FrameRenderer()
fr.render(scenes.config(2, 32, 18), bands=4)
print("all paths done")
