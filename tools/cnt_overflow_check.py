import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from paper_2507_16165_b200 import render, scenes
from test_gpu_edge import sphere
sb = scenes.config(2, 48, 27)
v = np.array(list(sb.s.cam_pos)) - np.array(list(sb.s.center)); v /= np.linalg.norm(v)
sb.set_spheres([sphere(tuple(-v * (10.0 + 2.5 * k)), 1.0) for k in range(12)])
ctx = render.Context(0); ctx.set_scene(sb)
out = torch.empty(48*27*3, dtype=torch.uint8, device="cuda")
ctx.render_async(out.data_ptr()); ctx.finish()
c = ctx.counters(); print("rays", c[2], "candidates (overflow counted 100)", c[6], "per ray", c[6]/c[2])
