"""Scene and ray cases shared by tests/golden/make_golden.py (which renders
them with the compiled reference) and the tests that replay them."""
from __future__ import annotations

import math

from paper_2507_16165_b200 import scenes


def impact_ray(b, r0):
    """test_util.hpp:70-73: in-plane ray with impact parameter b from (r0,0,0)."""
    a = math.asin(b / r0)
    return (r0, 0.0, 0.0), (-math.cos(a), math.sin(a), 0.0)


def image_cases():
    bg = scenes.gradient_background()
    cases = {}
    s = scenes.small_scene(bg, 16)
    s.s.spp = 2
    s.s.seed = 99
    cases["small16_spp2"] = s
    cases["flat24"] = scenes.small_scene(bg, 24, 0.0)
    s = scenes.SceneBuf()  # acceptance.cpp:162-186 geometry, smaller
    s.set(mass=1.0, cam_pos=(0, 0, -1000), cam_look_at=(0, 0, 0), vertical_fov=0.032, width=32,
          height=32, spp=1, seed=1, epsilon=2.0, escape_radius=4000.0, max_windings=10,
          rel_tol=1e-10, abs_tol=1e-12)
    s.set_sky(scenes.gradient_background(32, 16))
    cases["shadow32"] = s
    s = scenes.small_scene(scenes.ring_background(), 32)  # acceptance.cpp:288-321
    s.set(cam_pos=(0, 0, -15))
    cases["ring32"] = s
    cases["c0_skyonly32"] = scenes.sky_only_projection(scenes.config(0, 32, 32),
                                                       256, 128)
    return cases
