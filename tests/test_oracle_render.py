"""Camera, sky sampling and render known-answer tests of the reference
(test_camera.cpp, test_image.cpp, test_render.cpp, acceptance.cpp 1,5,6,9)
restated against the CPU oracle."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle_lib import d3, dbuf, oracle, orc_render
from paper_2507_16165_b200 import scenes
from paper_2507_16165_b200.abi import StatusInfo

PI = math.pi


def cam_scene(w, h, fov_deg=90.0, spp=1, seed=0):
    sb = scenes.SceneBuf()
    sb.set(cam_pos=(0, 0, -5), cam_look_at=(0, 0, 0), vertical_fov=fov_deg * PI / 180.0,
           width=w, height=h, spp=spp, seed=seed)
    return sb


def ray(sb, px, py, s=0):
    o, d = dbuf(3), dbuf(3)
    rc = oracle().orc_generate_ray(sb.ptr(), px, py, s, o, d)
    return rc, np.array(list(d))


def basis(sb):
    f, r, u = dbuf(3), dbuf(3), dbuf(3)
    rc = oracle().orc_camera_basis(sb.ptr(), f, r, u)
    return rc, np.array(list(f)), np.array(list(r)), np.array(list(u))


# ------------------------------------------------------------------ camera
def test_centre_pixel_looks_forward():  # test_camera.cpp:19-25
    sb = cam_scene(9, 9)
    _, f, _, _ = basis(sb)
    assert np.linalg.norm(ray(sb, 4, 4)[1] - f) < 1e-12


def test_jitter_deterministic_and_seeded():  # test_camera.cpp:27-42, 100-106
    sb = cam_scene(16, 16, spp=8, seed=12345)
    for s in range(8):
        assert np.array_equal(ray(sb, 3, 7, s)[1], ray(sb, 3, 7, s)[1])
    other = cam_scene(16, 16, spp=8, seed=999)
    assert np.linalg.norm(ray(sb, 3, 7, 1)[1] - ray(other, 3, 7, 1)[1]) > 0
    one = cam_scene(8, 8, spp=1, seed=1)
    two = cam_scene(8, 8, spp=1, seed=777)
    assert np.array_equal(ray(one, 2, 3)[1], ray(two, 2, 3)[1])


def test_unit_norm_and_mirror_symmetry():  # test_camera.cpp:55-79
    sb = cam_scene(13, 7, 70.0, spp=4, seed=5)
    for py in range(7):
        for px in range(13):
            for s in range(4):
                assert abs(np.linalg.norm(ray(sb, px, py, s)[1]) - 1) < 1e-12
    sb = cam_scene(16, 16, 75.0)
    _, f, r, u = basis(sb)
    for px in range(16):
        a, b = ray(sb, px, 5)[1], ray(sb, 15 - px, 5)[1]
        assert a @ r == pytest.approx(-(b @ r), rel=1e-12)
        assert a @ u == pytest.approx(b @ u, rel=1e-12)


def test_row_zero_is_top_and_degenerate_cameras():  # test_camera.cpp:81-98
    sb = cam_scene(9, 9)
    _, f, r, u = basis(sb)
    assert ray(sb, 4, 0)[1] @ u > 0 and ray(sb, 4, 8)[1] @ u < 0
    sb.set(cam_look_at=(0, 0, -5))
    assert basis(sb)[0] == 6
    sb = cam_scene(4, 4)
    sb.set(cam_pos=(0, -3, 0), cam_look_at=(0, 1, 0))
    assert basis(sb)[0] == 6


def test_hash_counter_reference_definition():  # camera.cpp:10-28
    def splitmix(x):
        M = (1 << 64) - 1
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    for seed, a, b, c in [(0, 0, 0, 0), (77, 3, 9, 5), (2**63 + 11, 12, 34, 56)]:
        h = splitmix(splitmix(splitmix(splitmix(seed) ^ a) ^ b) ^ c)
        assert oracle().orc_hash_counter(seed, a, b, c) == h


# ------------------------------------------------------------------ sky
def sample(img, d):
    o = dbuf(3)
    h, w = img.shape[:2]
    oracle().orc_sample_direction(np.ascontiguousarray(img).ctypes.data_as(C.POINTER(C.c_uint8)),
                                  w, h, d3(d), o)
    return np.array(list(o))


def test_sample_direction_uniform_poles_seam():  # test_image.cpp:86-127
    c = sample(scenes.uniform_background(90, 160, 210), (1, 0, 0))
    assert np.allclose(c, np.array([90, 160, 210]) / 255.0, rtol=1e-12)
    img = np.zeros((3, 4, 3), np.uint8)
    img[0, :, 0] = 200
    img[1, :, 1] = 200
    img[2, :, 2] = 200
    assert sample(img, (0, 1, 0))[0] == pytest.approx(200 / 255.0, rel=1e-12)
    assert sample(img, (0, -1, 0))[2] == pytest.approx(200 / 255.0, rel=1e-12)
    g = scenes.gradient_background(32, 16)
    v1 = np.array([-1.0, 0.1, -1e-9])
    v2 = np.array([-1.0, 0.1, 1e-9])
    assert np.abs(sample(g, v1 / np.linalg.norm(v1)) - sample(g, v2 / np.linalg.norm(v2))).max() < 1e-6


def test_sample_direction_range():  # test_image.cpp:141-153
    g = scenes.gradient_background()
    rng = np.random.default_rng(7)
    for _ in range(500):
        d = rng.uniform(-1, 1, 3)
        if np.linalg.norm(d) < 1e-3:
            continue
        c = sample(g, d / np.linalg.norm(d))
        assert (c >= 0).all() and (c <= 1).all()


# ------------------------------------------------------------------ render
def render(sb, threads=2, rows=None):
    rc, img, info, _ = orc_render(sb.s, rows, threads=threads)
    assert rc == 0, info.message
    return img.reshape(-1, sb.s.width, 3)


def test_make_bands():  # test_render.cpp:11-48
    L = oracle()

    def bands(h, w):
        n = min(h, w)
        rs = (C.c_int * n)()
        re = (C.c_int * n)()
        cnt = C.c_int()
        assert L.orc_make_bands(h, w, rs, re, n, C.byref(cnt)) == 0
        return [(rs[i], re[i]) for i in range(cnt.value)]

    assert bands(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert bands(4, 1) == [(0, 4)]
    assert bands(2, 5) == [(0, 1), (1, 2)]
    rng = np.random.default_rng(4242)
    for _ in range(300):
        h, w = int(rng.integers(1, 10001)), int(rng.integers(1, 10001))
        b = bands(h, w)
        assert len(b) == min(h, w) and b[0][0] == 0 and b[-1][1] == h
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        sizes = [e - s for s, e in b]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def direct_projection(sb):
    bg = sb.sky
    out = np.zeros((sb.s.height, sb.s.width, 3), np.int64)
    for py in range(sb.s.height):
        for px in range(sb.s.width):
            c = sample(bg, ray(sb, px, py)[1])
            out[py, px] = [int(math.floor(v * 255.0 + 0.5)) for v in c]
    return out


def test_flat_space_identity():  # test_render.cpp:50-66,131-144, acceptance.cpp:70-92
    sb = scenes.small_scene(scenes.gradient_background(), 12, 0.0)
    assert np.abs(render(sb).astype(int) - direct_projection(sb)).max() <= 1


def test_dead_centre_black():  # test_render.cpp:68-75
    sb = scenes.small_scene(scenes.uniform_background(200, 200, 200), 9)
    assert render(sb)[4, 4].tolist() == [0, 0, 0]


def test_shadow_radius():  # test_render.cpp:77-97, acceptance.cpp:162-186 (5%)
    sb = scenes.SceneBuf()
    sb.set(mass=1.0, cam_pos=(0, 0, -1000), cam_look_at=(0, 0, 0), vertical_fov=0.032, width=64,
           height=64, spp=1, epsilon=2.0, escape_radius=4000.0, rel_tol=1e-10, abs_tol=1e-12)
    sb.set_sky(scenes.gradient_background(32, 16))
    img = render(sb, threads=8)
    black = int((img.reshape(-1, 3).sum(axis=1) == 0).sum())
    measured = math.sqrt(black / PI) * (2 * math.tan(0.016) / 64)
    predicted = 3 * math.sqrt(3) / 1000.0
    assert abs(measured - predicted) / predicted <= 0.05


def test_band_slices_and_thread_determinism():  # test_render.cpp:99-129, acceptance.cpp:193-210
    sb = scenes.small_scene(scenes.gradient_background(), 16)
    sb.s.spp = 2
    sb.s.seed = 99
    base = render(sb, 1)
    for t in (2, 4, 8):
        assert np.array_equal(render(sb, t), base)
    for r0, r1 in [(0, 1), (1, 3), (5, 16)]:
        assert np.array_equal(render(sb, 2, (r0, r1)), base[r0:r1])


def test_render_error_lowest_pixel():  # test_render.cpp:146-161
    sb = scenes.small_scene(scenes.gradient_background(), 4, 0.0)
    sb.s.rel_tol = 1e-300
    sb.s.abs_tol = 1e-300
    rc, img, info, _ = orc_render(sb.s, threads=4)
    assert rc == 3 and (info.px, info.py) == (0, 0)
    assert b"pixel (0, 0)" in info.message


def test_validation():  # test_render.cpp:163-171, render.cpp:11-20,68-75
    L = oracle()
    sb = scenes.small_scene(scenes.gradient_background(), 4)
    sb.s.cam_pos[2] = -1.5
    info = StatusInfo()
    assert L.orc_validate_scene(sb.ptr(), C.byref(info)) == 1
    nob = scenes.small_scene(None, 4)
    assert L.orc_validate_scene(nob.ptr(), C.byref(info)) == 1
    ok = scenes.small_scene(scenes.gradient_background(), 4)
    assert orc_render(ok.s, (0, 5))[0] == 6
    assert orc_render(ok.s, (0, 0))[0] == 0  # empty range renders nothing


def test_rounding_half_away():  # test_render.cpp:173-183
    sb = scenes.small_scene(scenes.uniform_background(100, 100, 100), 3, 0.0)
    sb.s.spp = 4
    sb.s.seed = 3
    assert render(sb)[1, 1].tolist() == [100, 100, 100]


def test_ring_symmetry():  # acceptance.cpp:288-321
    sb = scenes.small_scene(scenes.ring_background(), 32)
    sb.set(cam_pos=(0, 0, -15))
    img = render(sb, 8).astype(int)
    n = 32
    for y in range(n):
        for x in range(n):
            assert np.abs(img[y, x] - img[x, n - 1 - y]).max() <= 1
