"""The C-ABI library without a GPU: it loads, exports every symbol
include/bhrt_cuda.h declares, its structs match the C compiler's layout,
and the host-only entry points (defaults, validation, bands, tiling,
sphere field) behave like the reference / the oracle."""
import ctypes as C
import os
import re
import subprocess
import textwrap

import numpy as np
import pytest

from oracle_lib import oracle
from paper_2507_16165_b200 import native, scenes
from paper_2507_16165_b200.abi import RayRecord, Scene, Sphere, StatusInfo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bhrt_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bhrt_\w+)\s*\(", src)) - {"bhrt_status", "bhrt_ctx"})


def test_library_loads_and_exports_every_declared_symbol():
    L = native.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) <= set(native.EXPORTS) | {"bhrt_cuda_abi_version"}
    assert L.bhrt_cuda_abi_version() == 1


def test_struct_layout_matches_c(tmp_path):
    fields = [f for f, _ in Scene._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    prog.append('printf("%zu %zu %zu %zu\\n", sizeof(bhrt_scene), sizeof(bhrt_sphere), '
                'sizeof(bhrt_ray_record), sizeof(bhrt_status_info));')
    for f in fields:
        prog.append(f'printf("%zu\\n", offsetof(bhrt_scene, {f}));')
    prog.append("return 0;}")
    c = tmp_path / "probe.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-o", str(exe), str(c)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(x) for x in out[:4]] == [C.sizeof(Scene), C.sizeof(Sphere), C.sizeof(RayRecord),
                                        C.sizeof(StatusInfo)]
    for f, off in zip(fields, out[4:]):
        assert getattr(Scene, f).offset == int(off), f


def test_defaults_agree_python_c_oracle():
    a, b, c = Scene(), Scene(), Scene()
    scenes.scene_defaults(a)
    native.lib().bhrt_scene_defaults(C.byref(b))
    oracle().orc_scene_defaults(C.byref(c))
    assert bytes(a) == bytes(b) == bytes(c)


def test_validation_codes_without_gpu():
    L = native.lib()
    info = StatusInfo()
    sb = scenes.small_scene(scenes.gradient_background(), 4)
    assert L.bhrt_validate_scene(sb.ptr(), C.byref(info)) == 0
    for mutate in (lambda s: setattr(s.s, "spp", 0), lambda s: setattr(s.s, "width", 0),
                   lambda s: s.set(cam_pos=(0, 0, -1.5)), lambda s: s.set_sky(None),
                   lambda s: setattr(s.s, "mass", -1.0)):
        bad = sb.clone()
        mutate(bad)
        assert L.bhrt_validate_scene(bad.ptr(), C.byref(info)) == 1
        assert info.code == 1 and info.message


def test_bands_and_tiles():
    L = native.lib()
    o = oracle()
    rng = np.random.default_rng(1)
    for _ in range(200):
        h, w = int(rng.integers(1, 3000)), int(rng.integers(1, 64))
        n = min(h, w)
        a0, a1, b0, b1 = ((C.c_int32 * n)() for _ in range(4))
        ca, cb = C.c_int32(), C.c_int32()
        assert L.bhrt_make_bands(h, w, a0, a1, n, C.byref(ca)) == 0
        assert o.orc_make_bands(h, w, b0, b1, n, C.byref(cb)) == 0
        assert list(a0) == list(b0) and list(a1) == list(b1)
        # cyclic tiles: counts partition the rows
        T = int(rng.integers(1, 9))
        assert sum(L.bhrt_tile_row_count(0, h, T, w, r) for r in range(w)) == h
    assert L.bhrt_tile_row_count(0, 10, 0, 1, 0) == -1
    assert L.bhrt_make_bands(0, 3, a0, a1, 3, C.byref(ca)) == 6


def test_sphere_field_identical_to_oracle():
    a = scenes.make_spheres()
    b = scenes.make_spheres(lib=oracle())
    assert bytes((Sphere * 64)(*a)) == bytes((Sphere * 64)(*b))


def test_render_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sb = scenes.config(1, 8, 8)
    out = np.zeros(8 * 8 * 3, np.uint8)
    info = StatusInfo()
    rc = native.lib().bhrt_cuda_render_rows(sb.ptr(), 0, 8, None, 0,
                                            out.ctypes.data_as(C.POINTER(C.c_uint8)), out.nbytes,
                                            None, C.byref(info))
    assert rc == 5  # BHRT_DEVICE: no silent CPU fallback


def test_cull_atan2_polynomial_error_bound():
    """trace_scene.cu atan2_cull (window / cull-bin angles only): the odd
    minimax polynomial in the source stays within 2e-6 rad of atan2 over all
    octants in fp32, far inside the 5e-4 rad window margin."""
    src = open(os.path.join(ROOT, "paper_2507_16165_b200", "csrc", "trace_scene.cu")).read()
    body = src[src.index("float atan2_cull"):]
    body = body[:body.index("return copysignf")]
    coef = [np.float32(c) for c in re.findall(r"(-?0\.\d+)f", body)]
    assert len(coef) >= 6
    c = coef[:6]  # innermost first, as written in the Horner chain
    rng = np.random.default_rng(7)
    ang = rng.uniform(-np.pi, np.pi, 400000)
    rad = rng.uniform(1e-3, 1e3, ang.size)
    y = (rad * np.sin(ang)).astype(np.float32)
    x = (rad * np.cos(ang)).astype(np.float32)
    ax, ay = np.abs(x), np.abs(y)
    a = (np.minimum(ax, ay) / np.maximum(ax, ay)).astype(np.float32)
    s = (a * a).astype(np.float32)
    r = np.full_like(s, c[0])
    for k in c[1:]:
        r = (r * s + k).astype(np.float32)
    r = (r * a).astype(np.float32)
    r = np.where(ay > ax, np.float32(1.57079637) - r, r)
    r = np.where(x < 0, np.float32(3.14159274) - r, r)
    r = np.copysign(r, y)
    err = np.abs(r.astype(np.float64) - np.arctan2(y.astype(np.float64), x.astype(np.float64)))
    assert err.max() < 2e-6


def test_trace_rays_host_validation_without_gpu():
    """bhrt_cuda_trace_rays validates like the reference's trace()
    (geodesic.cpp:19-27,166-172) before touching a device."""
    from paper_2507_16165_b200 import geodesic as G
    c = G.TraceConfig()
    with pytest.raises(G.InvalidArgument, match="epsilon"):
        G.trace_batch([(20, 0, 0)], [(0, 1, 0)], G.BlackHole(1.0), G.TraceConfig(epsilon=0.0))
    with pytest.raises(G.InvalidArgument, match="max_windings"):
        G.trace_batch([(20, 0, 0)], [(0, 1, 0)], G.BlackHole(1.0), G.TraceConfig(max_windings=0))
    with pytest.raises(G.InvalidArgument, match="mass"):
        G.trace_batch([(20, 0, 0)], [(0, 1, 0)], G.BlackHole(-1.0), c)
    with pytest.raises(G.InvalidArgument, match="horizon") as e:
        G.trace_batch([(20, 0, 0), (3, 0, 0), (1, 0, 0)], [(0, 1, 0)] * 3, G.BlackHole(2.0), c)
    assert e.value.px == 1
    rec, defl = G.trace_batch(np.zeros((0, 3)), np.zeros((0, 3)), G.BlackHole(1.0), c, deflection=True)
    assert len(rec) == 0 and len(defl) == 0
    with pytest.raises(G.InvalidArgument, match="deflection_angle"):
        G.deflection_angle(0.0)
    # the polyline entry point validates the same way, plus its own arguments
    with pytest.raises(G.InvalidArgument, match="epsilon"):
        G.trace_polylines([(20, 0, 0)], [(0, 1, 0)], G.BlackHole(1.0), G.TraceConfig(epsilon=0.0))
    with pytest.raises(G.InvalidArgument, match="horizon") as e:
        G.trace_polylines([(20, 0, 0), (1, 0, 0)], [(0, 1, 0)] * 2, G.BlackHole(1.0), c)
    assert e.value.px == 1
    with pytest.raises(G.InvalidArgument, match="bad arguments"):
        G.trace_polylines([(20, 0, 0)], [(0, 1, 0)], G.BlackHole(1.0), c, max_points=-1)
    rec, pts = G.trace_polylines(np.zeros((0, 3)), np.zeros((0, 3)), G.BlackHole(1.0), c)
    assert len(rec) == 0 and pts == []


def test_render_rows_rejects_duplicate_devices_without_gpu():
    from paper_2507_16165_b200 import render
    sb = scenes.config(1, 16, 8)
    for devs in ([0, 0], [1, -1]):
        with pytest.raises(render.InvalidArgument, match="device"):
            render.render_rows(sb, 0, 1, devices=devs)


def test_scaled_error_ratio_is_exact(tmp_path):
    """err_ratio() (csrc/trace_reference.cu) divides tiny error terms with the
    numerator scaled by 2^900; mode R's bit parity needs that to equal e / s."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "div_scale_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off",
                    os.path.join(root, "tools", "div_scale_check.c"), "-o", exe, "-lm"], check=True)
    out = subprocess.run([exe, "10000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.startswith("0 mismatches")


def test_sqrt_acceptance_threshold():
    """integrate_window (csrc/trace_reference.cu) tests err2 <= 1 + 2^-52
    instead of sqrt(err2) <= 1: equal for every double near 1 (IEEE sqrt)."""
    x = np.float64(1.0)
    xs = [x]
    lo = hi = x
    for _ in range(64):
        lo = np.nextafter(lo, 0.0)
        hi = np.nextafter(hi, 2.0)
        xs += [lo, hi]
    xs = np.array(xs + [0.0, 1e-300, 0.5, 2.0, np.inf, np.nan])
    with np.errstate(invalid="ignore"):
        assert np.array_equal(np.sqrt(xs) <= 1.0, xs <= 1.0 + 2.0 ** -52)


def test_camera_division_is_exact(tmp_path):
    """camera_ray (csrc/device_common.cuh) forms (px + sx) / width from the
    host's RN(1/width) and one fma correction; every width below 2^16 with
    random and edge numerators must give the IEEE quotient."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "div_check")
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off",
                    os.path.join(root, "tools", "div_check.c"), "-o", exe, "-lm"], check=True)
    out = subprocess.run([exe, "300"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.startswith("0 mismatches")


def test_row_division_magic_is_exact():
    """sample_of (csrc/device_common.cuh) divides the packed pixel index by
    the width as umul64hi(pix, floor(2^64 / width) + 1) (KParams::div_magic);
    exact for every pix < 2^31 (edges of each quotient, random) and width."""
    rng = np.random.default_rng(3)
    widths = list(range(2, 5000)) + [int(w) for w in rng.integers(5000, 1 << 20, 3000)] + [65535, 65536, 7680]
    for d in widths:
        m = (2**64 - 1) // d + 1
        top = (2**31 - 1) // d
        ns = {0, d - 1, d, 2**31 - 1, top * d, top * d - 1}
        ns.update(int(x) for x in rng.integers(0, 2**31 - 1, 20))
        for n in ns:
            assert (n * m) >> 64 == n // d, (n, d)
