"""Scene text: bhrt_scene_parse_text / _format_text
against the reference's own config code (config.cpp parse_kv /
serialize_scene / parse_scene, through the compiled reference in
oracle/_ref) — CPU only, no GPU needed."""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import have_ref, ref
from paper_2507_16165_b200 import native, scenes
from paper_2507_16165_b200.abi import (BHRT_USAGE, INTEGRATOR_RK4, INTEGRATOR_TABLE, SKY_CHECKER,
                                       Scene, StatusInfo)

REF_FIELDS = ["mass", "center", "cam_pos", "cam_look_at", "vertical_fov", "width", "height", "spp",
              "seed", "epsilon", "escape_radius", "max_windings", "rel_tol", "abs_tol"]
EXT_FIELDS = ["integrator", "sky_kind", "step", "max_step", "chord_dphi", "checker_nu", "checker_nv",
              "checker_color_a", "checker_color_b", "disk_enabled", "n_spheres", "disk_color_in",
              "disk_color_out", "light_dir", "ambient", "table_entries", "table_samples",
              "table_b_max", "table_dpsi"]


def val(s, f):
    v = getattr(s, f)
    return tuple(v) if isinstance(v, C.Array) else v


def same_fields(a, b, fields):
    for f in fields:
        assert val(a, f) == val(b, f), f


def roundtrip(sb):
    back = scenes.SceneBuf.from_text(sb.to_text())
    same_fields(sb.s, back.s, REF_FIELDS + EXT_FIELDS)
    if sb.s.disk_enabled:
        assert (back.s.disk_r_in, back.s.disk_r_out) == (sb.s.disk_r_in, sb.s.disk_r_out)
    for a, b in zip(sb.spheres, back.spheres):
        assert tuple(a.center) == tuple(b.center) and a.radius == b.radius
        assert tuple(a.albedo) == tuple(b.albedo)
    return back


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
def test_configs_roundtrip_bit_exact(idx):
    roundtrip(scenes.config(idx))


def test_odd_values_roundtrip():
    sb = scenes.config(2)
    sb.set(mass=0.1 + 0.2, cam_pos=(1e-300, -0.0, 5e300), seed=2**64 - 1, vertical_fov=np.pi / 3,
           integrator=INTEGRATOR_TABLE, table_entries=12345, ambient=1.0 / 3.0, chord_dphi=7e-3,
           checker_nu=5, checker_nv=3)
    back = roundtrip(sb)
    assert back.s.seed == 2**64 - 1


def test_generated_sphere_field_equals_make_spheres():
    base = scenes.config(2)
    lines = [l for l in base.to_text().splitlines() if not l.startswith("sphere.")]
    sb = scenes.SceneBuf.from_text("\n".join(lines + ["spheres = 64,2507"]))
    want = scenes.make_spheres()
    assert sb.s.n_spheres == 64
    for a, b in zip(sb.spheres, want):
        assert tuple(a.center) == tuple(b.center) and a.radius == b.radius


def test_reference_only_scene_and_comments():
    text = scenes.config(0).to_text()
    ref_lines = [l for l in text.splitlines() if "=" in l][:14]
    noisy = "# a comment\n\n" + "\n".join("  " + l.replace("=", " = ") + "  " for l in ref_lines)
    sb = scenes.SceneBuf.from_text(noisy)
    d = scenes.SceneBuf()
    same_fields(sb.s, d.s, EXT_FIELDS)  # extensions stay at the defaults


@pytest.mark.parametrize("text,msg", [
    ("mass=1\n", "scene config: missing key 'center'"),
    ("no equals sign", "config: expected key=value, got 'no equals sign'"),
    ("=3", "config: empty key in '=3'"),
])
def test_malformed_text_is_a_usage_error(text, msg):
    with pytest.raises(native.BhrtError) as e:
        scenes.SceneBuf.from_text(text)
    assert e.value.code == BHRT_USAGE and msg in str(e.value)


def test_bad_values_are_usage_errors():
    good = scenes.config(1).to_text()
    for key, bad, msg in (("mass", "abc", "invalid mass: 'abc' is not a number"),
                          ("center", "1,2", "invalid center: expected 'x,y,z', got '1,2'"),
                          ("width", "1.5", "invalid width: '1.5' is not an integer"),
                          ("integrator", "euler", "invalid integrator")):
        text = good + f"\n{key}={bad}\n"  # later keys win (config.hpp)
        with pytest.raises(native.BhrtError) as e:
            scenes.SceneBuf.from_text(text)
        assert e.value.code == BHRT_USAGE and msg in str(e.value)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_reference_scene_formats_exactly_like_serialize_scene():
    for idx in (0, 1, 2):
        sb = scenes.config(idx)
        ours = sb.to_text()
        n = ref().ref_serialize_scene(sb.ptr(), None, 0)
        buf = C.create_string_buffer(n + 1)
        ref().ref_serialize_scene(sb.ptr(), buf, n + 1)
        theirs = buf.value.decode()
        assert ours.startswith(theirs)  # reference keys first, byte for byte
        plain = scenes.SceneBuf()
        for f in REF_FIELDS:
            setattr(plain.s, f, getattr(sb.s, f))
        assert plain.to_text() == theirs  # no extensions -> identical text


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_reference_parser_reads_extended_text():
    """The reference's parse_scene accepts our extended text (unknown keys
    are ignored) and recovers the same SceneConfig fields."""
    for idx in (2, 3, 4):
        sb = scenes.config(idx)
        out = Scene()
        info = StatusInfo()
        assert ref().ref_parse_scene(sb.to_text().encode(), C.byref(out), C.byref(info)) == 0
        same_fields(sb.s, out, REF_FIELDS)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_error_messages_match_reference_parser():
    good = scenes.config(1).to_text()
    for text in ("mass=1\n", "no equals sign", "=3", good + "\nmass=abc\n", good + "\ncenter=1,2\n",
                 good + "\nheight=7x\n", good + "\nseed=-1\n"):
        info_r, info_o = StatusInfo(), StatusInfo()
        rc_r = ref().ref_parse_scene(text.encode(), C.byref(Scene()), C.byref(info_r))
        rc_o = native.lib().bhrt_scene_parse_text(text.encode(), C.byref(Scene()), None, 0, None,
                                                  C.byref(info_o))
        assert rc_r == rc_o == BHRT_USAGE
        assert info_r.message == info_o.message


def test_checker_and_rk4_keys():
    sb = scenes.config(0)
    assert sb.s.integrator == INTEGRATOR_RK4 and sb.s.sky_kind == SKY_CHECKER
    text = sb.to_text()
    assert "integrator=rk4" in text and "sky=checker" in text and "disk=" in text
