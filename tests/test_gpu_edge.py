"""Edge cases of the scene kernels against the CPU oracle (same contract as
tests/test_gpu_parity.py): flat space, a camera beyond the escape sphere,
candidate-slot overflow (the kernel's test-all sphere path), spheres that
contain the hole or the camera, sub-chord refinement extremes, the
non-fused (spp does not divide 32) record path, and ragged image sizes."""
import numpy as np
import pytest

from paper_2507_16165_b200 import scenes
from paper_2507_16165_b200.abi import INTEGRATOR_RK4, Sphere
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu


def sphere(c, r, alb=(0.8, 0.5, 0.2)):
    s = Sphere()
    s.center[:] = c
    s.radius = r
    s.albedo[:] = alb
    return s


@pytest.mark.parametrize("integ", ["rkf45", "rk4"])
def test_flat_space_scene(integ):
    sb = scenes.config(2, 64, 36)
    sb.set(mass=0.0)
    if integ == "rk4":
        sb.set(integrator=INTEGRATOR_RK4, step=2e-3)
    res = compare(sb)
    assert res["steps_equal"]


def test_camera_beyond_escape_sphere():
    """Rays start at u < u_esc moving inward (w > 0): no escape until they
    come back out (geodesic.cpp:204-215 tests u <= u_esc AND u' < 0)."""
    sb = scenes.config(2, 64, 36)
    sb.set(escape_radius=25.0)  # camera at r = 30
    res = compare(sb)
    assert res["steps_equal"]


def test_candidate_overflow_uses_all_spheres():
    """More than 8 candidate spheres in one orbital plane: the kernel falls
    back to testing every sphere on every step (nc = -1). Every orbital plane
    contains the camera-hole axis, so spheres centred on that axis (behind
    the hole) are candidates of every ray; rays bent around the hole hit
    them."""
    sb = scenes.config(2, 48, 27)
    v = np.array(list(sb.s.cam_pos)) - np.array(list(sb.s.center))
    v /= np.linalg.norm(v)
    rng = np.random.default_rng(11)
    sph = [sphere(tuple(-v * (10.0 + 2.5 * k)), 1.0, tuple(rng.random(3))) for k in range(12)]
    sph += [sphere((12.0, 0.5, 4.0), 1.5), sphere((-9.0, -2.0, 8.0), 1.0)]
    sb.set_spheres(sph)
    res = compare(sb)
    assert res["steps_equal"]


def test_spheres_containing_hole_or_camera():
    """A sphere around the camera (every ray starts inside it: no entering
    hit, infinite window) and one around the hole (the whole shadow region)."""
    sb = scenes.config(2, 48, 27)
    cam = tuple(sb.s.cam_pos)
    sb.set_spheres([sphere(cam, 3.0), sphere((0.0, 0.0, 0.0), 4.0, (0.1, 0.9, 0.1)),
                    sphere((12.0, 1.0, 3.0), 2.0)])
    res = compare(sb)
    assert res["steps_equal"]


@pytest.mark.parametrize("chord", [1e-3, 0.2])
def test_sub_chord_refinement_extremes(chord):
    sb = scenes.config(2, 48, 27)
    sb.set(chord_dphi=chord)
    res = compare(sb)
    assert res["steps_equal"]


def test_unfused_record_path_with_spheres():
    sb = scenes.config(2, 40, 24)
    sb.set(spp=3)
    res = compare(sb)
    assert res["steps_equal"]


@pytest.mark.parametrize("wh", [(1, 1), (37, 23), (5, 97)])
def test_ragged_sizes(wh):
    sb = scenes.config(2, *wh)
    res = compare(sb)
    assert res["steps_equal"]


def test_sphere_hits_after_a_full_winding():
    """Rays with impact parameter just above the critical one wind around
    the hole before escaping; small spheres hugging the photon sphere are
    then hit on a later winding, where the kernel tests a candidate window's
    k-th occurrence (window_at: the list keeps the first, rays derive the one
    in use). Same objects and hit points as the oracle, and some hits come
    after more than one full turn."""
    sb = scenes.config(2, 96, 96)
    sb.set(disk_enabled=0, cam_pos=scenes.inclined_camera(12.0, 60.0), vertical_fov=0.9)
    rng = np.random.default_rng(5)
    sph = []
    for _ in range(40):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        sph.append(sphere(tuple(d * rng.uniform(3.4, 4.2)), float(rng.uniform(0.15, 0.35)),
                          tuple(rng.random(3))))
    sb.set_spheres(sph)
    res = compare(sb)
    assert res["steps_equal"]
    from paper_2507_16165_b200 import render
    from paper_2507_16165_b200.abi import OBJ_SPHERE
    _, rec = render.render_rows(sb, 0, sb.s.height, 1, records=True)
    late = (rec["object"] == OBJ_SPHERE) & (rec["phi"] > 2.0 * np.pi)
    assert late.sum() > 0, "no sphere hit after a full winding"
