"""Seeded random scenes (camera radius/inclination/azimuth, field of view,
disk extent, sphere fields of random size and density, tolerances, chord
refinement, spp, RK4 or RKF45) rendered on the GPU and by the CPU oracle:
the parity contract of tests/test_gpu_parity.py must hold on every one. The
conservative culling (plane-angle table, fp32 windows, Hermite radial range)
is what these exercise most: a culling bug shows up as a missed sphere hit."""
import math

import numpy as np
import pytest

from paper_2507_16165_b200 import scenes
from paper_2507_16165_b200.abi import INTEGRATOR_RK4, INTEGRATOR_RKF45, Sphere
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu


def random_scene(seed):
    rng = np.random.default_rng(seed)
    sb = scenes.config(2, int(rng.integers(24, 48)), int(rng.integers(14, 30)))
    r = rng.uniform(12.0, 45.0)
    incl = rng.uniform(20.0, 89.0)
    psi = rng.uniform(0.0, 2 * math.pi)
    sb.set(cam_pos=scenes.inclined_camera(r, incl, psi),
           vertical_fov=math.radians(rng.uniform(30.0, 90.0)),
           spp=int(rng.choice([1, 2, 3, 4, 8])), seed=int(rng.integers(1, 1 << 30)),
           disk_enabled=int(rng.random() < 0.8), disk_r_in=rng.uniform(3.0, 8.0),
           disk_r_out=rng.uniform(10.0, 35.0), chord_dphi=float(rng.choice([0.003, 0.01, 0.05])),
           escape_radius=float(rng.choice([60.0, 100.0, 300.0])))
    if rng.random() < 0.25:
        sb.set(integrator=INTEGRATOR_RK4, step=float(rng.choice([2e-3, 5e-3])))
    else:
        tol = float(rng.choice([1e-7, 1e-9, 1e-11]))
        sb.set(integrator=INTEGRATOR_RKF45, rel_tol=tol, abs_tol=tol)
    n = int(rng.choice([0, 1, 5, 20, 64, 120]))
    sph = []
    for _ in range(n):
        s = Sphere()
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        s.center[:] = tuple(d * rng.uniform(4.0, 45.0))
        s.radius = rng.uniform(0.2, 4.0)
        s.albedo[:] = tuple(rng.random(3))
        sph.append(s)
    sb.set_spheres(sph)
    return sb


@pytest.mark.parametrize("seed", range(96))
def test_random_scene_matches_oracle(seed):
    sb = random_scene(1000 + seed)
    res = compare(sb)
    assert res["steps_equal"]


@pytest.mark.parametrize("seed", range(12))
def test_random_reference_mode_scene_matches_compiled_reference(seed):
    """Mode R (the reference's algorithm) on random reference scenes vs the
    compiled reference's own render_rows: pixels exact except <= 0.1% at +-1
    (north-star contract; the PI factor's pow may move a step)."""
    from oracle_lib import have_ref, orc_render, ref_render
    from paper_2507_16165_b200 import render
    rng = np.random.default_rng(500 + seed)
    bg = scenes.gradient_background(int(rng.integers(16, 64)), int(rng.integers(8, 32)))
    size = int(rng.integers(12, 28))
    sb = scenes.small_scene(bg, size, float(rng.choice([0.0, 0.5, 1.0, 2.0])))
    r = rng.uniform(12.0, 40.0)
    sb.set(cam_pos=scenes.inclined_camera(r, rng.uniform(10.0, 170.0), rng.uniform(0.0, 6.28)),
           vertical_fov=math.radians(rng.uniform(20.0, 100.0)), spp=int(rng.choice([1, 2, 3])),
           seed=int(rng.integers(1, 1000)), epsilon=float(rng.choice([0.05, 0.2, 1.0])),
           escape_radius=float(rng.choice([60.0, 150.0])))
    g = render.render_image(sb).reshape(-1).astype(int)
    rc, o, info, _ = orc_render(sb.s)
    assert rc == 0
    d = np.abs(g - o.astype(int))
    assert d.max() <= 1 and (d > 0).mean() <= 0.001
    if have_ref():
        rc, rimg, info = ref_render(sb.s)
        assert rc == 0
        d = np.abs(g - rimg.astype(int))
        assert d.max() <= 1 and (d > 0).mean() <= 0.001


@pytest.mark.parametrize("seed", range(24))
def test_random_table_mode_scene_matches_oracle(seed):
    """Approximate mode (b-table build on the GPU, per-frame bind, lookup)
    on random cameras, disks, table sizes and b ranges: same contract as the
    direct modes against the oracle's table."""
    rng = np.random.default_rng(700 + seed)
    sb = scenes.config(3, int(rng.integers(24, 64)), int(rng.integers(14, 36)))
    sb.set(cam_pos=scenes.inclined_camera(rng.uniform(12.0, 45.0), rng.uniform(20.0, 160.0),
                                          rng.uniform(0.0, 2 * math.pi)),
           vertical_fov=math.radians(rng.uniform(30.0, 90.0)),
           spp=int(rng.choice([1, 2, 4])), seed=int(rng.integers(1, 1 << 30)),
           disk_enabled=int(rng.random() < 0.8), disk_r_in=rng.uniform(3.0, 8.0),
           disk_r_out=rng.uniform(10.0, 35.0), table_entries=int(rng.choice([2000, 5000, 9000])),
           table_b_max=float(rng.choice([30.0, 50.0, 80.0])))
    compare(sb)
