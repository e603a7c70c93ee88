"""The reference's per-ray geodesic tests (proj/tests/test_geodesic.cpp,
acceptance.cpp criteria 2-4) run against the B200 kernel through the batch
ABI entry point bhrt_cuda_trace_rays (paper_2507_16165_b200.geodesic), plus
bit-level agreement with the CPU oracle and, where oracle/_ref exists, the
compiled reference's own trace(). Each test cites the case it restates."""
import math

import numpy as np
import pytest

from golden_cases import impact_ray
from oracle_lib import d3, have_ref, oracle, orc_trace_reference, ref_trace
from paper_2507_16165_b200 import geodesic as G
from paper_2507_16165_b200.abi import BHRT_NUMERICAL, OBJ_HORIZON, OBJ_SKY, OBJ_STALLED

pytestmark = pytest.mark.gpu

PI = math.pi
KIND = {0: OBJ_HORIZON, 1: OBJ_SKY, 2: OBJ_STALLED}


def cfg(eps=0.05, esc=1e4, mw=10, rt=1e-10, at=1e-12):
    return G.TraceConfig(eps, esc, mw, rt, at)


def random_rays(n, seed, rmin=8.0, rmax=200.0):
    rng = np.random.default_rng(seed)
    o = rng.normal(size=(n, 3))
    o *= (rng.uniform(rmin, rmax, n) / np.linalg.norm(o, axis=1))[:, None]
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    return o, d


def test_batch_matches_oracle():
    """Mode R parity: window arithmetic is bit-identical, but the PI
    controller's pow() (libdevice vs glibc, 1 ulp) may move a step hint, so
    step counts agree on almost every ray and escape directions to the
    north-star 1e-9."""
    o, d = random_rays(3000, 5)
    c = cfg(eps=0.1, esc=500.0)
    rec, _ = G.trace_batch(o, d, G.BlackHole(1.0), c)
    kind_mismatch = steps_mismatch = 0
    for i in range(len(o)):
        rc, kind, edir, _, _, ns, nr = orc_trace_reference(o[i], d[i], 1.0, (0, 0, 0), 0.1, 500.0, 10)
        assert rc == 0
        if rec[i]["object"] != KIND[kind]:
            kind_mismatch += 1
            continue
        steps_mismatch += int(rec[i]["steps"] != ns or rec[i]["rejected"] != nr)
        if kind == 1:
            assert np.abs(rec[i]["point"] - np.array(edir)).max() <= 1e-9
    assert kind_mismatch <= 3
    assert steps_mismatch <= 0.01 * len(o)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_batch_matches_compiled_reference_trace():
    o, d = random_rays(1500, 9)
    rec, _ = G.trace_batch(o, d, G.BlackHole(1.0), cfg(eps=0.1, esc=500.0))
    mismatch = 0
    for i in range(len(o)):
        rc, kind, edir, _, _ = ref_trace(o[i], d[i], 1.0, (0, 0, 0), 0.1, 500.0, 10)
        assert rc == 0
        if rec[i]["object"] != KIND[kind]:
            mismatch += 1
        elif kind == 1:
            assert np.abs(rec[i]["point"] - np.array(edir)).max() <= 1e-9
    assert mismatch <= 2


def test_capture_vs_escape_across_critical_b():  # test_geodesic.cpp:185-201
    for b, kind in ((5.0, "captured"), (5.4, "escaped")):
        o, d = impact_ray(b, 1000.0)
        assert G.trace(o, d, G.BlackHole(1.0), cfg()).kind == kind


def test_flat_space_escape_direction():  # test_geodesic.cpp:203-218
    rng = np.random.default_rng(23)
    os_, ds = [], []
    while len(os_) < 200:
        d = rng.uniform(-1, 1, 3)
        if np.linalg.norm(d) < 1e-2:
            continue
        d /= np.linalg.norm(d)
        o = np.array([12.0, 3 * rng.uniform(-1, 1), 3 * rng.uniform(-1, 1)])
        e1 = o / np.linalg.norm(o)
        if np.linalg.norm(d - e1 * (d @ e1)) < 1e-6:
            continue
        os_.append(o)
        ds.append(d)
    rec, _ = G.trace_batch(os_, ds, G.BlackHole(0.0), cfg(esc=50.0))
    assert (rec["object"] == OBJ_SKY).all()
    assert np.abs(rec["point"] - np.array(ds)).max() <= 1e-9


def test_radial_rays_analytic():  # test_geodesic.cpp:242-254
    inward = G.trace((10, 0, 0), (-1, 0, 0), G.BlackHole(1.0), cfg(esc=100.0))
    assert inward.kind == "captured" and inward.steps == 0
    outward = G.trace((10, 0, 0), (1, 0, 0), G.BlackHole(1.0), cfg(esc=100.0))
    assert outward.kind == "escaped" and outward.escape_direction == (1.0, 0.0, 0.0)


def test_origin_inside_horizon_rejected():  # test_geodesic.cpp:256-259
    with pytest.raises(G.InvalidArgument) as e:
        G.trace_batch([(50, 0, 0), (1.5, 0, 0)], [(0, 1, 0), (0, 1, 0)], G.BlackHole(1.0), cfg())
    assert e.value.px == 1  # lowest offending ray


def test_invalid_trace_config_rejected():  # geodesic.cpp:19-27
    for bad in (dict(eps=0.0), dict(esc=-1.0), dict(mw=0), dict(rt=0.0), dict(at=-1.0)):
        with pytest.raises(G.InvalidArgument):
            G.trace((20, 0, 0), (0, 1, 0), G.BlackHole(1.0), cfg(**bad))
    with pytest.raises(G.InvalidArgument):
        G.trace((20, 0, 0), (0, 1, 0), G.BlackHole(-1.0), cfg())


def test_near_critical_stalls():  # test_geodesic.cpp:261-268
    o, d = impact_ray(5.1961524227, 100.0)
    assert G.trace(o, d, G.BlackHole(1.0), cfg(mw=2)).kind == "stalled"


def test_numerical_failure_reported_like_the_reference():  # geodesic.cpp:233-234
    """A wide window carries a near-radial outgoing ray past u = 0 (SURVEY
    §8a row 10: triggered by large epsilon)."""
    o, d = (10.0, 0.0, 0.0), (math.cos(0.01), math.sin(0.01), 0.0)
    rc = orc_trace_reference(o, d, 1e-3, (0, 0, 0), 100.0, 1e4, 10)[0]
    assert rc == BHRT_NUMERICAL
    rec, _ = G.trace_batch([(40.0, 0.0, 0.0), o], [(0.0, 1.0, 0.0), d], G.BlackHole(1e-3), cfg(eps=100.0))
    assert rec[0]["object"] == OBJ_SKY and rec[1]["object"] == -BHRT_NUMERICAL
    with pytest.raises(G.NumericalError):
        G.trace(o, d, G.BlackHole(1e-3), cfg(eps=100.0))


def test_deflection_weak_flat_strong():  # test_geodesic.cpp:321-342, acceptance.cpp:113-121
    a = G.deflection_angle(1000.0, G.BlackHole(1.0), cfg(esc=1e6))
    assert abs(a - 0.004) <= 0.005 * 0.004
    assert G.deflection_angle(5.0, G.BlackHole(0.0), cfg(esc=100.0)) <= 1e-9
    a = G.deflection_angle(5.4, G.BlackHole(1.0), cfg(esc=1e3))
    assert 4.0 / 5.4 < a < 2 * PI
    with pytest.raises(G.NumericalError):
        G.deflection_angle(4.0, G.BlackHole(1.0), cfg(esc=1e3))


def test_deflection_matches_oracle():
    import ctypes as C
    L = oracle()
    bs = np.linspace(5.3, 60.0, 40)
    esc = 300.0
    o = [(math.sqrt(esc * esc - b * b), b, 0.0) for b in bs]
    d = [(-1.0, 0.0, 0.0)] * len(bs)
    rec, defl = G.trace_batch(o, d, G.BlackHole(1.0), cfg(eps=0.05, esc=esc), deflection=True)
    for i in range(len(bs)):
        ang = C.c_double()
        assert L.orc_deflection_of_ray(d3(o[i]), d3(d[i]), 1.0, d3((0, 0, 0)), 0.05, esc, 10, 1e-10,
                                       1e-12, C.byref(ang)) == 0
        assert abs(defl[i] - ang.value) <= 1e-11 * max(1.0, ang.value)


def rotate(v, axis, ang):
    k = np.asarray(axis, float) / np.linalg.norm(axis)
    v = np.asarray(v, float)
    return v * math.cos(ang) + np.cross(k, v) * math.sin(ang) + k * (k @ v) * (1 - math.cos(ang))


def test_deflection_isotropic():  # test_geodesic.cpp:344-361
    o, d = impact_ray(8.0, 100.0)
    axes = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, -1), (2, -1, 3), (-1, 4, 1)]
    os_ = [o] + [rotate(o, ax, 0.3 + 0.4 * i) for i, ax in enumerate(axes)]
    ds = [d] + [rotate(d, ax, 0.3 + 0.4 * i) for i, ax in enumerate(axes)]
    rec, defl = G.trace_batch(os_, ds, G.BlackHole(1.0), cfg(eps=0.1, esc=150.0), deflection=True)
    assert defl[0] > 0.3
    assert np.abs(defl[1:] - defl[0]).max() <= 1e-9


def test_capture_monotone_in_b():  # test_geodesic.cpp:363-380
    bc = 3.0 * math.sqrt(3.0)
    rays = [impact_ray(bc - 0.5 + i / 49.0, 100.0) for i in range(50)]
    rec, _ = G.trace_batch([r[0] for r in rays], [r[1] for r in rays], G.BlackHole(1.0),
                           cfg(eps=0.1, esc=300.0))
    kinds = rec["object"]
    assert not (kinds == OBJ_STALLED).any()
    first_escape = int(np.argmax(kinds == OBJ_SKY))
    assert kinds[first_escape] == OBJ_SKY
    assert (kinds[:first_escape] == OBJ_HORIZON).all() and (kinds[first_escape:] == OBJ_SKY).all()


def test_critical_b_bisection_batched():  # acceptance.cpp:97-121
    """The reference bisects b_c to 1e-3; one batch of 4001 impact parameters
    over [5.0, 5.4] locates the capture/escape edge to 1e-4."""
    bs = np.linspace(5.0, 5.4, 4001)
    rays = [impact_ray(b, 1000.0) for b in bs]
    rec, _ = G.trace_batch([r[0] for r in rays], [r[1] for r in rays], G.BlackHole(1.0), cfg())
    k = rec["object"]
    assert not (k == OBJ_STALLED).any()
    edge = int(np.argmax(k == OBJ_SKY))
    assert (k[:edge] == OBJ_HORIZON).all() and (k[edge:] == OBJ_SKY).all()
    assert abs(0.5 * (bs[edge - 1] + bs[edge]) - 3 * math.sqrt(3)) <= 1e-3


def test_empty_batch():
    rec, defl = G.trace_batch(np.zeros((0, 3)), np.zeros((0, 3)), G.BlackHole(1.0), cfg(),
                              deflection=True)
    assert len(rec) == 0 and len(defl) == 0


@pytest.mark.parametrize("eps,rt,at", [(1.0, 1e-10, 1e-12), (5.0, 1e-13, 1e-15), (0.02, 1e-8, 1e-10)])
def test_step_hint_regimes_match_oracle(eps, rt, at):
    """Wide windows / tight tolerances make the carried step hint binding
    (several DOPRI5 steps per window; the kernel forms the hint lazily,
    trace_reference.cu window_h0): outcomes and escape directions still
    match the oracle to the north-star 1e-9. Step counts are compared only
    where the hint rarely binds: where it does, the PI factor's pow()
    (libdevice vs glibc, <= 1 ulp) moves step boundaries (measured: 122/600
    and 539/600 rays in the first two regimes, identical before and after
    the lazy-hint change)."""
    o, d = random_rays(600, 21, 10.0, 80.0)
    rec, _ = G.trace_batch(o, d, G.BlackHole(1.0), cfg(eps=eps, esc=300.0, rt=rt, at=at))
    mism = steps = 0
    for i in range(len(o)):
        rc, kind, edir, _, _, ns, nr = orc_trace_reference(o[i], d[i], 1.0, (0, 0, 0), eps, 300.0, 10,
                                                           rt, at)
        if rc != 0 or rec[i]["object"] != KIND[kind]:
            mism += 1
            continue
        steps += int(rec[i]["steps"] != ns)
        if kind == 1:
            assert np.abs(rec[i]["point"] - np.array(edir)).max() <= 1e-9
    assert mism <= 2
    if eps < 0.1:
        assert steps <= 0.02 * len(o)
