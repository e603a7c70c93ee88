"""The reference's geodesic known-answer tests (proj/tests/test_geodesic.cpp,
acceptance.cpp criteria 2-4), restated against the CPU oracle. Each test
cites the case it restates."""
import ctypes as C
import math

import numpy as np
import pytest

from golden_cases import impact_ray
from oracle_lib import d3, dbuf, oracle, orc_trace_reference

PI = math.pi


def iw(state, dphi, mass, rt=1e-10, at=1e-12, hint=None):
    L = oracle()
    out = dbuf(3)
    h = C.c_double(hint) if hint is not None else None
    rc = L.orc_integrate_window(d3(state), dphi, mass, rt, at, C.byref(h) if h is not None else None,
                                out, None, None)
    return rc, list(out), (h.value if h is not None else None)


def ics(o, d, mass=1.0):
    st = dbuf(3)
    rc = oracle().orc_initial_conditions(d3(o), d3(d), d3((0, 0, 0)), st)
    return rc, list(st)


def trace(o, d, mass=1.0, eps=0.05, esc=1e4, mw=10):
    return orc_trace_reference(o, d, mass, (0, 0, 0), eps, esc, mw)


def test_ode_rhs_exact():  # test_geodesic.cpp:52-65
    out = dbuf(2)
    oracle().orc_ode_rhs(0.0, 0.1, 0.3, 0.0, out)
    assert list(out) == [0.3, -0.1]
    oracle().orc_ode_rhs(0.0, 0.5, 0.0, 1.0, out)
    assert list(out) == [0.0, 3.0 * 0.25 - 0.5]
    oracle().orc_ode_rhs(0.0, 1.0 / 3.0, 0.0, 1.0, out)
    assert abs(out[1]) < 1e-16


def basis(o, d):
    e1, e2 = dbuf(3), dbuf(3)
    ok = oracle().orc_plane_basis(d3(o), d3(d), d3((0, 0, 0)), e1, e2)
    return ok, np.array(list(e1)), np.array(list(e2))


def test_plane_basis_examples():  # test_geodesic.cpp:67-85
    ok, e1, e2 = basis((10, 0, 0), (0, 1, 0))
    assert ok and np.linalg.norm(e1 - [1, 0, 0]) < 1e-15 and np.linalg.norm(e2 - [0, 1, 0]) < 1e-15
    assert not basis((10, 0, 0), (-1, 0, 0))[0]
    assert not basis((10, 0, 0), (1, 0, 0))[0]
    s = math.sqrt(2.0) / 2.0
    ok, e1, e2 = basis((0, 5, 0), (0, -s, s))
    assert ok and np.linalg.norm(e1 - [0, 1, 0]) < 1e-12 and np.linalg.norm(e2 - [0, 0, 1]) < 1e-12


def test_plane_basis_invariants():  # test_geodesic.cpp:87-106
    rng = np.random.default_rng(11)
    for _ in range(200):
        o = 10.0 * rng.uniform(-1, 1, 3)
        d = rng.uniform(-1, 1, 3)
        if np.linalg.norm(o) < 1.0 or np.linalg.norm(d) < 1e-2:
            continue
        d /= np.linalg.norm(d)
        ok, e1, e2 = basis(o, d)
        if not ok:
            continue
        assert abs(np.linalg.norm(e1) - 1) < 1e-12 and abs(np.linalg.norm(e2) - 1) < 1e-12
        assert abs(e1 @ e2) < 1e-12 and d @ e2 > 0
        r0 = np.linalg.norm(o)
        assert np.linalg.norm(r0 * e1 - o) < 1e-9 * r0


def test_initial_conditions():  # test_geodesic.cpp:108-125
    rc, s = ics((10, 0, 0), (0, 1, 0))
    assert rc == 0 and s[0] == 0.0 and s[1] == pytest.approx(0.1, rel=1e-15) and abs(s[2]) < 1e-15
    s2 = math.sqrt(2.0) / 2.0
    rc, s = ics((10, 0, 0), (-s2, s2, 0))
    assert s[2] == pytest.approx(0.1, rel=1e-12)
    assert ics((10, 0, 0), (-1, 0, 0))[0] == 6  # radial -> std::invalid_argument


def test_step_dphi_clamp():  # test_geodesic.cpp:127-132
    L = oracle()
    assert L.orc_step_dphi(0.1, 0.1) == pytest.approx(0.01, rel=1e-15)
    assert L.orc_step_dphi(1e-9, 0.1) == 1e-6
    assert L.orc_step_dphi(10.0, 0.1) == 0.1


def test_hypot_restatement_matches_glibc():
    # the reference calls glibc hypot (geodesic.cpp:78); CPython's math.hypot
    # is a different algorithm, so compare against libm directly.
    libm = C.CDLL("libm.so.6")
    libm.hypot.restype = C.c_double
    libm.hypot.argtypes = [C.c_double, C.c_double]
    L = oracle()
    rng = np.random.default_rng(5)
    for _ in range(20000):
        x = float(rng.uniform(0, 1) * 10.0 ** rng.integers(-6, 3))
        y = float(rng.uniform(-1, 1) * 10.0 ** rng.integers(-6, 3))
        assert L.orc_hypot(x, y) == libm.hypot(x, y)


def test_flat_space_cosine():  # test_geodesic.cpp:134-141
    rc, out, _ = iw((0.0, 0.1, 0.0), PI / 2, 0.0)
    assert rc == 0 and abs(out[1]) <= 1e-10 and out[2] == pytest.approx(-0.1, rel=1e-9)


def test_photon_sphere_fixed_point():  # test_geodesic.cpp:143-150
    for dphi in (0.3, 2.0, 7.0):
        rc, out, _ = iw((0.0, 1.0 / 3.0, 0.0), dphi, 1.0)
        assert abs(out[1] - 1.0 / 3.0) < 1e-14 and abs(out[2]) < 1e-14


def test_integrate_window_vs_fine_rk4():  # test_geodesic.cpp:152-165
    o, d = impact_ray(10.0, 1000.0)
    _, s0 = ics(o, d)
    L = oracle()
    u, w = s0[1], s0[2]
    h = 3.0 / 300000
    out = dbuf(2)
    for _ in range(300000):
        L.orc_rk4_step(u, w, h, 1.0, out)
        u, w = out[0], out[1]
    rc, got, _ = iw(s0, 3.0, 1.0)
    assert abs(got[1] - u) <= 1e-11 and abs(got[2] - w) <= 1e-11


def test_underflow_near_singularity():  # test_geodesic.cpp:167-178
    rc, out, _ = iw((0.0, 0.6, 2.0), 2.5, 1.0)
    assert rc == 1 and out[1] > 1.0 and 0.0 < out[0] < 2.5


def test_rejects_nonpositive_window():  # test_geodesic.cpp:180-183
    assert iw((0.0, 0.1, 0.0), 0.0, 1.0)[0] == 6


def test_capture_vs_escape_across_critical_b():  # test_geodesic.cpp:185-201
    L = oracle()
    for b, fate, kind in ((5.0, 0, 0), (5.4, 1, 1)):
        o, d = impact_ray(b, 1000.0)
        _, s = ics(o, d)
        assert L.orc_classify(s[1], s[2], 1.0, 1e4, 20.0 * PI, 1e-3) == fate
        assert trace(o, d, eps=0.05, esc=1e4)[1] == kind


def test_flat_space_escape_direction():  # test_geodesic.cpp:203-218
    rng = np.random.default_rng(23)
    for _ in range(20):
        d = rng.uniform(-1, 1, 3)
        if np.linalg.norm(d) < 1e-2:
            continue
        d /= np.linalg.norm(d)
        o = np.array([12.0, 3 * rng.uniform(-1, 1), 3 * rng.uniform(-1, 1)])
        if not basis(o, d)[0]:
            continue
        rc, kind, edir, *_ = trace(o, d, mass=0.0, eps=0.05, esc=50.0)
        assert kind == 1 and np.linalg.norm(np.array(edir) - d) <= 1e-9


def test_radial_rays_analytic():  # test_geodesic.cpp:242-254
    rc, kind, edir, npts, l2, *_ = trace((10, 0, 0), (-1, 0, 0), esc=100.0)
    assert kind == 0 and npts == 2 and np.linalg.norm(np.array(l2[3:]) - [2, 0, 0]) < 1e-12
    rc, kind, edir, npts, l2, *_ = trace((10, 0, 0), (1, 0, 0), esc=100.0)
    assert kind == 1 and edir == [1.0, 0.0, 0.0] and npts == 2


def test_origin_inside_horizon_rejected():  # test_geodesic.cpp:256-259
    assert trace((1.5, 0, 0), (0, 1, 0))[0] == 6


def test_near_critical_stalls():  # test_geodesic.cpp:261-268
    o, d = impact_ray(5.1961524227, 100.0)
    assert trace(o, d, eps=0.05, esc=1e4, mw=2)[1] == 2


def run_to_escape(o, d, eps, esc, mass=1.0):
    L = oracle()
    _, s = ics(o, d)
    hint = C.c_double(0.0)
    states = [s]
    while not (states[-1][1] <= 1.0 / esc and states[-1][2] < 0.0):
        out = dbuf(3)
        L.orc_integrate_window(d3(states[-1]), L.orc_step_dphi(states[-1][1], eps), mass, 1e-10,
                               1e-12, C.byref(hint), out, None, None)
        states.append(list(out))
        assert out[0] < 2 * PI * 10
    return states


def test_first_integral_conserved():  # test_geodesic.cpp:308-319, acceptance.cpp:126-150
    L = oracle()
    rng = np.random.default_rng(97)
    for _ in range(25):
        o, d = impact_ray(rng.uniform(6.0, 100.0), 200.0)
        st = run_to_escape(o, d, 0.1, 200.0)
        e0 = L.orc_conserved_energy(st[0][1], st[0][2], 1.0)
        for s in st:
            assert abs(L.orc_conserved_energy(s[1], s[2], 1.0) - e0) <= 1e-8 * abs(e0)


def test_phi_monotone():  # test_geodesic.cpp:289-306
    o, d = impact_ray(8.0, 200.0)
    st = run_to_escape(o, d, 0.1, 200.0)
    assert all(b[0] > a[0] and b[1] > 0 for a, b in zip(st, st[1:]))


def deflection(b, mass, eps, esc):
    L = oracle()
    ang = C.c_double()
    a = math.sqrt(esc * esc - b * b)
    rc = L.orc_deflection_of_ray(d3((a, b, 0.0)), d3((-1.0, 0.0, 0.0)), mass, d3((0, 0, 0)), eps,
                                 esc, 10, 1e-10, 1e-12, C.byref(ang))
    return rc, ang.value


def test_deflection_weak_flat_strong():  # test_geodesic.cpp:321-342, acceptance.cpp:113-121
    rc, a = deflection(1000.0, 1.0, 0.05, 1e6)
    assert rc == 0 and abs(a - 0.004) <= 0.005 * 0.004
    assert deflection(5.0, 0.0, 0.05, 100.0)[1] <= 1e-9
    rc, a = deflection(5.4, 1.0, 0.05, 1e3)
    assert 4.0 / 5.4 < a < 2 * PI
    assert deflection(4.0, 1.0, 0.05, 1e3)[0] == 3  # captured -> NumericalError


def rotate(v, axis, ang):
    k = np.asarray(axis, float) / np.linalg.norm(axis)
    v = np.asarray(v, float)
    return v * math.cos(ang) + np.cross(k, v) * math.sin(ang) + k * (k @ v) * (1 - math.cos(ang))


def test_deflection_isotropic():  # test_geodesic.cpp:344-361
    L = oracle()
    o, d = impact_ray(8.0, 100.0)

    def defl(o, d):
        ang = C.c_double()
        assert L.orc_deflection_of_ray(d3(o), d3(d), 1.0, d3((0, 0, 0)), 0.1, 150.0, 10, 1e-10,
                                       1e-12, C.byref(ang)) == 0
        return ang.value

    ref = defl(o, d)
    assert ref > 0.3
    axes = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, -1), (2, -1, 3), (-1, 4, 1)]
    for i, ax in enumerate(axes):
        ang = 0.3 + 0.4 * i
        assert abs(defl(rotate(o, ax, ang), rotate(d, ax, ang)) - ref) <= 1e-9


def test_capture_monotone_in_b():  # test_geodesic.cpp:363-380
    bc = 3.0 * math.sqrt(3.0)
    seen = False
    for i in range(50):
        o, d = impact_ray(bc - 0.5 + i / 49.0, 100.0)
        kind = trace(o, d, eps=0.1, esc=300.0)[1]
        assert kind != 2
        if kind == 1:
            seen = True
        else:
            assert not seen
    assert seen


def test_critical_b_bisection():  # acceptance.cpp:97-121
    def captured(b):
        o, d = impact_ray(b, 1000.0)
        k = trace(o, d, eps=0.05, esc=1e4)[1]
        assert k != 2
        return k == 0

    lo, hi = 5.0, 5.4
    assert captured(lo) and not captured(hi)
    while hi - lo > 2e-4:
        mid = 0.5 * (lo + hi)
        if captured(mid):
            lo = mid
        else:
            hi = mid
    assert abs(0.5 * (lo + hi) - 3 * math.sqrt(3)) <= 1e-3


def test_tolerance_halving_monotone():  # test_geodesic.cpp:382-404
    for b in (6.0, 8.0, 12.0, 20.0, 40.0):
        o, d = impact_ray(b, 50.0)
        _, s0 = ics(o, d)
        ref = iw(s0, 2.5, 1.0, 1e-13, 1e-15)[1]
        prev = 1e300
        for k in range(6):
            got = iw(s0, 2.5, 1.0, 1e-6 / (1 << k), 1e-8 / (1 << k))[1]
            err = abs(got[1] - ref[1])
            assert err <= prev
            prev = err
