"""trace()'s polyline on the B200 (bhrt_cuda_trace_polylines, SURVEY §8f
row 3): the reference's polyline test cases (proj/tests/test_geodesic.cpp)
restated against the GPU points, the golden traces of the compiled
reference (point counts, last two points), the compiled reference's full
polylines where oracle/_ref exists, and consistency with the outcome-only
batch entry point (escape direction = normalised last chord, deflection
from the points = the kernel's deflection)."""
import math
import os

import numpy as np
import pytest

from golden_cases import impact_ray
from oracle_lib import D, DP, d3, dbuf, have_ref, ref
from paper_2507_16165_b200 import geodesic as G
from paper_2507_16165_b200.abi import BHRT_NUMERICAL, OBJ_HORIZON, OBJ_SKY, OBJ_STALLED

pytestmark = pytest.mark.gpu

KIND = {0: OBJ_HORIZON, 1: OBJ_SKY, 2: OBJ_STALLED}
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


def cfg(eps=0.05, esc=1e4, mw=10, rt=1e-10, at=1e-12):
    return G.TraceConfig(eps, esc, mw, rt, at)


def test_flat_space_points_on_the_straight_line():  # test_geodesic.cpp:220-240
    flat = G.BlackHole(0.0)
    o = np.array([10.0, 0.0, 0.0])
    d = np.array([-1.0, 0.35, 0.0])
    d /= np.linalg.norm(d)
    poly = G.trace(o, d, flat, cfg(0.05, 60.0), polyline=True)
    assert poly.outcome.kind == "escaped"
    b = np.linalg.norm(np.cross(o, d))
    u0 = 1.0 / np.linalg.norm(o)
    w0 = -np.dot(o, d) / (np.linalg.norm(o) * b)
    phi0 = math.atan2(u0 * b, w0 * b)
    e1 = o / np.linalg.norm(o)
    t = d - e1 * np.dot(d, e1)
    e2 = t / np.linalg.norm(t)
    assert len(poly.points) > 10
    for p in poly.points:
        r = np.linalg.norm(p)
        phi = math.atan2(np.dot(p, e2), np.dot(p, e1))
        if phi < -1e-9:
            phi += 2 * math.pi
        assert abs(1.0 / r - math.sin(phi + phi0) / b) <= 1e-9 * u0


def test_radial_polylines():  # test_geodesic.cpp:242-255
    c = cfg(0.05, 100.0)
    inn = G.trace((10, 0, 0), (-1, 0, 0), G.BlackHole(1.0), c, polyline=True)
    assert inn.outcome.kind == "captured"
    assert len(inn.points) == 2
    assert np.linalg.norm(inn.points[1] - np.array([2.0, 0.0, 0.0])) < 1e-12
    out = G.trace((10, 0, 0), (1, 0, 0), G.BlackHole(1.0), c, polyline=True)
    assert out.outcome.kind == "escaped"
    assert len(out.points) == 2
    assert np.array_equal(out.points[1], np.array([110.0, 0.0, 0.0]))


def test_launched_beyond_escape_radius():  # geodesic.cpp:203-209: two-point line
    o, d = (200.0, 5.0, 0.0), (1.0, 0.2, 0.0)
    dn = np.array(d) / np.linalg.norm(d)
    poly = G.trace(o, dn, G.BlackHole(1.0), cfg(0.05, 100.0), polyline=True)
    assert poly.outcome.kind == "escaped"
    assert len(poly.points) == 2
    assert np.array_equal(poly.points[1], np.array(o) + 100.0 * dn)


def test_segment_lengths_track_epsilon():  # test_geodesic.cpp:268-284
    c = cfg(0.05, 100.0)
    for b in (7.0, 0.5, 5.3):
        o, d = impact_ray(b, 50.0)
        poly = G.trace(o, d, G.BlackHole(1.0), c, polyline=True)
        assert len(poly.points) >= 2
        seg = np.linalg.norm(np.diff(poly.points, axis=0), axis=1)
        assert (seg > 0.0).all()
        assert (seg <= 10 * c.epsilon).all()
        assert (seg >= c.epsilon / 4).all() and (seg <= 4 * c.epsilon).all()


def _fidelity(ref_pts, coarse):
    worst = 0.0
    a = coarse[:-1]
    ab = coarse[1:] - a
    L2 = (ab * ab).sum(1)
    for p in ref_pts:
        t = np.clip(((p - a) * ab).sum(1) / L2, 0.0, 1.0)
        worst = max(worst, np.linalg.norm(p - (a + ab * t[:, None]), axis=1).min())
    return worst


def test_halving_epsilon_improves_fidelity():  # test_geodesic.cpp:405-436
    o, d = impact_ray(8.0, 20.0)
    fine = G.trace(o, d, G.BlackHole(1.0), cfg(0.01, 40.0, rt=1e-13, at=1e-15), polyline=True).points
    c04 = G.trace(o, d, G.BlackHole(1.0), cfg(0.4, 40.0), polyline=True).points
    c02 = G.trace(o, d, G.BlackHole(1.0), cfg(0.2, 40.0), polyline=True).points
    assert _fidelity(fine, c04) / _fidelity(fine, c02) >= 1.5


def test_outcome_consistent_with_points_and_batch():
    rng = np.random.default_rng(11)
    o = rng.normal(size=(300, 3))
    o *= (rng.uniform(8.0, 80.0, 300) / np.linalg.norm(o, axis=1))[:, None]
    d = rng.normal(size=(300, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    c = cfg(0.1, 150.0)
    rec, pts = G.trace_polylines(o, d, G.BlackHole(1.0), c)
    rec2, defl = G.trace_batch(o, d, G.BlackHole(1.0), c, deflection=True)
    assert np.array_equal(rec["object"], rec2["object"])
    assert np.array_equal(rec["steps"], rec2["steps"])
    for i in range(len(o)):
        P = pts[i]
        assert np.array_equal(P[0], o[i])
        if rec[i]["object"] == OBJ_SKY and len(P) >= 3:
            chord = P[-1] - P[-2]
            assert np.abs(rec[i]["point"] - chord / np.linalg.norm(chord)).max() <= 1e-12
            # deflection_of_ray from the points (geodesic.cpp:248-260)
            e1 = o[i] / np.linalg.norm(o[i])
            t = d[i] - e1 * np.dot(d[i], e1)
            e2 = t / np.linalg.norm(t)
            seg = np.diff(P, axis=0)
            sx, sy = seg @ e1, seg @ e2
            tot = np.arctan2(sx[:-1] * sy[1:] - sy[:-1] * sx[1:], sx[:-1] * sx[1:] + sy[:-1] * sy[1:]).sum()
            assert abs(abs(tot) - defl[i]) <= 1e-9


def test_counting_pass_and_truncation():
    o, d = impact_ray(7.0, 50.0)
    rec, pts = G.trace_polylines([o], [d], G.BlackHole(1.0), cfg(0.05, 100.0))
    n = len(pts[0])
    assert n > 10
    rec2, pts2 = G.trace_polylines([o], [d], G.BlackHole(1.0), cfg(0.05, 100.0), max_points=n)
    assert np.array_equal(pts[0], pts2[0])
    with pytest.raises(G.InvalidArgument):
        G.trace_polylines([o], [d], G.BlackHole(1.0), cfg(0.05, 100.0), max_points=n - 1)
    with pytest.raises(G.InvalidArgument):  # origin inside the horizon
        G.trace((1.5, 0, 0), (0, 1, 0), G.BlackHole(1.0), cfg(), polyline=True)


def test_golden_traces_point_counts_and_last_points():
    """The 250 golden traces of the compiled reference (tests/golden):
    same outcome and point count (the PI factor's pow may move a window on
    a few rays), and the last two points to 1e-9 relative."""
    z = np.load(GOLD)
    n = len(z["trace_rc"])
    bad_kind = bad_count = checked = 0
    for i in range(n):
        c = cfg(float(z["trace_eps"][i]), float(z["trace_esc"][i]), int(z["trace_mw"][i]),
                float(z["trace_rt"][i]), float(z["trace_at"][i]))
        hole = G.BlackHole(float(z["trace_mass"][i]))
        rc = int(z["trace_rc"][i])
        if rc != 0 and rc != BHRT_NUMERICAL:
            with pytest.raises(G.InvalidArgument):
                G.trace_polylines([z["trace_origin"][i]], [z["trace_dir"][i]], hole, c)
            continue
        rec, pts = G.trace_polylines([z["trace_origin"][i]], [z["trace_dir"][i]], hole, c)
        if rc == BHRT_NUMERICAL:
            assert rec[0]["object"] == -BHRT_NUMERICAL
            continue
        if rec[0]["object"] != KIND[int(z["trace_kind"][i])]:
            bad_kind += 1
            continue
        if len(pts[0]) != int(z["trace_npoints"][i]):
            bad_count += 1
            continue
        last2 = z["trace_last2"][i].reshape(2, 3)
        got = pts[0][-2:] if len(pts[0]) >= 2 else np.stack([pts[0][0], pts[0][0]])
        scale = max(1.0, float(np.abs(last2).max()))
        assert np.abs(got - last2).max() <= 1e-9 * scale
        checked += 1
    assert bad_kind <= 2 and bad_count <= 0.02 * n
    assert checked > 150


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_full_polylines_match_compiled_reference():
    L = ref()
    rng = np.random.default_rng(29)
    o = rng.normal(size=(120, 3))
    o *= (rng.uniform(8.0, 60.0, 120) / np.linalg.norm(o, axis=1))[:, None]
    d = rng.normal(size=(120, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    c = cfg(0.2, 120.0)
    rec, pts = G.trace_polylines(o, d, G.BlackHole(1.0), c)
    same = 0
    for i in range(len(o)):
        cap = 200000
        buf = dbuf(3 * cap)
        k = L.ref_trace_points(d3(o[i]), d3(d[i]), 1.0, d3((0, 0, 0)), 0.2, 120.0, 10, 1e-10, 1e-12, buf, cap)
        assert k > 0
        R = np.frombuffer(buf, dtype=np.float64, count=3 * min(k, cap)).reshape(-1, 3)
        if len(pts[i]) != k:
            continue
        scale = np.maximum(1.0, np.abs(R))
        assert (np.abs(pts[i] - R) <= 1e-9 * scale).all()
        same += 1
    assert same >= 0.98 * len(o)
