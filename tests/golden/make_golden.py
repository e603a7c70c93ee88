"""Generate the committed golden fixtures from the COMPILED REFERENCE.

    make -C oracle && python tests/golden/make_golden.py

Needs oracle/_ref/libbhrt_ref.so (built from /root/reference/proj by
oracle/Makefile). Every value below is produced by the reference's own code
(trace, integrate_window, hash_counter, generate_ray, sample_direction,
render_rows, deflection_angle); tests/test_oracle_golden.py checks the CPU
oracle against them, so the oracle stays pinned even where the reference
cannot be built.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_lib import d3, dbuf, ref, ref_trace  # noqa: E402
from paper_2507_16165_b200 import scenes  # noqa: E402
from paper_2507_16165_b200.abi import StatusInfo  # noqa: E402


from golden_cases import impact_ray  # noqa: E402


def traces(rng):
    rows = []
    # random rays around the hole (mass 1 and flat space)
    for i in range(240):
        o = rng.uniform(-30, 30, 3)
        if np.linalg.norm(o) < 4:
            continue
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        mass = 0.0 if i % 5 == 0 else 1.0
        eps = [0.05, 0.1, 0.5][i % 3]
        rows.append((o, d, mass, eps, 60.0, 10, 1e-10, 1e-12))
    # the reference's KAT geometries (test_geodesic.cpp, acceptance.cpp)
    for b in (5.0, 5.4, 5.1961524227, 7.0, 0.5, 5.3, 8.0, 12.0):
        o, d = impact_ray(b, 100.0)
        rows.append((np.array(o), np.array(d), 1.0, 0.05, 1e4 if b in (5.0, 5.4) else 100.0,
                     2 if b == 5.1961524227 else 10, 1e-10, 1e-12))
    rows.append((np.array([10.0, 0, 0]), np.array([-1.0, 0, 0]), 1.0, 0.05, 100.0, 10, 1e-10, 1e-12))
    rows.append((np.array([10.0, 0, 0]), np.array([1.0, 0, 0]), 1.0, 0.05, 100.0, 10, 1e-10, 1e-12))
    out = {k: [] for k in ("origin", "dir", "mass", "eps", "esc", "mw", "rt", "at", "rc", "kind",
                           "edir", "npoints", "last2")}
    for o, d, mass, eps, esc, mw, rt, at in rows:
        rc, kind, edir, npts, l2 = ref_trace(o, d, mass, (0, 0, 0), eps, esc, mw, rt, at)
        for k, v in zip(("origin", "dir", "mass", "eps", "esc", "mw", "rt", "at", "rc", "kind",
                         "edir", "npoints", "last2"),
                        (o, d, mass, eps, esc, mw, rt, at, rc, kind, edir, npts, l2)):
            out[k].append(v)
    return {f"trace_{k}": np.array(v) for k, v in out.items()}


def windows(rng):
    L = ref()
    st, dph, mass, rt, at, hint_in, outs, hints, rcs = [], [], [], [], [], [], [], [], []
    cases = [((0.0, 0.1, 0.0), math.pi / 2, 0.0, 1e-10, 1e-12, 0.0),
             ((0.0, 1 / 3, 0.0), 7.0, 1.0, 1e-10, 1e-12, 0.0),
             ((0.0, 0.6, 2.0), 2.5, 1.0, 1e-10, 1e-12, 0.0)]
    for _ in range(60):
        u = rng.uniform(0.01, 0.3)
        w = rng.uniform(-0.3, 0.3)
        cases.append(((0.0, u, w), rng.uniform(1e-3, 0.5), 1.0, 10 ** rng.uniform(-12, -6),
                      10 ** rng.uniform(-14, -8), rng.choice([0.0, 1e-3, 0.05])))
    for s, dphi, m, r, a, h in cases:
        hb = C.c_double(h)
        o = dbuf(3)
        rc = L.ref_integrate_window(d3(s), dphi, m, r, a, C.byref(hb), o)
        st.append(s); dph.append(dphi); mass.append(m); rt.append(r); at.append(a)
        hint_in.append(h); outs.append(list(o)); hints.append(hb.value); rcs.append(rc)
    return {"win_state": np.array(st), "win_dphi": np.array(dph), "win_mass": np.array(mass),
            "win_rt": np.array(rt), "win_at": np.array(at), "win_hint_in": np.array(hint_in),
            "win_out": np.array(outs), "win_hint_out": np.array(hints), "win_rc": np.array(rcs)}


def misc(rng):
    L = ref()
    seeds = rng.integers(0, 2**63, 50, dtype=np.uint64)
    hs = [L.ref_hash_counter(int(s), int(i), int(2 * i + 1), int(i % 7)) for i, s in enumerate(seeds)]
    bg = scenes.gradient_background(32, 16)
    dirs = rng.normal(size=(200, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    cols = []
    for d in dirs:
        o = dbuf(3)
        L.ref_sample_direction(bg.ctypes.data_as(C.POINTER(C.c_uint8)), 32, 16, d3(d), o)
        cols.append(list(o))
    sb = scenes.small_scene(bg, 13)
    sb.s.spp = 4
    sb.s.seed = 12345
    rays = []
    for px, py, s in [(0, 0, 0), (6, 6, 0), (12, 12, 3), (3, 9, 2), (7, 1, 1)]:
        o, d = dbuf(3), dbuf(3)
        L.ref_generate_ray(sb.ptr(), px, py, s, o, d)
        rays.append([px, py, s] + list(d))
    defl = []
    for b, mass, eps, esc in [(1000.0, 1.0, 0.05, 1e6), (5.0, 0.0, 0.05, 100.0), (5.4, 1.0, 0.05, 1e3)]:
        v = C.c_double()
        rc = L.ref_deflection_angle(b, mass, eps, esc, C.byref(v))
        defl.append([b, mass, eps, esc, rc, v.value])
    return {"hash_seed": seeds, "hash_out": np.array(hs, dtype=np.uint64),
            "sd_dirs": dirs, "sd_cols": np.array(cols), "ray_rows": np.array(rays),
            "defl": np.array(defl)}


def images():
    from golden_cases import image_cases
    out = {}
    L = ref()
    for name, sb in image_cases().items():
        px = np.zeros(sb.s.width * sb.s.height * 3, np.uint8)
        info = StatusInfo()
        rc = L.ref_render_rows(sb.ptr(), 0, sb.s.height, 4, px.ctypes.data_as(C.POINTER(C.c_uint8)),
                               C.byref(info))
        assert rc == 0, (name, info.message)
        out[f"img_{name}"] = px
    return out


def main():
    rng = np.random.default_rng(20261019)
    data = {}
    data.update(traces(rng))
    data.update(windows(rng))
    data.update(misc(rng))
    data.update(images())
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **data)
    print(path, os.path.getsize(path), "bytes,", len(data), "arrays")


if __name__ == "__main__":
    main()
