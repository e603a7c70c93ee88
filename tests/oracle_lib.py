"""Loaders for the CPU oracle (oracle/liboracle.so) and the compiled reference
(oracle/_ref/libbhrt_ref.so). TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2507_16165_b200.abi import RayRecord, Scene, Sphere, StatusInfo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libbhrt_ref.so")

P = C.POINTER
D = C.c_double
DP = P(C.c_double)
IP = P(C.c_int)

_oracle = None
_ref = None


def _ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def oracle():
    global _oracle
    if _oracle is None:
        _ensure_built()
        L = C.CDLL(ORACLE_SO)
        L.orc_hash_counter.restype = C.c_uint64
        L.orc_hash_counter.argtypes = [C.c_uint64] * 4
        L.orc_hypot.restype = D
        L.orc_hypot.argtypes = [D, D]
        L.orc_step_dphi.restype = D
        L.orc_step_dphi.argtypes = [D, D]
        L.orc_segment_dphi.restype = D
        L.orc_segment_dphi.argtypes = [D, D, D]
        L.orc_conserved_energy.restype = D
        L.orc_conserved_energy.argtypes = [D, D, D]
        L.orc_ode_rhs.argtypes = [D, D, D, D, DP]
        L.orc_camera_basis.argtypes = [P(Scene), DP, DP, DP]
        L.orc_generate_ray.argtypes = [P(Scene), C.c_int, C.c_int, C.c_int, DP, DP]
        L.orc_sample_direction.argtypes = [P(C.c_uint8), C.c_int, C.c_int, DP, DP]
        L.orc_plane_basis.argtypes = [DP, DP, DP, DP, DP]
        L.orc_initial_conditions.argtypes = [DP, DP, DP, DP]
        L.orc_integrate_window.argtypes = [DP, D, D, D, D, DP, DP, IP, IP]
        L.orc_trace_reference.argtypes = [DP, DP, D, DP, D, D, C.c_int, D, D, IP, DP, IP, DP, IP, IP]
        L.orc_deflection_of_ray.argtypes = [DP, DP, D, DP, D, D, C.c_int, D, D, DP]
        L.orc_rk4_step.argtypes = [D, D, D, D, DP]
        L.orc_classify.argtypes = [D, D, D, D, D, D]
        L.orc_rkf45_step.argtypes = [D, D, D, D, D, D, D, DP, DP]
        L.orc_rkf45_factor_tables.argtypes = [DP, DP, IP, IP]
        L.orc_trace_sample.argtypes = [P(Scene), C.c_int, C.c_int, C.c_int, P(RayRecord), DP]
        L.orc_shade_pixel.argtypes = [P(Scene), C.c_int, C.c_int, P(C.c_uint8), P(RayRecord)]
        L.orc_render_rows.argtypes = [P(Scene), C.c_int, C.c_int, C.c_int, P(C.c_uint8),
                                      P(RayRecord), P(StatusInfo)]
        L.orc_validate_scene.argtypes = [P(Scene), P(StatusInfo)]
        L.orc_make_bands.argtypes = [C.c_int, C.c_int, IP, IP, C.c_int, IP]
        L.orc_make_spheres.argtypes = [C.c_uint64, C.c_int, DP, D, D, D, D, P(Sphere)]
        L.orc_scene_defaults.argtypes = [P(Scene)]
        _oracle = L
    return _oracle


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_trace.argtypes = [DP, DP, D, DP, D, D, C.c_int, D, D, IP, DP, IP, DP]
        L.ref_trace_points.argtypes = [DP, DP, D, DP, D, D, C.c_int, D, D, DP, C.c_int]
        L.ref_integrate_window.argtypes = [DP, D, D, D, D, DP, DP]
        L.ref_plane_basis.argtypes = [DP, DP, DP, DP, DP]
        L.ref_initial_conditions.argtypes = [DP, DP, DP, DP]
        L.ref_step_dphi.restype = D
        L.ref_step_dphi.argtypes = [D, D]
        L.ref_deflection_angle.argtypes = [D, D, D, D, DP]
        L.ref_deflection_of_ray.argtypes = [DP, DP, D, D, D, DP]
        L.ref_hash_counter.restype = C.c_uint64
        L.ref_hash_counter.argtypes = [C.c_uint64] * 4
        L.ref_generate_ray.argtypes = [P(Scene), C.c_int, C.c_int, C.c_int, DP, DP]
        L.ref_sample_direction.argtypes = [P(C.c_uint8), C.c_int, C.c_int, DP, DP]
        L.ref_render_rows.argtypes = [P(Scene), C.c_int, C.c_int, C.c_int, P(C.c_uint8),
                                      P(StatusInfo)]
        L.ref_make_bands.argtypes = [C.c_int, C.c_int, IP, IP, C.c_int, IP]
        L.ref_strong_scaling_mean.restype = D
        L.ref_strong_scaling_mean.argtypes = [P(Scene), C.c_int, C.c_int]
        L.ref_strong_scaling_pixels_mean.restype = D
        L.ref_strong_scaling_pixels_mean.argtypes = [P(Scene), C.c_int, C.c_int, IP, IP, C.c_int]
        L.ref_serialize_scene.restype = C.c_size_t
        L.ref_serialize_scene.argtypes = [P(Scene), C.c_char_p, C.c_size_t]
        L.ref_parse_scene.argtypes = [C.c_char_p, P(Scene), P(StatusInfo)]
        L.ref_save_ppm.restype = C.c_size_t
        L.ref_save_ppm.argtypes = [C.c_int, C.c_int, P(C.c_uint8), P(C.c_uint8), C.c_size_t]
        _ref = L
    return _ref


def d3(x):
    return (C.c_double * 3)(*[float(v) for v in x])


def dbuf(n):
    return (C.c_double * n)()


def u8p(arr: np.ndarray):
    return arr.ctypes.data_as(P(C.c_uint8))


# ---------------------------------------------------------------- wrappers
def orc_trace_reference(o, d, mass=1.0, center=(0, 0, 0), eps=0.05, esc=1e4, mw=10,
                        rt=1e-10, at=1e-12):
    L = oracle()
    kind, npts, ns, nr = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    dr, l2 = dbuf(3), dbuf(6)
    rc = L.orc_trace_reference(d3(o), d3(d), mass, d3(center), eps, esc, mw, rt, at,
                               C.byref(kind), dr, C.byref(npts), l2, C.byref(ns), C.byref(nr))
    return rc, kind.value, list(dr), npts.value, list(l2), ns.value, nr.value


def ref_trace(o, d, mass=1.0, center=(0, 0, 0), eps=0.05, esc=1e4, mw=10, rt=1e-10, at=1e-12):
    L = ref()
    kind, npts = C.c_int(), C.c_int()
    dr, l2 = dbuf(3), dbuf(6)
    rc = L.ref_trace(d3(o), d3(d), mass, d3(center), eps, esc, mw, rt, at, C.byref(kind), dr,
                     C.byref(npts), l2)
    return rc, kind.value, list(dr), npts.value, list(l2)


def orc_render(scene, rows=None, threads=8, records=False):
    L = oracle()
    r0, r1 = rows if rows else (0, scene.height)
    out = np.zeros(((r1 - r0) * scene.width * 3,), np.uint8)
    info = StatusInfo()
    recs = None
    if records:
        recs = (RayRecord * ((r1 - r0) * scene.width * scene.spp))()
    rc = L.orc_render_rows(C.byref(scene), r0, r1, threads, u8p(out), recs, C.byref(info))
    return rc, out, info, recs


def orc_render_np(scene, rows=None, threads=None):
    """orc_render with the records as a numpy structured array (abi.record_dtype)."""
    from paper_2507_16165_b200.abi import record_dtype
    L = oracle()
    r0, r1 = rows if rows else (0, scene.height)
    out = np.zeros(((r1 - r0) * scene.width * 3,), np.uint8)
    rec = np.zeros((r1 - r0) * scene.width * scene.spp, record_dtype())
    info = StatusInfo()
    rc = L.orc_render_rows(C.byref(scene), r0, r1, threads or os.cpu_count() or 1, u8p(out),
                           rec.ctypes.data_as(C.POINTER(RayRecord)), C.byref(info))
    return rc, out, info, rec


def ref_render(scene, rows=None, threads=8):
    L = ref()
    r0, r1 = rows if rows else (0, scene.height)
    out = np.zeros(((r1 - r0) * scene.width * 3,), np.uint8)
    info = StatusInfo()
    rc = L.ref_render_rows(C.byref(scene), r0, r1, threads, u8p(out), C.byref(info))
    return rc, out, info


def table_entry(t, e, cap=4096):
    L = oracle()
    kind, n = C.c_int(), C.c_int()
    ends = dbuf(4)
    smp = dbuf(2 * cap)
    rc = L.orc_table_entry(t, e, C.byref(kind), C.byref(n), ends, smp, cap)
    assert rc == 0
    return kind.value, n.value, list(ends), np.array(list(smp)[:2 * n.value]).reshape(-1, 2)
