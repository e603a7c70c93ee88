"""Python mirror of the reference's per-ray geodesic API
(proj/include/bhrt/geodesic.hpp) on the B200 kernels, through the C ABI's
batch entry point `bhrt_cuda_trace_rays`:

    BlackHole, TraceConfig                     geodesic.hpp:14-45
    TraceOutcome                               geodesic.hpp:51-60
    RayPolyline                                geodesic.hpp:62-65
    trace(origin, dir, hole, cfg)              geodesic.hpp:107-108  (outcome; polyline=True: RayPolyline)
    deflection_of_ray(origin, dir, hole, cfg)  geodesic.hpp:110-113
    deflection_angle(b, hole, cfg)             geodesic.hpp:115-118
    trace_batch(origins, dirs, hole, cfg, deflection=False)   many rays, one launch
    trace_polylines(origins, dirs, hole, cfg)  many rays with their polylines

Errors follow the reference: invalid configuration or an origin inside the
horizon -> InvalidArgument (std::invalid_argument), numerical failure or a
deflection of a non-escaping ray -> NumericalError. Outcomes carry the
escape direction (the normalised last chord, geodesic.cpp:211-212), step
counts and the final phi; the polyline is written only when asked for
(bhrt_cuda_trace_polylines: a counting pass, then the points).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import native
from .abi import (BHRT_INVALID_ARGUMENT, BHRT_NUMERICAL, INTEGRATOR_REFERENCE, OBJ_HORIZON, OBJ_SKY,
                  OBJ_STALLED, RayRecord, StatusInfo, record_dtype)
from .scenes import SceneBuf


class InvalidArgument(native.BhrtError, ValueError):
    """std::invalid_argument from trace()/validate() (geodesic.cpp:19-27,166-172)."""


class NumericalError(native.BhrtError, ArithmeticError):
    """bhrt::NumericalError (errors.hpp)."""


@dataclass
class BlackHole:  # geodesic.hpp:14-20
    mass: float = 1.0
    center: tuple = (0.0, 0.0, 0.0)


@dataclass
class TraceConfig:  # geodesic.hpp:39-45 (reference defaults)
    epsilon: float = 0.05
    escape_radius: float = 1e4
    max_windings: int = 10
    rel_tol: float = 1e-10
    abs_tol: float = 1e-12


@dataclass
class TraceOutcome:  # geodesic.hpp:51-60
    kind: str  # "captured" | "escaped" | "stalled"
    escape_direction: tuple = field(default=(0.0, 0.0, 0.0))
    steps: int = 0
    rejected: int = 0
    phi: float = 0.0


_KIND = {OBJ_HORIZON: "captured", OBJ_SKY: "escaped", OBJ_STALLED: "stalled"}


def _scene(hole: BlackHole, cfg: TraceConfig) -> SceneBuf:
    sb = SceneBuf()
    sb.set(mass=hole.mass, center=tuple(hole.center), epsilon=cfg.epsilon,
           escape_radius=cfg.escape_radius, max_windings=cfg.max_windings, rel_tol=cfg.rel_tol,
           abs_tol=cfg.abs_tol, integrator=INTEGRATOR_REFERENCE)
    return sb


def trace_batch(origins, dirs, hole: BlackHole = BlackHole(), cfg: TraceConfig = TraceConfig(),
                deflection: bool = False, device: int = -1):
    """Traces n rays in one launch. Returns (records, deflections or None):
    records is a structured array of bhrt_ray_record (object = OBJ_HORIZON /
    OBJ_SKY / OBJ_STALLED, or -BHRT_NUMERICAL for a ray whose integration
    failed); deflections[i] is NaN unless ray i escaped. Raises
    InvalidArgument like the reference's trace(); numerical failures of
    individual rays are reported in the records, not raised."""
    o = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(dirs, np.float64).reshape(-1, 3))
    if o.shape != d.shape:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1, "trace_batch: origins/dirs shape mismatch")
    n = o.shape[0]
    rays = np.ascontiguousarray(np.concatenate([o, d], axis=1))
    rec = np.zeros(n, record_dtype())
    defl = np.full(n, np.nan) if deflection else None
    info = StatusInfo()
    sb = _scene(hole, cfg)
    rc = native.lib().bhrt_cuda_trace_rays(
        sb.ptr(), rays.ctypes.data_as(C.POINTER(C.c_double)), n, device,
        rec.ctypes.data_as(C.POINTER(RayRecord)),
        defl.ctypes.data_as(C.POINTER(C.c_double)) if deflection else None, C.byref(info))
    if rc == BHRT_INVALID_ARGUMENT:
        raise InvalidArgument(rc, info.px, info.py, info.message.decode(errors="replace"))
    if rc not in (0, BHRT_NUMERICAL):
        raise native.BhrtError(rc, info.px, info.py, info.message.decode(errors="replace"))
    return rec, defl


@dataclass
class RayPolyline:  # geodesic.hpp:62-65
    points: np.ndarray  # (k, 3) world points: the origin, then every window end
    outcome: TraceOutcome


def _outcome(r) -> TraceOutcome:
    kind = _KIND[int(r["object"])]
    edir = tuple(float(x) for x in r["point"]) if kind == "escaped" else (0.0, 0.0, 0.0)
    return TraceOutcome(kind, edir, int(r["steps"]), int(r["rejected"]), float(r["phi"]))


def trace_polylines(origins, dirs, hole: BlackHole = BlackHole(), cfg: TraceConfig = TraceConfig(),
                    device: int = -1, max_points: int | None = None):
    """Traces n rays and returns (records, [points (k_i, 3) arrays]). With
    max_points=None a counting pass sizes the buffer first; otherwise longer
    polylines raise InvalidArgument (truncated). Errors as trace_batch."""
    o = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(dirs, np.float64).reshape(-1, 3))
    if o.shape != d.shape:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1, "trace_polylines: origins/dirs shape mismatch")
    n = o.shape[0]
    rays = np.ascontiguousarray(np.concatenate([o, d], axis=1))
    sb = _scene(hole, cfg)
    L = native.lib()

    def run(cap):
        rec = np.zeros(n, record_dtype())
        cnt = np.zeros(n, np.int32)
        pts = np.zeros((n, max(cap, 0), 3))
        info = StatusInfo()
        rc = L.bhrt_cuda_trace_polylines(
            sb.ptr(), rays.ctypes.data_as(C.POINTER(C.c_double)), n, device, cap,
            pts.ctypes.data_as(C.POINTER(C.c_double)) if cap > 0 else None,
            cnt.ctypes.data_as(C.POINTER(C.c_int32)), rec.ctypes.data_as(C.POINTER(RayRecord)),
            C.byref(info))
        if rc == BHRT_INVALID_ARGUMENT:
            raise InvalidArgument(rc, info.px, info.py, info.message.decode(errors="replace"))
        if rc not in (0, BHRT_NUMERICAL):
            raise native.BhrtError(rc, info.px, info.py, info.message.decode(errors="replace"))
        return rec, cnt, pts

    cap = max_points
    if cap is None:
        _, cnt, _ = run(0)
        cap = int(cnt.max()) if n else 0
    rec, cnt, pts = run(cap)
    if n and int(cnt.max()) > cap:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, int(np.argmax(cnt)), -1,
                              "trace_polylines: polyline longer than max_points")
    return rec, [pts[i, :cnt[i]].copy() for i in range(n)]


def trace(ray_origin, ray_dir, hole: BlackHole = BlackHole(),
          cfg: TraceConfig = TraceConfig(), polyline: bool = False):
    """geodesic.hpp:107-108 for one ray: the TraceOutcome, or with
    polyline=True the reference's RayPolyline (points + outcome)."""
    if polyline:
        rec, pts = trace_polylines([ray_origin], [ray_dir], hole, cfg)
    else:
        rec, _ = trace_batch([ray_origin], [ray_dir], hole, cfg)
    r = rec[0]
    if r["object"] < 0:
        raise NumericalError(BHRT_NUMERICAL, 0, -1, "trace: numerical failure")
    out = _outcome(r)
    return RayPolyline(pts[0], out) if polyline else out


def deflection_of_ray(ray_origin, ray_dir, hole: BlackHole = BlackHole(),
                      cfg: TraceConfig = TraceConfig()) -> float:
    """geodesic.hpp:110-113: winding-aware total turning of an escaping ray."""
    rec, defl = trace_batch([ray_origin], [ray_dir], hole, cfg, deflection=True)
    if rec[0]["object"] != OBJ_SKY:
        raise NumericalError(BHRT_NUMERICAL, 0, -1, "deflection_angle: ray did not escape")
    return float(defl[0])


def deflection_angle(b: float, hole: BlackHole = BlackHole(),
                     cfg: TraceConfig = TraceConfig()) -> float:
    """geodesic.cpp:264-270: canonical launch at r0 = escape_radius, offset b."""
    if not (b > 0.0) or b >= cfg.escape_radius:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1,
                              "deflection_angle: need 0 < b < escape_radius")
    r0 = cfg.escape_radius
    c = hole.center
    origin = (c[0] + math.sqrt(r0 * r0 - b * b), c[1] + b, c[2])
    return deflection_of_ray(origin, (-1.0, 0.0, 0.0), hole, cfg)
