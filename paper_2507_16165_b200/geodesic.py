"""Python mirror of the reference's per-ray geodesic API
(proj/include/bhrt/geodesic.hpp) on the B200 kernels, through the C ABI's
batch entry point `bhrt_cuda_trace_rays`:

    BlackHole, TraceConfig                     geodesic.hpp:14-45
    TraceOutcome                               geodesic.hpp:51-60
    trace(origin, dir, hole, cfg)              geodesic.hpp:107-108  (outcome, no polyline)
    deflection_of_ray(origin, dir, hole, cfg)  geodesic.hpp:110-113
    deflection_angle(b, hole, cfg)             geodesic.hpp:115-118
    trace_batch(origins, dirs, hole, cfg, deflection=False)   many rays, one launch

Errors follow the reference: invalid configuration or an origin inside the
horizon -> InvalidArgument (std::invalid_argument), numerical failure or a
deflection of a non-escaping ray -> NumericalError. The polyline itself is
never materialised on the GPU; outcomes carry the escape direction (the
normalised last chord, geodesic.cpp:211-212), step counts and the final phi.
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


def trace(ray_origin, ray_dir, hole: BlackHole = BlackHole(),
          cfg: TraceConfig = TraceConfig()) -> TraceOutcome:
    """geodesic.hpp:107-108 for one ray (outcome only)."""
    rec, _ = trace_batch([ray_origin], [ray_dir], hole, cfg)
    r = rec[0]
    if r["object"] < 0:
        raise NumericalError(BHRT_NUMERICAL, 0, -1, "trace: numerical failure")
    kind = _KIND[int(r["object"])]
    edir = tuple(float(x) for x in r["point"]) if kind == "escaped" else (0.0, 0.0, 0.0)
    return TraceOutcome(kind, edir, int(r["steps"]), int(r["rejected"]), float(r["phi"]))


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
