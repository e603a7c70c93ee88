"""ctypes mirror of include/bhrt_cuda.h (the C ABI of the hot path).

The structs here are byte-for-byte the C structs; tests/test_abi.py checks
sizes and offsets against the C compiler's view (offsetof probe).
"""
from __future__ import annotations

import ctypes as C

BHRT_OK = 0
BHRT_USAGE = 1
BHRT_IO = 2
BHRT_NUMERICAL = 3
BHRT_PROTOCOL = 4
BHRT_DEVICE = 5
BHRT_INVALID_ARGUMENT = 6

INTEGRATOR_REFERENCE = 0
INTEGRATOR_RK4 = 1
INTEGRATOR_RKF45 = 2
INTEGRATOR_TABLE = 3

SKY_IMAGE = 0
SKY_CHECKER = 1

OBJ_NONE = 0
OBJ_HORIZON = 1
OBJ_SKY = 2
OBJ_STALLED = 3
OBJ_DISK = 4
OBJ_SPHERE = 5

D3 = C.c_double * 3


class Sphere(C.Structure):
    _fields_ = [("center", D3), ("radius", C.c_double), ("albedo", D3)]


class Scene(C.Structure):
    _fields_ = [
        ("mass", C.c_double),
        ("center", D3),
        ("cam_pos", D3),
        ("cam_look_at", D3),
        ("vertical_fov", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("spp", C.c_int32),
        ("max_windings", C.c_int32),
        ("seed", C.c_uint64),
        ("epsilon", C.c_double),
        ("escape_radius", C.c_double),
        ("rel_tol", C.c_double),
        ("abs_tol", C.c_double),
        ("sky_rgb", C.POINTER(C.c_uint8)),
        ("sky_width", C.c_int32),
        ("sky_height", C.c_int32),
        ("integrator", C.c_int32),
        ("sky_kind", C.c_int32),
        ("step", C.c_double),
        ("max_step", C.c_double),
        ("chord_dphi", C.c_double),
        ("checker_nu", C.c_int32),
        ("checker_nv", C.c_int32),
        ("checker_color_a", D3),
        ("checker_color_b", D3),
        ("disk_enabled", C.c_int32),
        ("n_spheres", C.c_int32),
        ("disk_r_in", C.c_double),
        ("disk_r_out", C.c_double),
        ("disk_color_in", D3),
        ("disk_color_out", D3),
        ("spheres", C.POINTER(Sphere)),
        ("light_dir", D3),
        ("ambient", C.c_double),
        ("table_entries", C.c_int32),
        ("table_samples", C.c_int32),
        ("table_b_max", C.c_double),
        ("table_dpsi", C.c_double),
    ]


class StatusInfo(C.Structure):
    _fields_ = [("code", C.c_int32), ("px", C.c_int32), ("py", C.c_int32),
                ("message", C.c_char * 256)]


class RayRecord(C.Structure):
    _fields_ = [("object", C.c_int32), ("sphere", C.c_int32), ("steps", C.c_int32),
                ("rejected", C.c_int32), ("point", D3), ("phi", C.c_double)]


# numpy dtype with the same layout as RayRecord (for bulk record arrays)
def record_dtype():
    import numpy as np
    return np.dtype([("object", "<i4"), ("sphere", "<i4"), ("steps", "<i4"),
                     ("rejected", "<i4"), ("point", "<f8", (3,)), ("phi", "<f8")])
