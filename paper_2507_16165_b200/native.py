"""ctypes binding of the C ABI (libbhrt_b200.so).

There is no fallback: if the CUDA library is missing the import of
`lib()` raises, and every render goes through the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

from .abi import RayRecord, Scene, Sphere, StatusInfo

_PKG = os.path.dirname(os.path.abspath(__file__))
# BHRT_B200_LIB: developer override to time alternative builds of the same sources
LIB_PATH = os.environ.get("BHRT_B200_LIB") or os.path.join(_PKG, "libbhrt_b200.so")

_lib = None

P = C.POINTER


class BhrtError(RuntimeError):
    """Raised for a non-zero bhrt_status; carries code/px/py like the
    reference's exception taxonomy (errors.hpp, render.hpp:39-47)."""

    def __init__(self, code: int, px: int, py: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code, self.px, self.py, self.message = code, px, py, message


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.bhrt_cuda_abi_version.restype = C.c_int32
        L.bhrt_scene_defaults.argtypes = [P(Scene)]
        L.bhrt_validate_scene.argtypes = [P(Scene), P(StatusInfo)]
        L.bhrt_make_spheres.argtypes = [C.c_uint64, C.c_int32, P(C.c_double), C.c_double,
                                        C.c_double, C.c_double, C.c_double, P(Sphere)]
        L.bhrt_make_bands.argtypes = [C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32),
                                      C.c_int32, P(C.c_int32)]
        L.bhrt_cuda_render_rows.argtypes = [P(Scene), C.c_int32, C.c_int32, P(C.c_int32),
                                            C.c_int32, P(C.c_uint8), C.c_size_t, P(RayRecord),
                                            P(StatusInfo)]
        L.bhrt_cuda_trace_rays.argtypes = [P(Scene), P(C.c_double), C.c_int64, C.c_int32,
                                           P(RayRecord), P(C.c_double), P(StatusInfo)]
        L.bhrt_cuda_trace_polylines.argtypes = [P(Scene), P(C.c_double), C.c_int64, C.c_int32,
                                                C.c_int32, P(C.c_double), P(C.c_int32),
                                                P(RayRecord), P(StatusInfo)]
        L.bhrt_scene_parse_text.argtypes = [C.c_char_p, P(Scene), P(Sphere), C.c_int32,
                                            P(C.c_int32), P(StatusInfo)]
        L.bhrt_scene_format_text.argtypes = [P(Scene), C.c_char_p, C.c_size_t, P(C.c_size_t)]
        L.bhrt_ctx_set_output_layout.argtypes = [C.c_void_p, C.c_int32]
        L.bhrt_device_alloc.argtypes = [C.c_int32, C.c_size_t, P(C.c_void_p), P(StatusInfo)]
        L.bhrt_device_free.argtypes = [C.c_int32, C.c_void_p]
        L.bhrt_ipc_export.argtypes = [C.c_int32, C.c_void_p, P(C.c_uint8), P(StatusInfo)]
        L.bhrt_ipc_open.argtypes = [C.c_int32, P(C.c_uint8), P(C.c_void_p), P(StatusInfo)]
        L.bhrt_ipc_close.argtypes = [C.c_int32, C.c_void_p]
        L.bhrt_ctx_create.argtypes = [C.c_int32, P(C.c_void_p), P(StatusInfo)]
        L.bhrt_ctx_destroy.argtypes = [C.c_void_p]
        L.bhrt_ctx_destroy.restype = None
        L.bhrt_ctx_set_scene.argtypes = [C.c_void_p, P(Scene), P(StatusInfo)]
        L.bhrt_ctx_render_async.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                            C.c_void_p, P(StatusInfo)]
        L.bhrt_ctx_finish.argtypes = [C.c_void_p, P(StatusInfo)]
        L.bhrt_ctx_frame_begin.argtypes = [C.c_void_p, C.c_void_p, P(StatusInfo)]
        L.bhrt_ctx_stats.argtypes = [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64),
                                     P(C.c_int32)]
        L.bhrt_ctx_counters.argtypes = [C.c_void_p, P(C.c_uint64)]
        L.bhrt_ctx_upload_bytes.argtypes = [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]
        L.bhrt_ctx_set_timing.argtypes = [C.c_void_p, C.c_int32]
        L.bhrt_ctx_kernel_ms.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float)]
        L.bhrt_tile_row_count.argtypes = [C.c_int32] * 5
        L.bhrt_tile_row_count.restype = C.c_int32
        L.bhrt_b200_fp64_peak_tflops.argtypes = [C.c_int, C.c_int, P(C.c_double)]
        L.bhrt_b200_fp64_peak_tflops.restype = C.c_double
        L.bhrt_flops_per_step.argtypes = [C.c_int32]
        L.bhrt_flops_per_step.restype = C.c_double
        _lib = L
    return _lib


# Symbols include/bhrt_cuda.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "bhrt_scene_defaults", "bhrt_validate_scene", "bhrt_make_spheres", "bhrt_make_bands",
    "bhrt_cuda_render_rows", "bhrt_cuda_trace_rays", "bhrt_cuda_trace_polylines", "bhrt_scene_parse_text",
    "bhrt_scene_format_text", "bhrt_ctx_set_output_layout", "bhrt_device_alloc",
    "bhrt_device_free", "bhrt_ipc_export", "bhrt_ipc_open", "bhrt_ipc_close", "bhrt_ctx_create", "bhrt_ctx_destroy", "bhrt_ctx_set_scene",
    "bhrt_ctx_render_async", "bhrt_ctx_frame_begin", "bhrt_ctx_finish", "bhrt_ctx_stats", "bhrt_ctx_set_timing",
    "bhrt_ctx_kernel_ms", "bhrt_ctx_counters", "bhrt_ctx_upload_bytes", "bhrt_tile_row_count",
    "bhrt_b200_fp64_peak_tflops", "bhrt_cuda_abi_version", "bhrt_flops_per_step",
]


def check(rc: int, info: StatusInfo):
    if rc != 0:
        raise BhrtError(rc, info.px, info.py, info.message.decode(errors="replace"))
