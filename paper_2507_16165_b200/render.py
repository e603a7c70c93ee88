"""Python mirror of the reference's render API (proj/include/bhrt/render.hpp)
over the C ABI. Same names, argument meaning and error behaviour:

    validate_scene(scene)                      render.hpp:26   (UsageError)
    make_bands(height, workers)                render.hpp:55
    render_rows(scene, row_start, row_end, threads)   render.hpp:60-61
    render_band(scene, band)                   render.hpp:63
    render_image(scene, threads)               render.hpp:66
    shade_pixel(scene, px, py)                 render.hpp:52

`threads` keeps its reference meaning only as a validity check (>= 1); the
work runs on the GPU(s) in `devices`. Output bytes are identical for every
`threads` and every device split, like the reference's contract
(render.hpp:58-59,65).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native
from .abi import (BHRT_INVALID_ARGUMENT, BHRT_NUMERICAL, BHRT_USAGE, RayRecord, StatusInfo,
                  record_dtype)
from .scenes import SceneBuf


class UsageError(native.BhrtError):
    pass


class RenderError(native.BhrtError):
    """render.hpp:39-47: numerical failure at pixel (px, py)."""


class InvalidArgument(native.BhrtError, ValueError):
    pass


_EXC = {BHRT_USAGE: UsageError, BHRT_NUMERICAL: RenderError, BHRT_INVALID_ARGUMENT: InvalidArgument}


def _raise(rc: int, info: StatusInfo):
    if rc:
        cls = _EXC.get(rc, native.BhrtError)
        raise cls(rc, info.px, info.py, info.message.decode(errors="replace"))


@dataclass(frozen=True)
class BandAssignment:
    worker_id: int
    row_start: int
    row_end: int

    def rows(self) -> int:
        return self.row_end - self.row_start


def validate_scene(scene: SceneBuf) -> None:
    info = StatusInfo()
    _raise(native.lib().bhrt_validate_scene(scene.ptr(), C.byref(info)), info)


def make_bands(height: int, workers: int) -> list[BandAssignment]:
    if height < 1 or workers < 1:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1,
                              "make_bands: height and workers must be >= 1")
    n = min(height, workers)
    rs = (C.c_int32 * n)()
    re = (C.c_int32 * n)()
    cnt = C.c_int32()
    rc = native.lib().bhrt_make_bands(height, workers, rs, re, n, C.byref(cnt))
    if rc:
        raise InvalidArgument(rc, -1, -1, "make_bands failed")
    return [BandAssignment(i, rs[i], re[i]) for i in range(cnt.value)]


def render_rows(scene: SceneBuf, row_start: int, row_end: int, threads: int = 1,
                devices: list[int] | None = None, records: bool = False):
    """Pixel bytes (flat uint8, row-major RGB8) for rows [row_start, row_end).
    With records=True also returns the per-sample bhrt_ray_record array."""
    validate_scene(scene)
    if threads < 1:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1, "render: threads must be >= 1")
    if row_start < 0 or row_end > scene.s.height or row_start > row_end:
        raise InvalidArgument(BHRT_INVALID_ARGUMENT, -1, -1, "render: row range out of bounds")
    rows = row_end - row_start
    out = np.zeros(rows * scene.s.width * 3, np.uint8)
    rec = None
    rec_ptr = None
    if records:
        rec = np.zeros(rows * scene.s.width * scene.s.spp, record_dtype())
        rec_ptr = rec.ctypes.data_as(C.POINTER(RayRecord))
    devs = None
    nd = 0
    if devices:
        devs = (C.c_int32 * len(devices))(*devices)
        nd = len(devices)
    info = StatusInfo()
    rc = native.lib().bhrt_cuda_render_rows(scene.ptr(), row_start, row_end, devs, nd,
                                            out.ctypes.data_as(C.POINTER(C.c_uint8)), out.nbytes,
                                            rec_ptr, C.byref(info))
    _raise(rc, info)
    return (out, rec) if records else out


def render_band(scene: SceneBuf, band: BandAssignment, **kw):
    return render_rows(scene, band.row_start, band.row_end, 1, **kw)


def render_image(scene: SceneBuf, threads: int = 1, **kw) -> np.ndarray:
    px = render_rows(scene, 0, scene.s.height, threads, **kw)
    return px.reshape(scene.s.height, scene.s.width, 3)


def shade_pixel(scene: SceneBuf, px: int, py: int) -> tuple[int, int, int]:
    """One pixel (a one-row render; kept for API parity with render.hpp:52)."""
    row = render_rows(scene, py, py + 1, 1)
    return tuple(int(v) for v in row[3 * px:3 * px + 3])


class Context:
    """Persistent device context: scene resident in HBM, async renders into
    caller-owned device buffers on a caller stream (bhrt_ctx_* in the ABI)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        info = StatusInfo()
        _raise(native.lib().bhrt_ctx_create(device, C.byref(self._h), C.byref(info)), info)
        self.device = device
        self.scene = None

    def close(self):
        if self._h:
            native.lib().bhrt_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_scene(self, scene: SceneBuf):
        info = StatusInfo()
        _raise(native.lib().bhrt_ctx_set_scene(self._h, scene.ptr(), C.byref(info)), info)
        self.scene = scene

    def render_async(self, d_out: int, row_start: int = 0, row_end: int | None = None,
                     tile_rows: int = 1, tile_stride: int = 1, tile_offset: int = 0,
                     d_records: int | None = None, stream: int | None = None):
        if row_end is None:
            row_end = self.scene.s.height
        info = StatusInfo()
        rc = native.lib().bhrt_ctx_render_async(self._h, row_start, row_end, tile_rows,
                                                tile_stride, tile_offset, C.c_void_p(d_out),
                                                C.c_void_p(d_records or 0),
                                                C.c_void_p(stream or 0), C.byref(info))
        _raise(rc, info)

    def set_output_layout(self, image: int):
        """0: rows packed in order of y (default); 1: d_out is the whole image
        (bhrt_ctx_set_output_layout)."""
        rc = native.lib().bhrt_ctx_set_output_layout(self._h, image)
        if rc:
            raise native.BhrtError(rc, -1, -1, "bad output layout")

    def frame_begin(self, stream: int | None = None):
        """Counters/failures accumulate over the following render_async calls
        (same stream) until finish() (bhrt_ctx_frame_begin)."""
        info = StatusInfo()
        _raise(native.lib().bhrt_ctx_frame_begin(self._h, C.c_void_p(stream or 0), C.byref(info)), info)

    def finish(self):
        info = StatusInfo()
        _raise(native.lib().bhrt_ctx_finish(self._h, C.byref(info)), info)

    def set_timing(self, enable: bool = True):
        native.lib().bhrt_ctx_set_timing(self._h, 1 if enable else 0)

    def kernel_ms(self) -> tuple[float, float]:
        """(trace_ms, shade_ms) of the last finished render (set_timing first)."""
        a, b = C.c_float(), C.c_float()
        rc = native.lib().bhrt_ctx_kernel_ms(self._h, C.byref(a), C.byref(b))
        if rc:
            raise native.BhrtError(rc, -1, -1, "kernel timing unavailable")
        return a.value, b.value

    def upload_bytes(self) -> tuple[int, int, int]:
        """(bytes staged host->device by the last set_scene, kernel parameter
        bytes per launch, render counter block bytes) — bhrt_ctx_upload_bytes."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        native.lib().bhrt_ctx_upload_bytes(self._h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def counters(self) -> list[int]:
        out = (C.c_uint64 * 8)()
        native.lib().bhrt_ctx_counters(self._h, out)
        return list(out)

    def stats(self) -> dict:
        st, rj, rays = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ln = C.c_int32()
        native.lib().bhrt_ctx_stats(self._h, C.byref(st), C.byref(rj), C.byref(rays), C.byref(ln))
        return {"steps": st.value, "rejected": rj.value, "rays": rays.value,
                "launches": ln.value}


def tile_row_count(row_start, row_end, tile_rows, tile_stride, tile_offset) -> int:
    return native.lib().bhrt_tile_row_count(row_start, row_end, tile_rows, tile_stride,
                                            tile_offset)
