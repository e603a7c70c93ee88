"""Scene construction: the reference's scene fields plus the BASELINE.json
configs 0-4, and the background fixtures the reference tests use.

Backgrounds restate the formulas of the reference fixtures
(proj/tests/test_util.hpp:18-55, acceptance.cpp:40-49,288-300); the
configs follow BASELINE.json `configs` with the conventions frozen in
DESIGN.md §Scene (disk plane, inclination, colours, light, sphere RNG).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from .abi import (INTEGRATOR_REFERENCE, INTEGRATOR_RK4, INTEGRATOR_RKF45, INTEGRATOR_TABLE,
                  SKY_CHECKER, SKY_IMAGE, Scene, Sphere)

PI = math.pi


# ------------------------------------------------------------ backgrounds
def gradient_background(w: int = 64, h: int = 32) -> np.ndarray:
    """test_util.hpp:18-26: smooth gradient with no pure-black texel."""
    x = np.arange(w)[None, :]
    y = np.arange(h)[:, None]
    img = np.zeros((h, w, 3), np.uint8)
    img[..., 0] = (30 + (x * 200) // w).astype(np.uint8)
    img[..., 1] = (30 + (y * 200) // h).astype(np.uint8)
    img[..., 2] = (40 + ((x + y) * 150) // (w + h)).astype(np.uint8)
    return img


def uniform_background(r: int, g: int, b: int, w: int = 16, h: int = 8) -> np.ndarray:
    """test_util.hpp:28-34."""
    img = np.zeros((h, w, 3), np.uint8)
    img[...] = (r, g, b)
    return img


def ring_background(w: int = 256, h: int = 128) -> np.ndarray:
    """test_util.hpp:38-55 / acceptance.cpp:288-300: colour depends only on the
    angle from +z (scalar libm math so every texel matches the reference)."""
    img = np.zeros((h, w, 3), np.uint8)
    for yy in range(h):
        for xx in range(w):
            u = (xx + 0.5) / w
            v = (yy + 0.5) / h
            lon = 2.0 * PI * u - PI
            lat_cos = math.sin(v * PI)
            dir_z = lat_cos * math.sin(lon)
            angle = math.acos(min(max(dir_z, -1.0), 1.0))
            img[yy, xx, 0] = int(40 + 215 * math.exp(-angle * angle / 0.02))
            img[yy, xx, 1] = int(30 + angle / PI * 120)
            img[yy, xx, 2] = 90
    return img


def checker_image(w: int, h: int, nu: int = 16, nv: int = 8,
                  a=(0.9, 0.9, 0.9), b=(0.1, 0.1, 0.15)) -> np.ndarray:
    """The procedural checker baked into an equirect RGB8 image, so the
    reference (which only knows PPM skies, image.cpp:131-169) can render the
    sky-only projection of the configs."""
    x = (np.arange(w) + 0.5) / w
    y = (np.arange(h) + 0.5) / h
    cu = np.floor(x * nu).astype(int)[None, :]
    cv = np.floor(y * nv).astype(int)[:, None]
    par = (cu + cv) & 1
    img = np.zeros((h, w, 3), np.uint8)
    for c in range(3):
        img[..., c] = np.where(par == 1, round(b[c] * 255), round(a[c] * 255))
    return img


# ------------------------------------------------------------ scene buffer
class SceneBuf:
    """A bhrt_scene plus the host arrays its pointers borrow (kept alive)."""

    def __init__(self):
        self.s = Scene()
        scene_defaults(self.s)
        self._sky = None
        self._spheres = None

    # convenience attribute access to the underlying struct
    def __getattr__(self, k):
        return getattr(self.s, k)

    def set(self, **kw):
        for k, v in kw.items():
            f = getattr(self.s, k)
            if isinstance(f, C.Array):
                for i, x in enumerate(v):
                    f[i] = x
            else:
                setattr(self.s, k, v)
        return self

    def set_sky(self, img: np.ndarray | None):
        if img is None:
            self._sky = None
            self.s.sky_rgb = C.POINTER(C.c_uint8)()
            self.s.sky_width = 0
            self.s.sky_height = 0
            return self
        img = np.ascontiguousarray(img, dtype=np.uint8)
        assert img.ndim == 3 and img.shape[2] == 3
        self._sky = img
        self.s.sky_rgb = img.ctypes.data_as(C.POINTER(C.c_uint8))
        self.s.sky_height, self.s.sky_width = int(img.shape[0]), int(img.shape[1])
        self.s.sky_kind = SKY_IMAGE
        return self

    def set_spheres(self, spheres):
        n = len(spheres)
        arr = (Sphere * max(n, 1))()
        for i, sp in enumerate(spheres):
            arr[i] = sp
        self._spheres = arr
        self.s.spheres = C.cast(arr, C.POINTER(Sphere)) if n else C.POINTER(Sphere)()
        self.s.n_spheres = n
        return self

    @property
    def spheres(self):
        return [self._spheres[i] for i in range(self.s.n_spheres)] if self.s.n_spheres else []

    def to_text(self) -> str:
        """Scene text (bhrt_scene_format_text): the reference's serialize_scene
        keys (config.cpp:96-112) plus the extension keys that differ from the
        defaults. The sky image is not part of the text."""
        from . import native
        n = C.c_size_t()
        native.lib().bhrt_scene_format_text(self.ptr(), None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        rc = native.lib().bhrt_scene_format_text(self.ptr(), buf, n.value + 1, C.byref(n))
        if rc:
            raise RuntimeError(f"bhrt_scene_format_text failed ({rc})")
        return buf.value.decode()

    @staticmethod
    def from_text(text: str, sky: np.ndarray | None = None) -> "SceneBuf":
        """Inverse of to_text (bhrt_scene_parse_text; parse_scene semantics for
        the reference keys, config.cpp:114-130). Raises UsageError-coded
        BhrtError on a malformed text, like the reference's UsageError."""
        from . import native
        from .abi import StatusInfo
        sb = SceneBuf()
        info = StatusInfo()
        need = C.c_int32()
        raw = text.encode()
        rc = native.lib().bhrt_scene_parse_text(raw, sb.ptr(), None, 0, C.byref(need), C.byref(info))
        if rc == 6 and need.value > 0:  # sphere buffer too small: retry with the count
            arr = (Sphere * need.value)()
            rc = native.lib().bhrt_scene_parse_text(raw, sb.ptr(), arr, need.value, C.byref(need),
                                                    C.byref(info))
            if rc == 0:
                sb.set_spheres(list(arr))
        native.check(rc, info)
        if sky is not None:
            sb.set_sky(sky)
        return sb

    @property
    def sky(self):
        return self._sky

    def clone(self) -> "SceneBuf":
        o = SceneBuf()
        C.memmove(C.byref(o.s), C.byref(self.s), C.sizeof(Scene))
        o._sky = self._sky
        o._spheres = self._spheres
        return o

    def ptr(self):
        return C.byref(self.s)


def scene_defaults(s: Scene) -> None:
    """Python mirror of bhrt_scene_defaults (checked against the C one)."""
    C.memset(C.byref(s), 0, C.sizeof(Scene))
    s.mass = 1.0
    s.cam_pos[2] = -20.0
    s.vertical_fov = 60.0 * PI / 180.0
    s.width = 256
    s.height = 256
    s.spp = 1
    s.max_windings = 10
    s.seed = 1
    s.epsilon = 0.05
    s.escape_radius = 1e4
    s.rel_tol = 1e-10
    s.abs_tol = 1e-12
    s.integrator = INTEGRATOR_REFERENCE
    s.sky_kind = SKY_IMAGE
    s.step = 1e-2
    s.max_step = 0.1
    s.chord_dphi = 0.01
    s.checker_nu = 16
    s.checker_nv = 8
    for i, v in enumerate((0.9, 0.9, 0.9)):
        s.checker_color_a[i] = v
    for i, v in enumerate((0.1, 0.1, 0.15)):
        s.checker_color_b[i] = v
    s.disk_r_in = 6.0
    s.disk_r_out = 20.0
    for i, v in enumerate((1.0, 0.95, 0.8)):
        s.disk_color_in[i] = v
    for i, v in enumerate((0.8, 0.25, 0.05)):
        s.disk_color_out[i] = v
    for i, v in enumerate((0.5, 1.0, -1.0)):
        s.light_dir[i] = v
    s.ambient = 0.1
    s.table_entries = 100000
    s.table_samples = 2048
    s.table_b_max = 50.0
    s.table_dpsi = 0.01


# ------------------------------------------------------------ reference scenes
def small_scene(bg: np.ndarray | None, size: int = 16, mass: float = 1.0) -> SceneBuf:
    """test_util.hpp:58-66."""
    sb = SceneBuf()
    sb.set(mass=mass, center=(0, 0, 0), cam_pos=(0, 0, -20), cam_look_at=(0, 0, 0),
           vertical_fov=60.0 * PI / 180.0, width=size, height=size, spp=1, seed=1,
           epsilon=0.1, escape_radius=60.0, max_windings=10, rel_tol=1e-10, abs_tol=1e-12)
    sb.set_sky(bg)
    return sb


def inclined_camera(radius: float, incl_deg: float, azimuth: float = 0.0):
    """Camera on a sphere of `radius` about the hole; inclination = angle
    between the view axis and the disk normal +y."""
    i = incl_deg * PI / 180.0
    return (radius * math.sin(i) * math.sin(azimuth), radius * math.cos(i),
            -radius * math.sin(i) * math.cos(azimuth))


SPHERE_SEED = 2507
JITTER_SEED = 2507


def make_spheres(n=64, seed=SPHERE_SEED, center=(0.0, 0.0, 0.0), shell=(8.0, 40.0),
                 radius=(0.5, 2.0), lib=None):
    """Seeded sphere field via the C ABI (bhrt_make_spheres) so that GPU path
    and oracle get identical doubles. `lib` defaults to the product library."""
    if lib is None:
        from . import native
        lib = native.lib()
        fn = lib.bhrt_make_spheres
    else:
        fn = lib.orc_make_spheres
    arr = (Sphere * n)()
    rc = fn(C.c_uint64(seed), n, (C.c_double * 3)(*center), shell[0], shell[1], radius[0],
            radius[1], C.cast(arr, C.POINTER(Sphere)))
    if rc != 0:
        raise ValueError(f"make_spheres failed: {rc}")
    return list(arr)


def config(idx: int, width: int | None = None, height: int | None = None,
           sphere_lib=None, frame: int = 0) -> SceneBuf:
    """BASELINE.json configs[idx] (sizes overridable for parity tests)."""
    sb = SceneBuf()
    sb.set(mass=1.0, center=(0, 0, 0), cam_look_at=(0, 0, 0), vertical_fov=60.0 * PI / 180.0,
           escape_radius=100.0, max_windings=10, sky_kind=SKY_CHECKER, checker_nu=16,
           checker_nv=8, disk_enabled=1, disk_r_in=6.0, disk_r_out=20.0)
    sb.set_sky(None)
    sb.s.sky_kind = SKY_CHECKER
    if idx in (0, 1, 3):
        sb.set(cam_pos=inclined_camera(20.0, 80.0), spp=1, seed=1)
        if idx == 0:
            sb.set(width=256, height=256, integrator=INTEGRATOR_RK4, step=1e-3)
        elif idx == 1:
            sb.set(width=1920, height=1080, integrator=INTEGRATOR_RKF45, step=1e-2,
                   rel_tol=1e-9, abs_tol=1e-9)
        else:
            sb.set(width=7680, height=4320, integrator=INTEGRATOR_TABLE, step=1e-2,
                   rel_tol=1e-9, abs_tol=1e-9, table_entries=100000, table_b_max=50.0)
    elif idx in (2, 4):
        sb.set(disk_r_out=30.0, spp=4, seed=JITTER_SEED, integrator=INTEGRATOR_RKF45, step=1e-2,
               rel_tol=1e-9, abs_tol=1e-9)
        sb.set_spheres(make_spheres(lib=sphere_lib))
        if idx == 2:
            sb.set(width=3840, height=2160, cam_pos=inclined_camera(30.0, 75.0))
        else:
            r = 15.0 + 35.0 * frame / 119.0
            psi = 2.0 * PI * frame / 120.0
            sb.set(width=1920, height=1080, cam_pos=inclined_camera(r, 75.0, psi))
    else:
        raise ValueError(idx)
    if width is not None:
        sb.s.width = width
    if height is not None:
        sb.s.height = height
    return sb


def sky_only_projection(sb: SceneBuf, sky_w: int = 2048, sky_h: int = 1024) -> SceneBuf:
    """What the reference can render of a config: same camera/hole/tolerances,
    no disk/spheres, the checker baked into a PPM, the reference integrator
    (DOPRI5 + epsilon windows, default epsilon 0.05) — SURVEY §8(d)."""
    o = sb.clone()
    o.set(integrator=INTEGRATOR_REFERENCE, disk_enabled=0, epsilon=0.05)
    o.set_spheres([])
    o.set_sky(checker_image(sky_w, sky_h, sb.s.checker_nu, sb.s.checker_nv,
                            tuple(sb.s.checker_color_a), tuple(sb.s.checker_color_b)))
    return o
