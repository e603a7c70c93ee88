// device_common.cuh — device helpers shared by the trace kernels.
//
// Everything here follows the reference's operation order (vec3.hpp:7-44,
// camera.cpp:10-68, geodesic.cpp:49-65) or the normative order of the
// oracle (oracle/bhrt_oracle.c) for the extensions; the kernels are compiled
// with --fmad=false so only the fma() calls written out below are fused.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "bhrt_kernel_params.h"

// Device bounds checks of the debug build (libbhrt_b200_debug.so,
// -DBHRT_DEBUG_BOUNDS; compute-sanitizer is not available on the GPU pool):
// a failed check traps the kernel and the render reports BHRT_DEVICE.
#ifdef BHRT_DEBUG_BOUNDS
#include <cassert>
#define BHRT_ASSERT(c) assert(c)
#else
#define BHRT_ASSERT(c) ((void)0)
#endif

namespace bhrt_b200 {

#define PI_D 3.141592653589793

// ----------------------------------------------------------------- vec3 (vec3.hpp:7-44 order)
struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 mk(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ V3 vld(const double* a) { return {a[0], a[1], a[2]}; }
__device__ __forceinline__ V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 scl(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ V3 dvd(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(V3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ V3 normalized(V3 a) {
    const double n = norm(a);
    return {a.x / n, a.y / n, a.z / n};
}
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// Order tests of doubles on the integer pipe (the FP64 pipe is the step
// loop's bound). For t > 0 and any x but NaN, x < t, x > t, x >= t agree
// with the signed comparison of the bit patterns (negative x and -0 pattern
// below every positive one, positive doubles in increasing order, +inf on
// top); a +NaN x compares above t (callers say why that cannot change
// a result).
__device__ __forceinline__ long long dbits(double x) { return __double_as_longlong(x); }
__device__ __forceinline__ bool lt_pos(double x, double t) { return dbits(x) < dbits(t); }
__device__ __forceinline__ bool gt_pos(double x, double t) { return dbits(x) > dbits(t); }
__device__ __forceinline__ bool ge_pos(double x, double t) { return dbits(x) >= dbits(t); }

// ----------------------------------------------------------------- camera (camera.cpp:10-68)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

__device__ __forceinline__ V3 camera_dir_raw(const KParams& p, int px, int py, int sample) {
    double sx = 0.5, sy = 0.5;
    if (p.spp > 1) {
        // hash_counter(seed, px, py, 2s [+1]) (camera.cpp:21-28): the first
        // round is the per-frame KParams::seed_mix = splitmix64(seed), the
        // next two are shared by the sample's x and y offsets
        const uint64_t h = splitmix64(splitmix64(p.seed_mix ^ (uint64_t)px) ^ (uint64_t)py);
        sx = to_unit(splitmix64(h ^ (2 * (uint64_t)sample)));
        sy = to_unit(splitmix64(h ^ (2 * (uint64_t)sample + 1)));
    }
    // (px + sx) / width as RN(a y) plus one Markstein correction with the
    // host's y = RN(1/width): the correctly rounded quotient for these
    // operands (a in [0, 2^16), width < 2^16: no under/overflow), i.e. the
    // same double as the division (tools/div_check.c checks every width < 2^16;
    // tests/test_abi.py::test_camera_division_is_exact).
    const double au = px + sx, av = py + sy;
    const double qu = au * p.inv_width, qv = av * p.inv_height;
    const double u = fma(fma(-qu, (double)p.width, au), p.inv_width, qu);
    const double v = fma(fma(-qv, (double)p.height, av), p.inv_height, qv);
    return add(add(vld(p.forward), scl(vld(p.right), (2.0 * u - 1.0) * p.tan_half_x)),
               scl(vld(p.up), (1.0 - 2.0 * v) * p.tan_half_y));
}

// generate_ray's unit direction (camera.cpp:49-52), reference-exact (mode R)
__device__ __forceinline__ V3 camera_ray(const KParams& p, int px, int py, int sample) {
    return normalized(camera_dir_raw(p, px, py, sample));
}

// Unit vector by one reciprocal (scene modes; oracle unit_fast).
__device__ __forceinline__ V3 unit_fast(V3 a) {
    const double inv = 1.0 / norm(a);
    return scl(a, inv);
}

// Scene-mode ray setup (RK4 / RKF45 / TABLE; oracle scene_frame):
// the orbital frame straight from the raw camera direction D. e1 and u0 are
// per-frame (KParams::cam_e1 / cam_u0); c = D.e1, T = D - c e1, e2 = T/|T|
// by one reciprocal, u0' = -(c/|T|) u0 (= the reference's -(v.d)/(r0 b),
// geodesic.cpp:57-65); radial iff |T|^2 < 1e-24 |D|^2 (geodesic.cpp:53).
struct Frame {
    V3 e2;
    double w;
    bool ok;
};
__device__ __forceinline__ Frame scene_frame(const KParams& p, V3 D) {
    Frame f;
    const V3 e1 = vld(p.cam_e1);
    const double c = dot(D, e1);
    const V3 T = sub(D, scl(e1, c));
    const double t2 = dot(T, T);
    f.ok = !(t2 < 1e-24 * dot(D, D));
    const double inv = 1.0 / sqrt(t2);
    f.e2 = scl(T, inv);
    f.w = -((c * inv) * p.cam_u0);
    return f;
}

// ----------------------------------------------------------------- geodesic helpers
// glibc 2.39 hypot restated (Borges, non-FMA kernel); bit-identical to the
// reference's std::hypot at geodesic.cpp:78 (verified: tests/test_oracle_geodesic.py).
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double t1, t2;
    double h = sqrt(ax * ax + ay * ay);
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    const double c = t1 + t2;
    if (c != 0.0) h -= c / (2.0 * h);  // c = +-0: h - (+-0) = h; skips the division's zero slow path
    return h;
}
__device__ inline double glibc_hypot(double x, double y) {
    {  // the common case first: finite, unscaled, neither term negligible —
       // exactly the branch of the full logic below that ends in hypot_kernel
       // (NaN/inf fail these comparisons and take the full logic). Mode R
       // 1080p sky-only: 84.6 -> 83.0 ms.
        const double fx = fabs(x), fy = fabs(y);
        const double hi = fx < fy ? fy : fx, lo = fx < fy ? fx : fy;
        if (hi <= 0x1p+511 && lo >= 0x1p-511 && lo > hi * 0x1p-54) return hypot_kernel(hi, lo);
    }
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return CUDART_INF;
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x;
    const double ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= ax * 0x1p-54) return ax + ay;
        return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
    }
    if (ay < 0x1p-511) {
        if (ax >= ay / 0x1p-54) return ax + ay;
        return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
    }
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax, ay);
}

struct Basis {
    V3 e1, e2;
    bool ok;
};

// geodesic.cpp:49-55. Every camera ray starts at the camera, so
// e1 = normalized(origin - center) is a per-frame constant (KParams::cam_e1,
// computed on the host with the same operations).
__device__ __forceinline__ Basis plane_basis(const KParams& p, V3 dir) {
    Basis b;
    b.e1 = vld(p.cam_e1);
    const V3 tangential = sub(dir, scl(b.e1, dot(dir, b.e1)));
    const double tn = norm(tangential);
    b.ok = !(tn < 1e-12);
    b.e2 = b.ok ? dvd(tangential, tn) : mk(0, 0, 0);
    return b;
}

// geodesic.cpp:57-65 (called only with a non-radial ray); v = origin - center,
// r0 = |v| and u0 = 1/r0 are per-frame constants (KParams::cam_v/cam_r0/cam_u0).
__device__ __forceinline__ void initial_conditions(const KParams& p, V3 dir, double& u, double& w) {
    const V3 v = vld(p.cam_v);
    const double b = norm(cross(v, dir));
    u = p.cam_u0;
    w = -dot(v, dir) / (p.cam_r0 * b);
}

// atan2 for the disk-line angle of the scene modes: t =
// min/max of |x|, |y| (one division), atan(t) = t + t s Q(s), s = t^2, with
// Q a degree-19 Chebyshev fit (mpmath, |rel err| < 2.3e-16 on [0, 1])
// evaluated by Estrin's scheme (8 dependent operations instead of 19 for
// Horner), then the octant fix-up with two-part pi/2, pi. Normative op order
// (oracle/bhrt_oracle.c atan2_est = device_common.cuh atan2_est). Finite
// arguments, not both zero.
// atan2_est's Chebyshev coefficients in the constant bank (as literals each
// costs two UMOV/IMAD per use); pairs (odd, even) of the Estrin first level.
static __constant__ double kAtanC[20] = {
    0x1.9999999999620p-3, -0x1.5555555555555p-2,
    0x1.c71c71bb00a6cp-4, -0x1.24924924753ecp-3,
    0x1.3b1399d1dcdc7p-4, -0x1.745d15ee35819p-4,
    0x1.e1d0239d392a6p-5, -0x1.110fff599e4d2p-4,
    0x1.841dcf603a209p-5, -0x1.aebbb1647a168p-5,
    0x1.3328700bb8169p-5, -0x1.5d02278205cc7p-5,
    0x1.843f4bca23369p-6, -0x1.00390504e9f2fp-5,
    0x1.123baedb61abdp-7, -0x1.fd0e4de8fed90p-7,
    0x1.1325b2f8964bep-10, -0x1.ca3677db66678p-9,
    0x1.2f07811f9f6e9p-16, -0x1.a359b96a4eee4p-13,
};
__device__ __forceinline__ double atan2_est(double y, double x) {
    const double ax = fabs(x), ay = fabs(y);
    const double mx = ax < ay ? ay : ax, mn = ax < ay ? ax : ay;
    const double t = mn / mx;
    const double s = t * t, s2 = s * s, s4 = s2 * s2, s8 = s4 * s4, s16 = s8 * s8;
    const double b0 = fma(kAtanC[0], s, kAtanC[1]);
    const double b1 = fma(kAtanC[2], s, kAtanC[3]);
    const double b2 = fma(kAtanC[4], s, kAtanC[5]);
    const double b3 = fma(kAtanC[6], s, kAtanC[7]);
    const double b4 = fma(kAtanC[8], s, kAtanC[9]);
    const double b5 = fma(kAtanC[10], s, kAtanC[11]);
    const double b6 = fma(kAtanC[12], s, kAtanC[13]);
    const double b7 = fma(kAtanC[14], s, kAtanC[15]);
    const double b8 = fma(kAtanC[16], s, kAtanC[17]);
    const double b9 = fma(kAtanC[18], s, kAtanC[19]);
    const double d0 = fma(b1, s2, b0);
    const double d1 = fma(b3, s2, b2);
    const double d2 = fma(b5, s2, b4);
    const double d3 = fma(b7, s2, b6);
    const double d4 = fma(b9, s2, b8);
    const double e0 = fma(d1, s4, d0), e1 = fma(d3, s4, d2);
    const double g0 = fma(e1, s8, e0);
    const double q = fma(d4, s16, g0);
    double r = fma(t * s, q, t);
    if (ay > ax) r = (0x1.921fb54442d18p+0 - r) + 0x1.1a62633145c07p-54;
    if (x < 0.0) r = (0x1.921fb54442d18p+1 - r) + 0x1.1a62633145c07p-53;
    return copysign(r, y);
}

// ----------------------------------------------------------------- record / stats helpers
// Per-warp counter totals, one 64-bit atomic per counter from lane 0. The
// per-lane counts are 32-bit; while every lane's count is below 2^26 the
// warp sum fits 32 bits and one REDUX (__reduce_add_sync) forms it,
// otherwise the 64-bit shuffle tree does.
__device__ __forceinline__ void warp_add_stats(unsigned long long* stats, unsigned steps, unsigned rej,
                                               unsigned rays) {
    unsigned long long s, r, n;
    if (__all_sync(0xffffffffu, steps < (1u << 26) && rej < (1u << 26))) {
        s = __reduce_add_sync(0xffffffffu, steps);
        r = __reduce_add_sync(0xffffffffu, rej);
        n = __reduce_add_sync(0xffffffffu, rays);
    } else {
        s = steps;
        r = rej;
        n = rays;
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, o);
            r += __shfl_down_sync(0xffffffffu, r, o);
            n += __shfl_down_sync(0xffffffffu, n, o);
        }
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* slot = stats + kStatStride * (blockIdx.x & (kStatSlots - 1));
        atomicAdd(&slot[0], s);
        atomicAdd(&slot[1], r);
        atomicAdd(&slot[2], n);
    }
}

struct SampleId {
    int x, y, s;
    long long rec;  // record index
};

// Thread i -> (pixel, sample). Fused shading: the spp samples of a pixel are
// adjacent lanes (i = pix*spp + s). Otherwise sample-major (i = s*plane + pix)
// and a separate shade kernel reads the records.
__device__ __forceinline__ SampleId sample_of(const KParams& p, long long i) {
    const long long plane = (long long)p.n_rows * p.width;
    SampleId id;
    long long pix;
    if (p.fused_shade) {  // spp divides 32: a power of two, so a shift
        const int sh = __ffs(p.spp) - 1;
        pix = i >> sh;
        id.s = (int)(i & (p.spp - 1));
    } else {
        id.s = (int)(i / plane);
        pix = i - (long long)id.s * plane;
    }
    int j;
    if (pix < 0x7fffffffLL) {  // 32-bit division when it fits (it does for 8K frames)
        // pix / width as the high word of pix * (floor(2^64 / width) + 1):
        // exact for pix < 2^31, width < 2^33 (the excess pix e / 2^64, e <= 1,
        // stays below 1 / width); width 1 has no 64-bit magic (div_magic = 0)
        j = p.div_magic ? (int)__umul64hi((unsigned long long)pix, p.div_magic) : (int)pix;
    } else {
        j = (int)(pix / p.width);
    }
    id.x = (int)(pix - (long long)j * p.width);
    id.y = packed_row_to_y(p, j);
    id.rec = pix * p.spp + id.s;
    return id;
}

// ----------------------------------------------------------------- shading
// image.cpp:131-169
__device__ static __noinline__ void sample_direction(const KParams& p, V3 d, double out[3]) {
    const double u_tex = (atan2(d.z, d.x) + PI_D) / (2.0 * PI_D);
    const double v_tex = (PI_D / 2.0 - asin(clampd(d.y, -1.0, 1.0))) / PI_D;
    const int w = p.sky_w, h = p.sky_h;
    const double x = u_tex * w - 0.5;
    const double y = v_tex * h - 0.5;
    const double fx = x - floor(x);
    const double fy = y - floor(y);
    int i0 = (int)floor(x) % w;
    if (i0 < 0) i0 += w;
    int i1 = ((int)floor(x) + 1) % w;
    if (i1 < 0) i1 += w;
    int j0 = (int)floor(y);
    j0 = j0 < 0 ? 0 : (j0 > h - 1 ? h - 1 : j0);
    int j1 = (int)floor(y) + 1;
    j1 = j1 < 0 ? 0 : (j1 > h - 1 ? h - 1 : j1);
    const uint8_t* p00 = p.sky + 3 * ((size_t)j0 * w + i0);
    const uint8_t* p10 = p.sky + 3 * ((size_t)j0 * w + i1);
    const uint8_t* p01 = p.sky + 3 * ((size_t)j1 * w + i0);
    const uint8_t* p11 = p.sky + 3 * ((size_t)j1 * w + i1);
    const double w00 = (1.0 - fx) * (1.0 - fy);
    const double w10 = fx * (1.0 - fy);
    const double w01 = (1.0 - fx) * fy;
    const double w11 = fx * fy;
#pragma unroll
    for (int c = 0; c < 3; ++c)
        out[c] = (__ldg(p00 + c) * w00 + __ldg(p10 + c) * w10 + __ldg(p01 + c) * w01 +
                  __ldg(p11 + c) * w11) / 255.0;
}

// Colour of one sample (oracle shade_object / sky): black for horizon and
// stalled rays (render.cpp:30-34), sky, disk ramp, Lambertian sphere.
// Inlining of the per-ray cold paths (measured on B200: inlining beats the
// call ABI's register spills, 11.6 -> 10.6 ms on config 2).
#ifndef BHRT_INL_SHADE
#define BHRT_INL_SHADE __forceinline__
#endif
#ifndef BHRT_INL_ESC
#define BHRT_INL_ESC __forceinline__
#endif
#ifndef BHRT_INL_EVT
#define BHRT_INL_EVT __forceinline__
#endif
#ifndef BHRT_INL_SPH
#define BHRT_INL_SPH __noinline__
#endif
#ifndef BHRT_INL_SETUP
#define BHRT_INL_SETUP  // compiler's choice (single call site)
#endif
__device__ static __forceinline__ void shade_sample_body(const KParams& p, int obj, int sphere, V3 pt,
                                                         double rgb[3]) {
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    if (obj == BHRT_OBJ_SKY) {
        if (p.sky_kind == BHRT_SKY_CHECKER) {
            int cu, cv;
            if (p.checker_nu <= kCheckerMax && p.checker_nv <= kCheckerMax) {
                // cell indices without atan2/asin: cu = #{k : atan2(z,x) >= theta_k},
                // cv = #{k : y <= cos(pi k / nv)}, thresholds from the host;
                // equal to the floor() form except within ulps of a cell edge
                // Both counts are monotone in k (ge(0) and y <= tab_v[0] = 1
                // always hold), so an fp32 estimate k0 whose exact tests give
                // ge(k0) && !ge(k0 + 1) is the count; the binary search decides
                // the rest (directions within ~1e-5 rad of a cell edge).
                const bool upper = !signbit(pt.z);  // atan2's half plane
                auto ge_u = [&](int k) {
                    const double ck = __ldg(p.checker_tab + k), sk = __ldg(p.checker_tab + kCheckerMax + k);
                    const bool kup = sk > 0.0 || (sk == 0.0 && ck > 0.0);
                    return upper != kup ? upper : (ck * pt.z - sk * pt.x >= 0.0);
                };
                const int nu = p.checker_nu, nv = p.checker_nv;
                const double y = clampd(pt.y, -1.0, 1.0);
                auto le_v = [&](int k) { return y <= __ldg(p.checker_tab + 2 * kCheckerMax + k); };
                const float fu = (atan2f((float)pt.z, (float)pt.x) + 3.14159265f) * (0.15915494f * (float)nu);
                const float fv = acosf((float)y) * (0.31830989f * (float)nv);
                const int ku = min(max((int)fu, 0), nu - 1), kv = min(max((int)fv, 0), nv - 1);
                if ((ku == 0 || ge_u(ku)) && (ku + 1 >= nu || !ge_u(ku + 1))) {
                    cu = ku;
                } else {
                    int lo = 0, hi = nu;  // count in [lo, hi)
                    while (hi - lo > 1) {
                        const int k = (lo + hi) >> 1;
                        if (ge_u(k)) lo = k; else hi = k;
                    }
                    cu = lo;
                }
                if ((kv == 0 || le_v(kv)) && (kv + 1 >= nv || !le_v(kv + 1))) {
                    cv = kv;
                } else {
                    int lo = 0, hi = nv;
                    while (hi - lo > 1) {
                        const int k = (lo + hi) >> 1;
                        if (le_v(k)) lo = k; else hi = k;
                    }
                    cv = lo;
                }
            } else {
                const double u_tex = (atan2(pt.z, pt.x) + PI_D) / (2.0 * PI_D);
                const double v_tex = (PI_D / 2.0 - asin(clampd(pt.y, -1.0, 1.0))) / PI_D;
                cu = (int)floor(u_tex * p.checker_nu);
                cv = (int)floor(v_tex * p.checker_nv);
                cu = cu < 0 ? 0 : (cu > p.checker_nu - 1 ? p.checker_nu - 1 : cu);
                cv = cv < 0 ? 0 : (cv > p.checker_nv - 1 ? p.checker_nv - 1 : cv);
            }
            const double* c = ((cu + cv) & 1) ? p.checker_b : p.checker_a;
            rgb[0] = c[0];
            rgb[1] = c[1];
            rgb[2] = c[2];
        } else {
            sample_direction(p, pt, rgb);
        }
    } else if (obj == BHRT_OBJ_DISK) {
        const V3 q = sub(pt, vld(p.center));
        const double rr = sqrt(q.x * q.x + q.z * q.z);
        const double t = (rr - p.disk_r_in) * p.disk_inv_width;  // oracle: one host reciprocal
#pragma unroll
        for (int c = 0; c < 3; ++c) rgb[c] = p.disk_c_in[c] + t * (p.disk_c_out[c] - p.disk_c_in[c]);
    } else if (obj == BHRT_OBJ_SPHERE) {
        const bhrt_sphere& sp = p.spheres[sphere];
        const V3 nrm = scl(sub(pt, vld(sp.center)), 1.0 / sp.radius);
        const double lam = dmax(0.0, dot(nrm, vld(p.light)));
        const double k = p.ambient + (1.0 - p.ambient) * lam;
#pragma unroll
        for (int c = 0; c < 3; ++c) rgb[c] = sp.albedo[c] * k;
    }
}

// Per translation unit: inlined (default) or a call (BHRT_INL_SHADE), see
// finish_sample's INL_SHADE for the per-instantiation choice.
__device__ static BHRT_INL_SHADE void shade_sample(const KParams& p, int obj, int sphere, V3 pt, double rgb[3]) {
    shade_sample_body(p, obj, sphere, pt, rgb);
}

// render.cpp:42-48: inv = 1/spp, round-half-away-from-zero, clamp to [0,255].
__device__ __forceinline__ void store_pixel(uint8_t* o, const double acc[3], double inv) {
    // inv = 1.0 / spp, formed once on the host (KParams::inv_spp)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double scaled = round(acc[c] * inv * 255.0);
        o[c] = (uint8_t)clampd(scaled, 0.0, 255.0);
    }
}

// Per-sample epilogue, called by EVERY lane of the warp (valid or not): the
// optional record, and in fused mode the sample colour, the pixel sum in
// sample order over the spp adjacent lanes (render.cpp:25-32) and the 8-bit
// store. A failed sample fails its pixel (lowest failing pixel -> stats[3]).
template <bool INL_SHADE = false>
__device__ __forceinline__ void finish_sample(const KParams& p, bool valid, const SampleId& id, int obj,
                                              int sphere, V3 point, double phi, unsigned steps,
                                              unsigned rej) {
    // failed samples carry (u at the failure, kind: 1 u <= 0, 2 step underflow)
    // for the host's failure text (bhrt_cuda.cu failure_text)
    const bool has_point = obj == BHRT_OBJ_SKY || obj == BHRT_OBJ_DISK || obj == BHRT_OBJ_SPHERE || obj < 0;
    if (valid && p.records) {
        bhrt_ray_record rec;
        BHRT_ASSERT(id.rec >= 0 && id.rec < (long long)p.n_rows * p.width * p.spp);
        rec.object = obj;
        rec.sphere = sphere;
        rec.steps = (int)steps;
        rec.rejected = (int)rej;
        rec.point[0] = has_point ? point.x : 0.0;
        rec.point[1] = has_point ? point.y : 0.0;
        rec.point[2] = has_point ? point.z : 0.0;
        rec.phi = phi;
        p.records[id.rec] = rec;
    }
    if (!p.fused_shade) return;
    double rgb[3] = {0.0, 0.0, 0.0};
    int bad = 0;
    if (valid) {
        if (obj < 0)
            bad = 1;
        else
#ifdef BHRT_EXPERIMENT_NOSHADE
            rgb[0] = point.x;  // timing experiment only: no shading code
#else
        {
            if (INL_SHADE)
                shade_sample_body(p, obj, sphere, point, rgb);
            else
                shade_sample(p, obj, sphere, point, rgb);
        }
#endif
    }
    const int lane = threadIdx.x & 31;
    const int base = lane & ~(p.spp - 1);
    double acc[3] = {0.0, 0.0, 0.0};
    int anybad = 0;
    for (int q = 0; q < p.spp; ++q) {
        acc[0] += __shfl_sync(0xffffffffu, rgb[0], base + q);
        acc[1] += __shfl_sync(0xffffffffu, rgb[1], base + q);
        acc[2] += __shfl_sync(0xffffffffu, rgb[2], base + q);
        anybad |= __shfl_sync(0xffffffffu, bad, base + q);
    }
    if (valid && id.s == 0) {
        const long long pix = id.rec >> (__ffs(p.spp) - 1);  // fused: spp is a power of two
        BHRT_ASSERT(id.x >= 0 && id.x < p.width && id.y >= p.row_start && id.y < p.row_end &&
                    pix >= 0 && pix < (long long)p.n_rows * p.width);
        uint8_t* o = p.out + 3 * (p.out_image ? (long long)id.y * p.width + id.x : pix);
        if (anybad) {
            atomicMin(&p.stats[3], (unsigned long long)id.y * p.width + id.x);  // image order
            o[0] = o[1] = o[2] = 0;
        } else {
            store_pixel(o, acc, p.inv_spp);
        }
    }
}

// ================================================================= RK4 / RKF45 scene modes
// Fehlberg tableau. Entries that are short fp64 immediates (low word zero)
// stay literal; the rest live in constant bank 3, which DFMA reads as an
// operand — as literals each would be rematerialised with two UMOVs per use
// inside the step loop (128-register cap). Same double values either way.
#define F21 (1.0 / 4.0)
#define F31 (3.0 / 32.0)
#define F32 (9.0 / 32.0)
#define F52 (-8.0)
#define F62 (2.0)
static __constant__ double kRkf[20] = {
    1932.0 / 2197.0, -7200.0 / 2197.0, 7296.0 / 2197.0,                       // F41 F42 F43
    439.0 / 216.0, 3680.0 / 513.0, -845.0 / 4104.0,                           // F51 F53 F54
    -8.0 / 27.0, -3544.0 / 2565.0, 1859.0 / 4104.0, -11.0 / 40.0,             // F61 F63 F64 F65
    16.0 / 135.0, 6656.0 / 12825.0, 28561.0 / 56430.0, -9.0 / 50.0, 2.0 / 55.0,  // G1 G3 G4 G5 G6
    1.0 / 360.0, -128.0 / 4275.0, -2197.0 / 75240.0, 1.0 / 50.0, 2.0 / 55.0};    // H1 H3 H4 H5 H6
#define F41 (kRkf[0])
#define F42 (kRkf[1])
#define F43 (kRkf[2])
#define F51 (kRkf[3])
#define F53 (kRkf[4])
#define F54 (kRkf[5])
#define F61 (kRkf[6])
#define F63 (kRkf[7])
#define F64 (kRkf[8])
#define F65 (kRkf[9])
#define G1 (kRkf[10])
#define G3 (kRkf[11])
#define G4 (kRkf[12])
#define G5 (kRkf[13])
#define G6 (kRkf[14])
#define H1 (kRkf[15])
#define H3 (kRkf[16])
#define H4 (kRkf[17])
#define H5 (kRkf[18])
#define H6 (kRkf[19])

__device__ __forceinline__ double g_of(double U, double M3) { return U * fma(M3, U, -1.0); }

// One RKF45 step; normative operation order = oracle/bhrt_oracle.c rkf45_step.
__device__ __forceinline__ bool rkf45_step(double u, double w, double h, double M3, double rtol,
                                           double atol, double hmax, const double* grow,
                                           const double* shrink, double& un, double& wn, double& hn) {
    const double ku1 = w, kw1 = g_of(u, M3);
    double su, sw;
    su = F21 * ku1; sw = F21 * kw1;
    const double U2 = fma(h, su, u), W2 = fma(h, sw, w);
    const double ku2 = W2, kw2 = g_of(U2, M3);
    su = F31 * ku1; su = fma(F32, ku2, su);
    sw = F31 * kw1; sw = fma(F32, kw2, sw);
    const double U3 = fma(h, su, u), W3 = fma(h, sw, w);
    const double ku3 = W3, kw3 = g_of(U3, M3);
    su = F41 * ku1; su = fma(F42, ku2, su); su = fma(F43, ku3, su);
    sw = F41 * kw1; sw = fma(F42, kw2, sw); sw = fma(F43, kw3, sw);
    const double U4 = fma(h, su, u), W4 = fma(h, sw, w);
    const double ku4 = W4, kw4 = g_of(U4, M3);
    su = F51 * ku1; su = fma(F52, ku2, su); su = fma(F53, ku3, su); su = fma(F54, ku4, su);
    sw = F51 * kw1; sw = fma(F52, kw2, sw); sw = fma(F53, kw3, sw); sw = fma(F54, kw4, sw);
    const double U5 = fma(h, su, u), W5 = fma(h, sw, w);
    const double ku5 = W5, kw5 = g_of(U5, M3);
    su = F61 * ku1; su = fma(F62, ku2, su); su = fma(F63, ku3, su); su = fma(F64, ku4, su);
    su = fma(F65, ku5, su);
    sw = F61 * kw1; sw = fma(F62, kw2, sw); sw = fma(F63, kw3, sw); sw = fma(F64, kw4, sw);
    sw = fma(F65, kw5, sw);
    const double U6 = fma(h, su, u), W6 = fma(h, sw, w);
    const double ku6 = W6, kw6 = g_of(U6, M3);
    su = G1 * ku1; su = fma(G3, ku3, su); su = fma(G4, ku4, su); su = fma(G5, ku5, su);
    su = fma(G6, ku6, su);
    sw = G1 * kw1; sw = fma(G3, kw3, sw); sw = fma(G4, kw4, sw); sw = fma(G5, kw5, sw);
    sw = fma(G6, kw6, sw);
    const double u_new = fma(h, su, u), w_new = fma(h, sw, w);
    su = H1 * ku1; su = fma(H3, ku3, su); su = fma(H4, ku4, su); su = fma(H5, ku5, su);
    su = fma(H6, ku6, su);
    sw = H1 * kw1; sw = fma(H3, kw3, sw); sw = fma(H4, kw4, sw); sw = fma(H5, kw5, sw);
    sw = fma(H6, kw6, sw);
    // |.| as operand modifiers of the compares and an integer mask of the
    // high word (hiword(|x|) = hiword(x) & 0x7fffffff for every x), max by
    // compare-select
    const double eus = h * su, ews = h * sw;
    const double du = fma(rtol, dmax(fabs(u), fabs(u_new)), atol);
    const double dw = fma(rtol, dmax(fabs(w), fabs(w_new)), atol);
    const bool err_ok = (fabs(eus) <= du) && (fabs(ews) <= dw);
    const bool geo_ok = u_new >= 0.5 * u;  // (the integer form: more instructions, 5.97 vs 5.92 ms)
    const int du_ = (__double2hiint(eus) & 0x7fffffff) - __double2hiint(du);
    const int dw_ = (__double2hiint(ews) & 0x7fffffff) - __double2hiint(dw);
    int q = (du_ > dw_ ? du_ : dw_) >> 18;
    q = q < kQMin ? kQMin : (q > kQMin + kQN - 1 ? kQMin + kQN - 1 : q);
    BHRT_ASSERT(q - kQMin >= 0 && q - kQMin < kQN);
    if (err_ok && geo_ok) {
        un = u_new;
        wn = w_new;
        const double hg = h * grow[q - kQMin];  // positive: min by the integer order
        hn = lt_pos(hmax, hg) ? hmax : hg;
        return true;
    }
    hn = err_ok ? 0.5 * h : h * shrink[q - kQMin];
    return false;
}

// tests/oracles.hpp:23-30 (reference arithmetic, no FMA)
__device__ __forceinline__ void rk4_step(double u, double w, double h, double mass, double& un,
                                         double& wn) {
    const double k1u = w, k1w = 3.0 * mass * u * u - u;
    const double a2 = u + 0.5 * h * k1u, b2 = w + 0.5 * h * k1w;
    const double k2u = b2, k2w = 3.0 * mass * a2 * a2 - a2;
    const double a3 = u + 0.5 * h * k2u, b3 = w + 0.5 * h * k2w;
    const double k3u = b3, k3w = 3.0 * mass * a3 * a3 - a3;
    const double a4 = u + h * k3u, b4 = w + h * k3w;
    const double k4u = b4, k4w = 3.0 * mass * a4 * a4 - a4;
    un = u + h / 6.0 * (k1u + 2.0 * k2u + 2.0 * k3u + k4u);
    wn = w + h / 6.0 * (k1w + 2.0 * k2w + 2.0 * k3w + k4w);
}

// Cubic Hermite interpolant of u over one step in monomial form (oracle
// hermite_coef / hermite_eval / hermite_deval, same op order).
struct Cubic {
    double a0, a1, a2, a3;
};
__device__ __forceinline__ Cubic hermite_coef(double h, double ua, double wa, double ub, double wb) {
    Cubic c;
    c.a0 = ua;
    c.a1 = h * wa;
    c.a2 = 3.0 * (ub - ua) - h * (2.0 * wa + wb);
    c.a3 = 2.0 * (ua - ub) + h * (wa + wb);
    return c;
}
__device__ __forceinline__ double hermite_eval(const Cubic& c, double t) {
    return fma(fma(fma(c.a3, t, c.a2), t, c.a1), t, c.a0);
}
__device__ __forceinline__ double hermite_deval(const Cubic& c, double t) {
    return fma(fma(3.0 * c.a3, t, 2.0 * c.a2), t, c.a1);
}

}  // namespace bhrt_b200
