// trace.cu — sm_100a kernels of the Schwarzschild ray-tracing hot path.
//
//   trace_reference_kernel : the reference algorithm (DOPRI5(4)+PI inside
//                            epsilon-windows, geodesic.cpp:84-238) per sample
//   trace_scene_kernel<I>  : RK4 (tests/oracles.hpp:23-55) / RKF45 renderers
//                            with disk + sphere polyline hit tests
//   shade_kernel           : per-pixel sample average + 8-bit quantisation
//                            (render.cpp:22-49) from the per-sample records
//
// Compiled with --fmad=false: every a*b+c written below is two roundings,
// exactly like the reference's x86-64 build and the oracle; the RKF45 path
// spells its fused multiply-adds out with fma(). Division and sqrt are IEEE
// (no fast-math), so all integration arithmetic is bit-identical to the CPU
// oracle; only libdevice transcendentals (sin/cos/atan2/asin/pow) may differ
// from glibc by ulps, and those sit outside the per-step path.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "bhrt_kernel_params.h"

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

// ----------------------------------------------------------------- camera (camera.cpp:10-68)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
__device__ __forceinline__ uint64_t hash_counter(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t h = splitmix64(seed);
    h = splitmix64(h ^ a);
    h = splitmix64(h ^ b);
    h = splitmix64(h ^ c);
    return h;
}

__device__ __forceinline__ V3 camera_ray(const KParams& p, int px, int py, int sample) {
    double sx = 0.5, sy = 0.5;
    if (p.spp > 1) {
        sx = to_unit(hash_counter(p.seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample));
        sy = to_unit(hash_counter(p.seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample + 1));
    }
    const double u = (px + sx) / p.width;
    const double v = (py + sy) / p.height;
    const V3 d = add(add(vld(p.forward), scl(vld(p.right), (2.0 * u - 1.0) * p.tan_half_x)),
                     scl(vld(p.up), (1.0 - 2.0 * v) * p.tan_half_y));
    return normalized(d);
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
    h -= (t1 + t2) / (2.0 * h);
    return h;
}
__device__ double glibc_hypot(double x, double y) {
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

// geodesic.cpp:49-55
__device__ __forceinline__ Basis plane_basis(V3 origin, V3 dir, V3 center) {
    Basis b;
    b.e1 = normalized(sub(origin, center));
    const V3 tangential = sub(dir, scl(b.e1, dot(dir, b.e1)));
    b.ok = !(norm(tangential) < 1e-12);
    b.e2 = b.ok ? normalized(tangential) : mk(0, 0, 0);
    return b;
}

// geodesic.cpp:57-65 (called only with a non-radial ray)
__device__ __forceinline__ void initial_conditions(V3 origin, V3 dir, V3 center, double& u, double& w) {
    const V3 v = sub(origin, center);
    const double r0 = norm(v);
    const double b = norm(cross(v, dir));
    u = 1.0 / r0;
    w = -dot(v, dir) / (r0 * b);
}

// ----------------------------------------------------------------- record / stats helpers
__device__ __forceinline__ void warp_add_stats(unsigned long long* stats, unsigned long long steps,
                                               unsigned long long rej, unsigned long long rays) {
    for (int o = 16; o > 0; o >>= 1) {
        steps += __shfl_down_sync(0xffffffffu, steps, o);
        rej += __shfl_down_sync(0xffffffffu, rej, o);
        rays += __shfl_down_sync(0xffffffffu, rays, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&stats[0], steps);
        atomicAdd(&stats[1], rej);
        atomicAdd(&stats[2], rays);
    }
}

struct SampleId {
    int x, y, s;
    long long rec;  // record index
};

__device__ __forceinline__ SampleId sample_of(const KParams& p, long long i) {
    const long long plane = (long long)p.n_rows * p.width;
    SampleId id;
    id.s = (int)(i / plane);
    const long long pix = i - (long long)id.s * plane;
    const int j = (int)(pix / p.width);
    id.x = (int)(pix - (long long)j * p.width);
    id.y = packed_row_to_y(p, j);
    id.rec = pix * p.spp + id.s;
    return id;
}

// ================================================================= mode R
// Dormand-Prince 5(4) tableau (geodesic.cpp:89-100), same constant expressions.
#define A21 (1.0 / 5.0)
#define A31 (3.0 / 40.0)
#define A32 (9.0 / 40.0)
#define A41 (44.0 / 45.0)
#define A42 (-56.0 / 15.0)
#define A43 (32.0 / 9.0)
#define A51 (19372.0 / 6561.0)
#define A52 (-25360.0 / 2187.0)
#define A53 (64448.0 / 6561.0)
#define A54 (-212.0 / 729.0)
#define A61 (9017.0 / 3168.0)
#define A62 (-355.0 / 33.0)
#define A63 (46732.0 / 5247.0)
#define A64 (49.0 / 176.0)
#define A65 (-5103.0 / 18656.0)
#define B1 (35.0 / 384.0)
#define B3 (500.0 / 1113.0)
#define B4 (125.0 / 192.0)
#define B5 (-2187.0 / 6784.0)
#define B6 (11.0 / 84.0)
#define E1 (71.0 / 57600.0)
#define E3 (-71.0 / 16695.0)
#define E4 (71.0 / 1920.0)
#define E5 (-17253.0 / 339200.0)
#define E6 (22.0 / 525.0)
#define E7 (-1.0 / 40.0)

__device__ __forceinline__ double rhs_w(double u, double mass) { return 3.0 * mass * u * u - u; }

// geodesic.cpp:84-162. Returns false on StepSizeUnderflow (phi/u/w then hold
// the failure state, as StepSizeUnderflow::state does).
__device__ bool integrate_window(double& phi, double& u, double& w, double dphi, double mass,
                                 double rtol, double atol, double& hint, unsigned& nsteps,
                                 unsigned& nrej) {
    double y0 = u, y1 = w;
    double k10 = y1, k11 = rhs_w(y0, mass);
    double remaining = dphi;
    double h = hint > 0.0 ? dmin(hint, dphi) : dphi;
    double err_prev = 1e-4;
    while (remaining > 0.0) {
        const double h_try = dmin(h, remaining);
        double t0, t1;
        t0 = y0 + h_try * A21 * k10;
        t1 = y1 + h_try * A21 * k11;
        const double k20 = t1, k21 = rhs_w(t0, mass);
        t0 = y0 + h_try * (A31 * k10 + A32 * k20);
        t1 = y1 + h_try * (A31 * k11 + A32 * k21);
        const double k30 = t1, k31 = rhs_w(t0, mass);
        t0 = y0 + h_try * (A41 * k10 + A42 * k20 + A43 * k30);
        t1 = y1 + h_try * (A41 * k11 + A42 * k21 + A43 * k31);
        const double k40 = t1, k41 = rhs_w(t0, mass);
        t0 = y0 + h_try * (A51 * k10 + A52 * k20 + A53 * k30 + A54 * k40);
        t1 = y1 + h_try * (A51 * k11 + A52 * k21 + A53 * k31 + A54 * k41);
        const double k50 = t1, k51 = rhs_w(t0, mass);
        t0 = y0 + h_try * (A61 * k10 + A62 * k20 + A63 * k30 + A64 * k40 + A65 * k50);
        t1 = y1 + h_try * (A61 * k11 + A62 * k21 + A63 * k31 + A64 * k41 + A65 * k51);
        const double k60 = t1, k61 = rhs_w(t0, mass);
        const double n0 = y0 + h_try * (B1 * k10 + B3 * k30 + B4 * k40 + B5 * k50 + B6 * k60);
        const double n1 = y1 + h_try * (B1 * k11 + B3 * k31 + B4 * k41 + B5 * k51 + B6 * k61);
        const double k70 = n1, k71 = rhs_w(n0, mass);
        const double e0 = h_try * (E1 * k10 + E3 * k30 + E4 * k40 + E5 * k50 + E6 * k60 + E7 * k70);
        const double e1 = h_try * (E1 * k11 + E3 * k31 + E4 * k41 + E5 * k51 + E6 * k61 + E7 * k71);
        const double s0 = atol + rtol * dmax(fabs(y0), fabs(n0));
        const double s1 = atol + rtol * dmax(fabs(y1), fabs(n1));
        double err = 0.0;
        err += (e0 / s0) * (e0 / s0);
        err += (e1 / s1) * (e1 / s1);
        err = sqrt(err / 2.0);
        if (err <= 1.0) {
            y0 = n0;
            y1 = n1;
            k10 = k70;
            k11 = k71;
            remaining -= h_try;
            const double factor =
                clampd(0.9 * pow(err, -0.7 / 5.0) * pow(err_prev, 0.4 / 5.0), 0.2, 5.0);
            h = h_try * factor;
            err_prev = dmax(err, 1e-4);
            ++nsteps;
        } else {
            h = h_try * clampd(0.9 * pow(err, -0.2), 0.1, 0.9);
            ++nrej;
        }
        if (h < 1e-14 && remaining > 0.0) {
            phi = phi + (dphi - remaining);
            u = y0;
            w = y1;
            return false;
        }
    }
    hint = h;
    phi = phi + dphi;
    u = y0;
    w = y1;
    return true;
}

// OrbitalPlaneBasis::point (geodesic.cpp:37-39)
__device__ __forceinline__ V3 plane_point(V3 origin, V3 e1, V3 e2, double r, double phi) {
    return add(origin, scl(add(scl(e1, cos(phi)), scl(e2, sin(phi))), r));
}

__global__ void __launch_bounds__(128) trace_reference_kernel(const KParams p) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned nsteps = 0, nrej = 0;
    if (i < n) {
        const SampleId id = sample_of(p, i);
        bhrt_ray_record rec;
        rec.sphere = -1;
        rec.point[0] = rec.point[1] = rec.point[2] = 0.0;
        rec.phi = 0.0;
        const V3 origin = vld(p.cam_pos), center = vld(p.center);
        const V3 dir = camera_ray(p, id.x, id.y, id.s);
        const V3 v = sub(origin, center);
        const double r0 = norm(v);
        const Basis B = plane_basis(origin, dir, center);
        int obj;
        V3 edir = dir;
        if (!B.ok) {  // radial: geodesic.cpp:175-187
            obj = dot(dir, sub(center, origin)) > 0.0 ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY;
            (void)r0;
        } else {
            double u, w, phi = 0.0, hint = 0.0;
            initial_conditions(origin, dir, center, u, w);
            double prev_phi = 0.0, prev_u = 0.0, last_phi = 0.0, last_u = 0.0;
            int npts = 1;
            obj = BHRT_OBJ_NONE;
            for (;;) {
                if (u >= p.u_cap) { obj = BHRT_OBJ_HORIZON; break; }
                if (u <= p.u_esc && w < 0.0) {
                    obj = BHRT_OBJ_SKY;
                    if (npts >= 2) {
                        const V3 last = plane_point(center, B.e1, B.e2, 1.0 / last_u, last_phi);
                        const V3 prev = npts == 2 ? origin
                                                  : plane_point(center, B.e1, B.e2, 1.0 / prev_u, prev_phi);
                        edir = normalized(sub(last, prev));
                    }
                    break;
                }
                if (phi > p.phi_max) { obj = BHRT_OBJ_STALLED; break; }
                // segment_dphi, geodesic.cpp:76-80
                const double hyp = glibc_hypot(u, w);
                const double dphi = clampd(p.epsilon * u * u / hyp, 1e-6, 0.1);
                if (!integrate_window(phi, u, w, dphi, p.mass, p.rel_tol, p.abs_tol, hint, nsteps, nrej)) {
                    if (p.mass > 0.0 && u >= p.u_cap) { obj = BHRT_OBJ_HORIZON; break; }
                    obj = -BHRT_NUMERICAL;
                    break;
                }
                if (!(u > 0.0)) { obj = -BHRT_NUMERICAL; break; }
                prev_phi = last_phi;
                prev_u = last_u;
                last_phi = phi;
                last_u = u;
                ++npts;
            }
            rec.phi = phi;
        }
        rec.object = obj;
        if (obj == BHRT_OBJ_SKY) {
            rec.point[0] = edir.x;
            rec.point[1] = edir.y;
            rec.point[2] = edir.z;
        }
        rec.steps = (int)nsteps;
        rec.rejected = (int)nrej;
        p.records[id.rec] = rec;
    }
    warp_add_stats(p.stats, nsteps, nrej, i < n ? 1ull : 0ull);
}

// ================================================================= RK4 / RKF45 scene modes
#define F21 (1.0 / 4.0)
#define F31 (3.0 / 32.0)
#define F32 (9.0 / 32.0)
#define F41 (1932.0 / 2197.0)
#define F42 (-7200.0 / 2197.0)
#define F43 (7296.0 / 2197.0)
#define F51 (439.0 / 216.0)
#define F52 (-8.0)
#define F53 (3680.0 / 513.0)
#define F54 (-845.0 / 4104.0)
#define F61 (-8.0 / 27.0)
#define F62 (2.0)
#define F63 (-3544.0 / 2565.0)
#define F64 (1859.0 / 4104.0)
#define F65 (-11.0 / 40.0)
#define G1 (16.0 / 135.0)
#define G3 (6656.0 / 12825.0)
#define G4 (28561.0 / 56430.0)
#define G5 (-9.0 / 50.0)
#define G6 (2.0 / 55.0)
#define H1 (1.0 / 360.0)
#define H3 (-128.0 / 4275.0)
#define H4 (-2197.0 / 75240.0)
#define H5 (1.0 / 50.0)
#define H6 (2.0 / 55.0)

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
    const double eu = fabs(h * su), ew = fabs(h * sw);
    const double du = fma(rtol, fmax(fabs(u), fabs(u_new)), atol);
    const double dw = fma(rtol, fmax(fabs(w), fabs(w_new)), atol);
    const bool err_ok = (eu <= du) && (ew <= dw);
    const bool geo_ok = u_new >= 0.5 * u;
    const int du_ = __double2hiint(eu) - __double2hiint(du);
    const int dw_ = __double2hiint(ew) - __double2hiint(dw);
    int q = (du_ > dw_ ? du_ : dw_) >> 18;
    q = q < kQMin ? kQMin : (q > kQMin + kQN - 1 ? kQMin + kQN - 1 : q);
    if (err_ok && geo_ok) {
        un = u_new;
        wn = w_new;
        hn = fmin(h * grow[q - kQMin], hmax);
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

struct SphereSm {  // per-block staged sphere data, relative to the hole centre
    double cx[kMaxSpheres], cy[kMaxSpheres], cz[kMaxSpheres], r[kMaxSpheres];
};

// Per-thread sphere-candidate slots live in shared memory, lane-major
// ([slot][thread]) so slot accesses are bank-conflict free. A slot holds the
// sphere index and a CONSERVATIVE fp32 angular window: the window only decides
// which steps run the exact fp64 hit test, so any superset of the oracle's
// windows gives bit-identical results.
constexpr int kBlock = 128;
constexpr int kSlots = 8;
constexpr float kWinMargin = 5e-4f;

struct CandSm {
    float lo[kSlots][kBlock];
    float hi[kSlots][kBlock];
    unsigned char k[kSlots][kBlock];
};

struct SceneRay {
    V3 O, e1, e2, n;
    double next_disk;   // +inf: no disk events
    double disk_sigma;  // +-1: half of the disk line of the next event
    double disk_lx, disk_ly;
    V3 disk_L;
    float next_sph;     // min window start over slots (-inf: test all)
    int nc;             // slots in use; -1: test every sphere every step
    int obj, sphere;
    V3 point;
};

__device__ __forceinline__ void sphere_window_f(double cx, double cy, double rho2, float& lo, float& hi) {
    const double rc2 = cx * cx + cy * cy;
    const double q = rc2 - rho2;  // rc^2 - rho^2
    if (!(q > 0.0)) {
        lo = -CUDART_INF_F;
        hi = CUDART_INF_F;
        return;
    }
    const float a = atan2f((float)sqrt(rho2), (float)sqrt(q));  // half-width asin(rho/rc)
    const float pc = atan2f((float)cy, (float)cx);
    lo = pc - a - kWinMargin;
    hi = pc + a + kWinMargin;
    if (hi < 0.0f) {
        lo += 2.0f * (float)PI_D;
        hi += 2.0f * (float)PI_D;
    }
}

__device__ void ray_events_setup(const KParams& p, const SphereSm& sm, CandSm& cs, SceneRay& R) {
    const int t = threadIdx.x;
    R.next_disk = CUDART_INF;
    R.disk_sigma = 1.0;
    if (p.disk_enabled) {
        const V3 L = mk(-R.n.z, 0.0, R.n.x);
        const double nl = norm(L);
        if (nl >= 1e-12) {
            const double lx = dot(L, R.e1), ly = dot(L, R.e2);
            const double pl = atan2(ly, lx);
            R.next_disk = pl > 0.0 ? pl : pl + PI_D;
            R.disk_sigma = pl > 0.0 ? 1.0 : -1.0;
            R.disk_lx = lx / nl;
            R.disk_ly = ly / nl;
            R.disk_L = dvd(L, nl);
        }
    }
    R.nc = 0;
    R.next_sph = CUDART_INF_F;
    for (int k = 0; k < p.n_spheres; ++k) {
        const V3 c = mk(sm.cx[k], sm.cy[k], sm.cz[k]);
        const double dn = dot(c, R.n);
        if (!(fabs(dn) < sm.r[k])) continue;
        if (R.nc == kSlots) {
            R.nc = -1;
            break;
        }
        const double cx = dot(c, R.e1), cy = dot(c, R.e2);
        const double rho2 = sm.r[k] * sm.r[k] - dn * dn;
        float lo, hi;
        sphere_window_f(cx, cy, rho2, lo, hi);
        cs.lo[R.nc][t] = lo;
        cs.hi[R.nc][t] = hi;
        cs.k[R.nc][t] = (unsigned char)k;
        R.next_sph = fminf(R.next_sph, lo);
        ++R.nc;
    }
    if (R.nc < 0) R.next_sph = -CUDART_INF_F;
}

__device__ __forceinline__ double hermite(double t, double h, double ua, double wa, double ub, double wb) {
    const double t2 = t * t, omt = 1.0 - t;
    const double h00 = (1.0 + 2.0 * t) * omt * omt;
    const double h10 = t * omt * omt;
    const double h01 = t2 * (3.0 - 2.0 * t);
    const double h11 = t2 * (t - 1.0);
    return h00 * ua + h10 * h * wa + h01 * ub + h11 * h * wb;
}

// Hit tests over one accepted step; mirrors oracle step_events() (same
// operation order): disk = exact phi-event on the Hermite interpolant,
// spheres = first entering hit on the step's equal-angle sub-chords.
__device__ __forceinline__ bool step_events(const KParams& p, const SphereSm& sm, CandSm& cs, SceneRay& R,
                                         double pa, double ua, double wa, double pb, double ub,
                                         double wb) {
    const int tid = threadIdx.x;
    const double h = pb - pa;
    // ---- disk
    bool disk_hit = false;
    double r_ev = 0.0, dlx = 0.0, dly = 0.0;
    if (R.next_disk > pa && R.next_disk <= pb) {
        const double t = (R.next_disk - pa) / h;
        const double u_ev = hermite(t, h, ua, wa, ub, wb);
        if (u_ev > 0.0) {
            r_ev = 1.0 / u_ev;
            if (r_ev >= p.disk_r_in && r_ev <= p.disk_r_out) {
                disk_hit = true;
                dlx = R.disk_sigma * R.disk_lx;
                dly = R.disk_sigma * R.disk_ly;
            }
        }
    }
    // ---- spheres
    const bool test_all = R.nc < 0;
    unsigned act = 0;
    if (!test_all) {
        const float fa = (float)pa, fb = (float)pb;
        for (int i = 0; i < R.nc; ++i)
            if (cs.lo[i][tid] <= fb && cs.hi[i][tid] >= fa) act |= 1u << i;
    }
    bool sph_hit = false;
    int bsph = -1;
    double bqx = 0.0, bqy = 0.0;
    if (act || test_all) {
        int S = 1;
        if (h > p.chord_dphi) S = (int)ceil(h / p.chord_dphi);
        const double dl = h / S;
        const double cd_ = cos(dl), sd_ = sin(dl);
        double cj = cos(pa), sj = sin(pa);
        const double rj = 1.0 / ua;
        double xj = cj * rj, yj = sj * rj;
        for (int j = 0; j < S && !sph_hit; ++j) {
            const double ck = cj * cd_ - sj * sd_;
            const double sk = sj * cd_ + cj * sd_;
            const double uk = (j + 1 == S) ? ub : hermite((double)(j + 1) / S, h, ua, wa, ub, wb);
            const double rk = 1.0 / uk;
            const double xk = ck * rk, yk = sk * rk;
            const double dx = xk - xj, dy = yk - yj;
            double best = CUDART_INF;
            const int ncand = test_all ? p.n_spheres : R.nc;
            for (int a = 0; a < ncand; ++a) {
                int k;
                if (test_all) {
                    k = a;
                } else {
                    if (!(act & (1u << a))) continue;
                    k = cs.k[a][tid];
                }
                const V3 c = mk(sm.cx[k], sm.cy[k], sm.cz[k]);
                const double dn = dot(c, R.n);
                if (!(fabs(dn) < sm.r[k])) continue;
                const double ccx = dot(c, R.e1), ccy = dot(c, R.e2);
                const double rho2 = sm.r[k] * sm.r[k] - dn * dn;
                const double mx = xj - ccx, my = yj - ccy;
                const double A = dx * dx + dy * dy;
                const double Bq = mx * dx + my * dy;
                const double Cq = mx * mx + my * my - rho2;
                if (!(Cq > 0.0)) continue;
                const double disc = Bq * Bq - A * Cq;
                if (disc < 0.0) continue;
                const double t = (-Bq - sqrt(disc)) / A;
                if (t >= 0.0 && t <= 1.0 && t < best) {
                    best = t;
                    sph_hit = true;
                    bsph = k;
                    bqx = xj + t * dx;
                    bqy = yj + t * dy;
                }
            }
            cj = ck;
            sj = sk;
            xj = xk;
            yj = yk;
        }
    }
    if (sph_hit && disk_hit) {
        if (bqx * dly - bqy * dlx > 0.0)
            disk_hit = false;
        else
            sph_hit = false;
    }
    bool hit = false;
    if (disk_hit) {
        hit = true;
        R.obj = BHRT_OBJ_DISK;
        R.sphere = -1;
        R.point = add(R.O, scl(R.disk_L, R.disk_sigma * r_ev));
    } else if (sph_hit) {
        hit = true;
        R.obj = BHRT_OBJ_SPHERE;
        R.sphere = bsph;
        R.point = add(R.O, add(scl(R.e1, bqx), scl(R.e2, bqy)));
    }
    while (R.next_disk <= pb) {
        R.next_disk += PI_D;
        R.disk_sigma = -R.disk_sigma;
    }
    if (!test_all) {
        R.next_sph = CUDART_INF_F;
        const float fb = (float)pb;
        for (int i = 0; i < R.nc; ++i) {
            float lo = cs.lo[i][tid], hi = cs.hi[i][tid];
            bool moved = false;
            while (hi < fb) {
                lo += 2.0f * (float)PI_D;
                hi += 2.0f * (float)PI_D;
                moved = true;
            }
            if (moved) {
                cs.lo[i][tid] = lo;
                cs.hi[i][tid] = hi;
            }
            R.next_sph = fminf(R.next_sph, lo);
        }
    }
    return hit;
}

__device__ __forceinline__ V3 tangent_dir(const SceneRay& R, double phi, double u, double w) {
    const double c = cos(phi), sn = sin(phi);
    const double tx = -u * sn - w * c, ty = u * c - w * sn;
    return normalized(add(scl(R.e1, tx), scl(R.e2, ty)));
}

__device__ __forceinline__ double hermite_d(double t, double h, double ua, double wa, double ub,
                                            double wb) {
    const double t2 = t * t;
    const double d00 = 6.0 * t2 - 6.0 * t;
    const double d10 = 3.0 * t2 - 4.0 * t + 1.0;
    const double d11 = 3.0 * t2 - 2.0 * t;
    return d00 * ua + d10 * h * wa - d00 * ub + d11 * h * wb;
}

// Tangent at the r = escape_radius crossing of the last step (oracle escape_dir).
__device__ __forceinline__ V3 escape_dir(const SceneRay& R, bool has_step, double pa, double ua, double wa,
                                      double pb, double ub, double wb, double u_esc, double energy,
                                      double M2) {
    if (!has_step || !(ua > u_esc)) return tangent_dir(R, pb, ub, wb);
    const double h = pb - pa;
    double t = (ua - u_esc) / (ua - ub);
    for (int it = 0; it < 2; ++it) {
        const double f = hermite(t, h, ua, wa, ub, wb) - u_esc;
        const double df = hermite_d(t, h, ua, wa, ub, wb);
        if (df != 0.0) t = t - f / df;
        t = clampd(t, 0.0, 1.0);
    }
    const double us = hermite(t, h, ua, wa, ub, wb);
    const double q = energy - us * us + M2 * us * us * us;
    const double ws = -sqrt(q > 0.0 ? q : 0.0);
    return tangent_dir(R, pa + h * t, us, ws);
}

__device__ void radial_scene(const KParams& p, const SphereSm& sm, SceneRay& R, V3 origin, V3 dir,
                             double seg_len, bool captured) {
    double best = seg_len;
    int obj = captured ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY, sph = -1;
    if (p.disk_enabled && dir.y != 0.0) {
        const double t = (R.O.y - origin.y) / dir.y;
        if (t >= 0.0 && t <= best) {
            const V3 q = sub(add(origin, scl(dir, t)), R.O);
            const double rq = sqrt(q.x * q.x + q.z * q.z);
            if (rq >= p.disk_r_in && rq <= p.disk_r_out) {
                best = t;
                obj = BHRT_OBJ_DISK;
            }
        }
    }
    for (int k = 0; k < p.n_spheres; ++k) {
        const bhrt_sphere& sp = p.spheres[k];
        const V3 m = sub(origin, vld(sp.center));
        const double B = dot(m, dir), Cq = dot(m, m) - sp.radius * sp.radius;
        if (!(Cq > 0.0)) continue;
        const double disc = B * B - Cq;
        if (disc < 0.0) continue;
        const double t = -B - sqrt(disc);
        if (t >= 0.0 && t < best) {
            best = t;
            obj = BHRT_OBJ_SPHERE;
            sph = k;
        }
    }
    R.obj = obj;
    R.sphere = sph;
    R.point = obj == BHRT_OBJ_SKY ? dir : add(origin, scl(dir, best));
}

template <int INTEG>
__global__ void __launch_bounds__(kBlock) trace_scene_kernel(const KParams p) {
    __shared__ SphereSm sm;
    __shared__ double s_grow[kQN], s_shrink[kQN];
    __shared__ CandSm cs;
    for (int k = threadIdx.x; k < p.n_spheres; k += blockDim.x) {
        const bhrt_sphere sp = p.spheres[k];
        sm.cx[k] = sp.center[0] - p.center[0];
        sm.cy[k] = sp.center[1] - p.center[1];
        sm.cz[k] = sp.center[2] - p.center[2];
        sm.r[k] = sp.radius;
    }
    if (INTEG == BHRT_INTEGRATOR_RKF45)
        for (int k = threadIdx.x; k < kQN; k += blockDim.x) {
            s_grow[k] = p.grow[k];
            s_shrink[k] = p.shrink[k];
        }
    __syncthreads();

    const long long n = (long long)p.n_rows * p.width * p.spp;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned nsteps = 0, nrej = 0;
    if (i < n) {
        const SampleId id = sample_of(p, i);
        bhrt_ray_record rec;
        rec.sphere = -1;
        rec.point[0] = rec.point[1] = rec.point[2] = 0.0;
        rec.phi = 0.0;
        const V3 origin = vld(p.cam_pos);
        const V3 dir = camera_ray(p, id.x, id.y, id.s);
        SceneRay R;
        R.O = vld(p.center);
        R.obj = BHRT_OBJ_NONE;
        R.sphere = -1;
        const Basis B = plane_basis(origin, dir, R.O);
        double phi = 0.0;
        if (!B.ok) {
            const double r0 = norm(sub(origin, R.O));
            const bool cap = dot(dir, sub(R.O, origin)) > 0.0;
            radial_scene(p, sm, R, origin, dir, cap ? r0 - 2.0 * p.mass : p.escape_radius, cap);
        } else {
            R.e1 = B.e1;
            R.e2 = B.e2;
            R.n = cross(R.e1, R.e2);
            double u, w;
            initial_conditions(origin, dir, R.O, u, w);
            ray_events_setup(p, sm, cs, R);
            double pp = 0.0, up = 0.0, wp = 0.0;  // state before the last accepted step
            bool has_step = false;
            const double M2 = 2.0 * p.mass;
            const double energy = w * w + u * u - M2 * u * u * u;
            if (INTEG == BHRT_INTEGRATOR_RK4) {
                const double h = p.step;
                for (;;) {
                    if (!(phi < p.phi_max)) { R.obj = BHRT_OBJ_STALLED; break; }
                    if (u >= p.u_cap) { R.obj = BHRT_OBJ_HORIZON; break; }
                    if (u <= p.u_esc && w < 0.0) {
                        R.obj = BHRT_OBJ_SKY;
                        break;
                    }
                    double un, wn;
                    rk4_step(u, w, h, p.mass, un, wn);
                    const double pn = phi + h;
                    ++nsteps;
                    if (pn >= dmin(R.next_disk, R.next_sph) && step_events(p, sm, cs, R, phi, u, w, pn, un, wn)) {
                        phi = pn;
                        break;
                    }
                    pp = phi;
                    up = u;
                    wp = w;
                    has_step = true;
                    phi = pn;
                    u = un;
                    w = wn;
                    if (!(u > 0.0)) { R.obj = -BHRT_NUMERICAL; break; }
                }
            } else {
                double h = p.step;
                for (;;) {
                    if (u >= p.u_cap) { R.obj = BHRT_OBJ_HORIZON; break; }
                    if (u <= p.u_esc && w < 0.0) {
                        R.obj = BHRT_OBJ_SKY;
                        break;
                    }
                    if (phi > p.phi_max) { R.obj = BHRT_OBJ_STALLED; break; }
                    double un, wn, hn;
                    if (rkf45_step(u, w, h, p.M3, p.rel_tol, p.abs_tol, p.max_step, s_grow, s_shrink, un, wn, hn)) {
                        const double pn = phi + h;
                        ++nsteps;
                        if (pn >= dmin(R.next_disk, R.next_sph) && step_events(p, sm, cs, R, phi, u, w, pn, un, wn)) {
                            phi = pn;
                            break;
                        }
                        pp = phi;
                        up = u;
                        wp = w;
                        has_step = true;
                        phi = pn;
                        u = un;
                        w = wn;
                        if (!(u > 0.0)) { R.obj = -BHRT_NUMERICAL; break; }
                    } else {
                        ++nrej;
                    }
                    h = hn;
                    if (h < 1e-14) {
                        R.obj = (p.mass > 0.0 && u >= p.u_cap) ? BHRT_OBJ_HORIZON : -BHRT_NUMERICAL;
                        break;
                    }
                }
            }
            if (R.obj == BHRT_OBJ_SKY)
                R.point = escape_dir(R, has_step, pp, up, wp, phi, u, w, p.u_esc, energy, M2);
        }
        rec.object = R.obj;
        rec.sphere = R.sphere;
        if (R.obj == BHRT_OBJ_SKY || R.obj == BHRT_OBJ_DISK || R.obj == BHRT_OBJ_SPHERE) {
            rec.point[0] = R.point.x;
            rec.point[1] = R.point.y;
            rec.point[2] = R.point.z;
        }
        rec.phi = phi;
        rec.steps = (int)nsteps;
        rec.rejected = (int)nrej;
        p.records[id.rec] = rec;
    }
    warp_add_stats(p.stats, nsteps, nrej, i < n ? 1ull : 0ull);
}

// ================================================================= shading
// image.cpp:131-169
__device__ void sample_direction(const KParams& p, V3 d, double out[3]) {
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

__device__ void shade_record(const KParams& p, const bhrt_ray_record& r, double rgb[3]) {
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    const V3 pt = vld(r.point);
    if (r.object == BHRT_OBJ_SKY) {
        if (p.sky_kind == BHRT_SKY_CHECKER) {
            const double u_tex = (atan2(pt.z, pt.x) + PI_D) / (2.0 * PI_D);
            const double v_tex = (PI_D / 2.0 - asin(clampd(pt.y, -1.0, 1.0))) / PI_D;
            int cu = (int)floor(u_tex * p.checker_nu);
            int cv = (int)floor(v_tex * p.checker_nv);
            cu = cu < 0 ? 0 : (cu > p.checker_nu - 1 ? p.checker_nu - 1 : cu);
            cv = cv < 0 ? 0 : (cv > p.checker_nv - 1 ? p.checker_nv - 1 : cv);
            const double* c = ((cu + cv) & 1) ? p.checker_b : p.checker_a;
            rgb[0] = c[0];
            rgb[1] = c[1];
            rgb[2] = c[2];
        } else {
            sample_direction(p, pt, rgb);
        }
    } else if (r.object == BHRT_OBJ_DISK) {
        const V3 q = sub(pt, vld(p.center));
        const double rr = sqrt(q.x * q.x + q.z * q.z);
        const double t = (rr - p.disk_r_in) / (p.disk_r_out - p.disk_r_in);
#pragma unroll
        for (int c = 0; c < 3; ++c) rgb[c] = p.disk_c_in[c] + t * (p.disk_c_out[c] - p.disk_c_in[c]);
    } else if (r.object == BHRT_OBJ_SPHERE) {
        const bhrt_sphere& sp = p.spheres[r.sphere];
        const V3 nrm = dvd(sub(pt, vld(sp.center)), sp.radius);
        const double lam = dmax(0.0, dot(nrm, vld(p.light)));
        const double k = p.ambient + (1.0 - p.ambient) * lam;
#pragma unroll
        for (int c = 0; c < 3; ++c) rgb[c] = sp.albedo[c] * k;
    }
}

// render.cpp:22-49: sample-order accumulation, inv = 1/spp, round-half-away, clamp.
__global__ void __launch_bounds__(256) shade_kernel(const KParams p) {
    const long long npix = (long long)p.n_rows * p.width;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    double acc[3] = {0.0, 0.0, 0.0};
    bool failed = false;
    for (int s = 0; s < p.spp; ++s) {
        const bhrt_ray_record r = p.records[i * p.spp + s];
        if (r.object < 0) {
            failed = true;
            break;
        }
        double c[3];
        shade_record(p, r, c);
        acc[0] += c[0];
        acc[1] += c[1];
        acc[2] += c[2];
    }
    uint8_t* o = p.out + 3 * i;
    if (failed) {
        // lowest failing pixel in image order: packed rows are ordered by y
        atomicMin(&p.stats[3], (unsigned long long)i);
        o[0] = o[1] = o[2] = 0;
        return;
    }
    const double inv = 1.0 / p.spp;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double scaled = round(acc[c] * inv * 255.0);
        o[c] = (uint8_t)clampd(scaled, 0.0, 255.0);
    }
}

// ----------------------------------------------------------------- launch wrappers
int launch_trace(const KParams& p, cudaStream_t st, int* launches, cudaEvent_t* ev) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    if (n <= 0) return 0;
    const int threads = 128;
    if (ev) cudaEventRecord(ev[0], st);
    const long long blocks = (n + threads - 1) / threads;
    switch (p.integrator) {
        case BHRT_INTEGRATOR_REFERENCE:
            trace_reference_kernel<<<(unsigned)blocks, threads, 0, st>>>(p);
            break;
        case BHRT_INTEGRATOR_RK4:
            trace_scene_kernel<BHRT_INTEGRATOR_RK4><<<(unsigned)blocks, threads, 0, st>>>(p);
            break;
        case BHRT_INTEGRATOR_RKF45:
            trace_scene_kernel<BHRT_INTEGRATOR_RKF45><<<(unsigned)blocks, threads, 0, st>>>(p);
            break;
        default:
            return -1;
    }
    ++*launches;
    if (ev) cudaEventRecord(ev[1], st);
    const long long npix = (long long)p.n_rows * p.width;
    shade_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(p);
    ++*launches;
    if (ev) cudaEventRecord(ev[2], st);
    return 0;
}

}  // namespace bhrt_b200
