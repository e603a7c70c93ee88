/*
 * bhrt_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY (see bhrt_oracle.h).
 *
 * Plain C restatement of the reference hot path. Build flags matter:
 * -ffp-contract=off so that every a*b+c is two roundings exactly like the
 * reference's x86-64 build (no FMA contraction), while the RKF45
 * path calls fma() explicitly where DESIGN.md §RKF45 specifies a fused op.
 * Reference citations are relative to /root/reference/proj.
 */
#include "bhrt_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.141592653589793 /* std::numbers::pi */

/* ------------------------------------------------------------------ */
/* Vec3 in the reference's operation order (vec3.hpp:7-44).           */
/* ------------------------------------------------------------------ */
typedef struct { double x, y, z; } v3;

static inline v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 vld(const double* a) { return mk(a[0], a[1], a[2]); }
static inline void vst(double* a, v3 v) { a[0] = v.x; a[1] = v.y; a[2] = v.z; }
static inline v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); } /* v*s and s*v */
static inline v3 dvd(v3 a, double s) { return mk(a.x / s, a.y / s, a.z / s); }
static inline double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 cross(v3 a, v3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double norm(v3 a) { return sqrt(dot(a, a)); }
static inline v3 normalized(v3 a) { const double n = norm(a); return mk(a.x / n, a.y / n, a.z / n); }
static inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static inline double dmax(double a, double b) { return a < b ? b : a; } /* std::max */
static inline double dmin(double a, double b) { return b < a ? b : a; } /* std::min */

/* ------------------------------------------------------------------ */
/* camera (camera.cpp:10-68)                                           */
/* ------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) { /* camera.cpp:12-17 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static double to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; } /* camera.cpp:20 */

uint64_t orc_hash_counter(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { /* camera.cpp:21-28 */
    uint64_t h = splitmix64(seed);
    h = splitmix64(h ^ a);
    h = splitmix64(h ^ b);
    h = splitmix64(h ^ c);
    return h;
}

int orc_camera_basis(const bhrt_scene* s, double f[3], double r[3], double u[3]) { /* camera.cpp:30-43 */
    const v3 axis = sub(vld(s->cam_look_at), vld(s->cam_pos));
    const double len = norm(axis);
    if (len == 0.0) return BHRT_INVALID_ARGUMENT;
    const v3 forward = dvd(axis, len);
    const v3 rr = cross(forward, mk(0.0, 1.0, 0.0));
    if (norm(rr) < 1e-9) return BHRT_INVALID_ARGUMENT;
    const v3 right = normalized(rr);
    const v3 up = cross(right, forward);
    vst(f, forward); vst(r, right); vst(u, up);
    return 0;
}

typedef struct {
    v3 forward, right, up;
    double tan_half_x, tan_half_y;
} cam_t;

static int cam_setup(const bhrt_scene* s, cam_t* c) {
    double f[3], r[3], u[3];
    const int st = orc_camera_basis(s, f, r, u);
    if (st) return st;
    c->forward = vld(f); c->right = vld(r); c->up = vld(u);
    /* camera.cpp:46-48 */
    c->tan_half_y = tan(s->vertical_fov / 2.0);
    const double aspect = (double)s->width / s->height;
    c->tan_half_x = c->tan_half_y * aspect;
    return 0;
}

/* camera.cpp:49-51 before the normalisation: D = f + (2u-1) thx r + (1-2v) thy up */
static v3 cam_dir_raw(const bhrt_scene* s, const cam_t* c, int px, int py, int sample) {
    double sx = 0.5, sy = 0.5; /* camera.cpp:55-65 */
    if (s->spp > 1) {
        sx = to_unit(orc_hash_counter(s->seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample));
        sy = to_unit(orc_hash_counter(s->seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample + 1));
    }
    const double u = (px + sx) / s->width;
    const double v = (py + sy) / s->height;
    return add(add(c->forward, scl(c->right, (2.0 * u - 1.0) * c->tan_half_x)),
               scl(c->up, (1.0 - 2.0 * v) * c->tan_half_y));
}

/* Unit vector by one reciprocal (scene modes; the reference's normalized()
 * divides three times, vec3.hpp:36-39). */
static inline v3 unit_fast(v3 a) { const double inv = 1.0 / norm(a); return scl(a, inv); }

static v3 cam_ray(const bhrt_scene* s, const cam_t* c, int px, int py, int sample) {
    double sx = 0.5, sy = 0.5; /* camera.cpp:55-65 */
    if (s->spp > 1) {
        sx = to_unit(orc_hash_counter(s->seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample));
        sy = to_unit(orc_hash_counter(s->seed, (uint64_t)px, (uint64_t)py, 2 * (uint64_t)sample + 1));
    }
    const double u = (px + sx) / s->width;
    const double v = (py + sy) / s->height;
    /* camera.cpp:49-51: f + ((2u-1)*thx)*r + ((1-2v)*thy)*up, normalised */
    const v3 d = add(add(c->forward, scl(c->right, (2.0 * u - 1.0) * c->tan_half_x)),
                     scl(c->up, (1.0 - 2.0 * v) * c->tan_half_y));
    return normalized(d);
}

int orc_generate_ray(const bhrt_scene* s, int px, int py, int sample, double origin[3], double dir[3]) {
    cam_t c;
    const int st = cam_setup(s, &c);
    if (st) return st;
    vst(dir, cam_ray(s, &c, px, py, sample));
    memcpy(origin, s->cam_pos, sizeof(double) * 3);
    return 0;
}

/* ------------------------------------------------------------------ */
/* sky (image.cpp:131-169) + procedural checker                        */
/* ------------------------------------------------------------------ */
void orc_sample_direction(const uint8_t* img, int w, int h, const double dir[3], double out[3]) {
    const double u_tex = (atan2(dir[2], dir[0]) + PI) / (2.0 * PI);
    const double v_tex = (PI / 2.0 - asin(clampd(dir[1], -1.0, 1.0))) / PI;
    const double x = u_tex * w - 0.5;
    const double y = v_tex * h - 0.5;
    const double fx = x - floor(x);
    const double fy = y - floor(y);
    int i0 = (int)floor(x) % w; if (i0 < 0) i0 += w;
    int i1 = ((int)floor(x) + 1) % w; if (i1 < 0) i1 += w;
    int j0 = (int)floor(y); j0 = j0 < 0 ? 0 : (j0 > h - 1 ? h - 1 : j0);
    int j1 = (int)floor(y) + 1; j1 = j1 < 0 ? 0 : (j1 > h - 1 ? h - 1 : j1);
    const uint8_t* p00 = img + 3 * ((size_t)j0 * w + i0);
    const uint8_t* p10 = img + 3 * ((size_t)j0 * w + i1);
    const uint8_t* p01 = img + 3 * ((size_t)j1 * w + i0);
    const uint8_t* p11 = img + 3 * ((size_t)j1 * w + i1);
    const double w00 = (1.0 - fx) * (1.0 - fy);
    const double w10 = fx * (1.0 - fy);
    const double w01 = (1.0 - fx) * fy;
    const double w11 = fx * fy;
    for (int c = 0; c < 3; ++c)
        out[c] = (p00[c] * w00 + p10[c] * w10 + p01[c] * w01 + p11[c] * w11) / 255.0;
}

/* Checker: same (u_tex, v_tex) map as image.cpp:133-134; cell parity. */
static void checker(const bhrt_scene* s, v3 d, double out[3]) {
    const double u_tex = (atan2(d.z, d.x) + PI) / (2.0 * PI);
    const double v_tex = (PI / 2.0 - asin(clampd(d.y, -1.0, 1.0))) / PI;
    int cu = (int)floor(u_tex * s->checker_nu);
    int cv = (int)floor(v_tex * s->checker_nv);
    cu = cu < 0 ? 0 : (cu > s->checker_nu - 1 ? s->checker_nu - 1 : cu);
    cv = cv < 0 ? 0 : (cv > s->checker_nv - 1 ? s->checker_nv - 1 : cv);
    const double* c = ((cu + cv) & 1) ? s->checker_color_b : s->checker_color_a;
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2];
}

static void sky(const bhrt_scene* s, v3 d, double out[3]) {
    if (s->sky_kind == BHRT_SKY_CHECKER) {
        checker(s, d, out);
    } else {
        const double dd[3] = {d.x, d.y, d.z};
        orc_sample_direction(s->sky_rgb, s->sky_width, s->sky_height, dd, out);
    }
}

/* ------------------------------------------------------------------ */
/* geodesic (geodesic.cpp)                                             */
/* ------------------------------------------------------------------ */
void orc_ode_rhs(double phi, double u, double w, double mass, double out[2]) {
    (void)phi;
    out[0] = w;
    out[1] = 3.0 * mass * u * u - u; /* geodesic.cpp:45-47 */
}

int orc_plane_basis(const double o[3], const double d[3], const double c[3], double e1o[3],
                    double e2o[3]) { /* geodesic.cpp:49-55 */
    const v3 dir = vld(d);
    const v3 e1 = normalized(sub(vld(o), vld(c)));
    const v3 tangential = sub(dir, scl(e1, dot(dir, e1)));
    if (norm(tangential) < 1e-12) return 0;
    vst(e1o, e1);
    vst(e2o, normalized(tangential));
    return 1;
}

int orc_initial_conditions(const double o[3], const double d[3], const double c[3], double st[3]) {
    const v3 v = sub(vld(o), vld(c)); /* geodesic.cpp:57-65 */
    const v3 dir = vld(d);
    const double r0 = norm(v);
    const double b = norm(cross(v, dir));
    if (b < 1e-12) return BHRT_INVALID_ARGUMENT;
    st[0] = 0.0;
    st[1] = 1.0 / r0;
    st[2] = -dot(v, dir) / (r0 * b);
    return 0;
}

double orc_step_dphi(double u, double epsilon) { return clampd(epsilon * u, 1e-6, 0.1); } /* :67-69 */

/* glibc 2.39 sysdeps/ieee754/dbl-64/e_hypot.c: Borges, "An Improved
 * Algorithm for hypot(a,b)", non-FMA kernel (x86-64 baseline build). The
 * reference calls std::hypot at geodesic.cpp:78; restating the library
 * algorithm lets the GPU reproduce it bit-for-bit. */
static double hypot_kernel(double ax, double ay) {
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
double orc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
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

double orc_segment_dphi(double u, double w, double epsilon) { /* geodesic.cpp:76-80 */
    const double hyp = hypot(u, w);
    return clampd(epsilon * u * u / hyp, 1e-6, 0.1);
}

/* Dormand-Prince 5(4) tableau, geodesic.cpp:89-100 (same constant expressions). */
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

static inline void rhs2(const double y[2], double mass, double k[2]) { /* geodesic.cpp:31-33 */
    k[0] = y[1];
    k[1] = 3.0 * mass * y[0] * y[0] - y[0];
}

int orc_integrate_window(const double state[3], double dphi, double mass, double rel_tol,
                         double abs_tol, double* step_hint, double out[3], int* nsteps,
                         int* nrej) { /* geodesic.cpp:84-162 */
    if (!(dphi > 0.0)) return BHRT_INVALID_ARGUMENT;
    double y[2] = {state[1], state[2]};
    double k1[2];
    rhs2(y, mass, k1);
    double remaining = dphi;
    double h = (step_hint && *step_hint > 0.0) ? dmin(*step_hint, dphi) : dphi;
    double err_prev = 1e-4;
    while (remaining > 0.0) {
        const double h_try = dmin(h, remaining);
        double k2[2], k3[2], k4[2], k5[2], k6[2], k7[2], ynew[2], t[2];
        for (int i = 0; i < 2; ++i) t[i] = y[i] + h_try * A21 * k1[i];
        rhs2(t, mass, k2);
        for (int i = 0; i < 2; ++i) t[i] = y[i] + h_try * (A31 * k1[i] + A32 * k2[i]);
        rhs2(t, mass, k3);
        for (int i = 0; i < 2; ++i) t[i] = y[i] + h_try * (A41 * k1[i] + A42 * k2[i] + A43 * k3[i]);
        rhs2(t, mass, k4);
        for (int i = 0; i < 2; ++i)
            t[i] = y[i] + h_try * (A51 * k1[i] + A52 * k2[i] + A53 * k3[i] + A54 * k4[i]);
        rhs2(t, mass, k5);
        for (int i = 0; i < 2; ++i)
            t[i] = y[i] + h_try * (A61 * k1[i] + A62 * k2[i] + A63 * k3[i] + A64 * k4[i] + A65 * k5[i]);
        rhs2(t, mass, k6);
        for (int i = 0; i < 2; ++i)
            ynew[i] = y[i] + h_try * (B1 * k1[i] + B3 * k3[i] + B4 * k4[i] + B5 * k5[i] + B6 * k6[i]);
        rhs2(ynew, mass, k7);

        double err = 0.0;
        for (int i = 0; i < 2; ++i) {
            const double ei =
                h_try * (E1 * k1[i] + E3 * k3[i] + E4 * k4[i] + E5 * k5[i] + E6 * k6[i] + E7 * k7[i]);
            const double scale = abs_tol + rel_tol * dmax(fabs(y[i]), fabs(ynew[i]));
            err += (ei / scale) * (ei / scale);
        }
        err = sqrt(err / 2.0);

        if (err <= 1.0) {
            y[0] = ynew[0]; y[1] = ynew[1];
            k1[0] = k7[0]; k1[1] = k7[1];
            remaining -= h_try;
            const double factor =
                clampd(0.9 * pow(err, -0.7 / 5.0) * pow(err_prev, 0.4 / 5.0), 0.2, 5.0);
            h = h_try * factor;
            err_prev = dmax(err, 1e-4);
            if (nsteps) ++*nsteps;
        } else {
            h = h_try * clampd(0.9 * pow(err, -0.2), 0.1, 0.9);
            if (nrej) ++*nrej;
        }
        if (h < 1e-14 && remaining > 0.0) {
            out[0] = state[0] + (dphi - remaining);
            out[1] = y[0];
            out[2] = y[1];
            return 1;
        }
    }
    if (step_hint) *step_hint = h;
    out[0] = state[0] + dphi;
    out[1] = y[0];
    out[2] = y[1];
    return 0;
}

/* OrbitalPlaneBasis::point, geodesic.cpp:37-39 */
static inline v3 plane_point(v3 origin, v3 e1, v3 e2, double r, double phi) {
    return add(origin, scl(add(scl(e1, cos(phi)), scl(e2, sin(phi))), r));
}

int orc_trace_reference(const double o[3], const double d[3], double mass, const double c[3],
                        double epsilon, double escape_radius, int max_windings, double rel_tol,
                        double abs_tol, int* kind, double dir_out[3], int* npoints, double last2[6],
                        int* nsteps, int* nrej) { /* geodesic.cpp:164-238 */
    if (!(epsilon > 0.0) || !(escape_radius > 0.0) || max_windings < 1 || !(rel_tol > 0.0) ||
        !(abs_tol > 0.0) || mass < 0.0)
        return BHRT_INVALID_ARGUMENT;
    const v3 origin = vld(o), dir = vld(d), center = vld(c);
    const v3 v = sub(origin, center);
    const double r0 = norm(v);
    if (mass > 0.0 && r0 <= 2.0 * mass) return BHRT_INVALID_ARGUMENT;
    if (nsteps) *nsteps = 0;
    if (nrej) *nrej = 0;

    double e1a[3], e2a[3];
    if (!orc_plane_basis(o, d, c, e1a, e2a)) { /* radial: geodesic.cpp:175-187 */
        v3 p1;
        if (dot(dir, sub(center, origin)) > 0.0) {
            p1 = add(origin, scl(dir, r0 - 2.0 * mass));
            *kind = 0;
        } else {
            p1 = add(origin, scl(dir, escape_radius));
            *kind = 1;
            vst(dir_out, dir);
        }
        *npoints = 2;
        vst(last2, origin);
        vst(last2 + 3, p1);
        return 0;
    }
    const v3 e1 = vld(e1a), e2 = vld(e2a);
    double st[3];
    orc_initial_conditions(o, d, c, st);
    const double u_capture = mass > 0.0 ? 1.0 / (2.0 * mass) : INFINITY;
    const double u_escape = 1.0 / escape_radius;
    const double phi_max = 2.0 * PI * max_windings;

    v3 prev = origin, last = origin; /* the polyline's last two points */
    int npts = 1;
    double hint = 0.0;
    for (;;) {
        if (st[1] >= u_capture) { *kind = 0; break; }
        if (st[1] <= u_escape && st[2] < 0.0) {
            *kind = 1;
            if (npts < 2) {
                prev = origin;
                last = add(origin, scl(dir, escape_radius));
                npts = 2;
                vst(dir_out, dir);
            } else {
                vst(dir_out, normalized(sub(last, prev)));
            }
            break;
        }
        if (st[0] > phi_max) { *kind = 2; break; }
        const double dphi = orc_segment_dphi(st[1], st[2], epsilon);
        double nx[3];
        const int rc = orc_integrate_window(st, dphi, mass, rel_tol, abs_tol, &hint, nx, nsteps, nrej);
        if (rc == 1) { /* StepSizeUnderflow: geodesic.cpp:224-231 */
            if (mass > 0.0 && nx[1] >= u_capture) {
                const v3 p = plane_point(center, e1, e2, 1.0 / nx[1], nx[0]);
                if (norm(sub(p, last)) > 0.0) { prev = last; last = p; ++npts; }
                *kind = 0;
                break;
            }
            return BHRT_NUMERICAL;
        }
        st[0] = nx[0]; st[1] = nx[1]; st[2] = nx[2];
        if (!(st[1] > 0.0)) return BHRT_NUMERICAL; /* geodesic.cpp:233-234 */
        prev = last;
        last = plane_point(center, e1, e2, 1.0 / st[1], st[0]);
        ++npts;
    }
    *npoints = npts;
    vst(last2, prev);
    vst(last2 + 3, last);
    return 0;
}

int orc_deflection_of_ray(const double o[3], const double d[3], double mass, const double c[3],
                          double epsilon, double escape_radius, int max_windings, double rel_tol,
                          double abs_tol, double* out) { /* geodesic.cpp:240-262 */
    /* Needs the whole polyline: re-run the window loop keeping every point. */
    double e1a[3], e2a[3];
    const int has_basis = orc_plane_basis(o, d, c, e1a, e2a);
    int kind, np, ns, nr;
    double dir[3], l2[6];
    const int rc = orc_trace_reference(o, d, mass, c, epsilon, escape_radius, max_windings, rel_tol,
                                       abs_tol, &kind, dir, &np, l2, &ns, &nr);
    if (rc) return rc;
    if (kind != 1) return BHRT_NUMERICAL;
    if (!has_basis) { *out = 0.0; return 0; }
    const v3 origin = vld(o), center = vld(c), e1 = vld(e1a), e2 = vld(e2a);
    double st[3];
    orc_initial_conditions(o, d, c, st);
    const double u_escape = 1.0 / escape_radius;
    double hint = 0.0, total = 0.0, prev_x = 0.0, prev_y = 0.0;
    v3 p_prev = origin;
    int i = 0;
    while (!(st[1] <= u_escape && st[2] < 0.0)) {
        const double dphi = orc_segment_dphi(st[1], st[2], epsilon);
        double nx[3];
        orc_integrate_window(st, dphi, mass, rel_tol, abs_tol, &hint, nx, NULL, NULL);
        memcpy(st, nx, sizeof st);
        const v3 p = plane_point(center, e1, e2, 1.0 / st[1], st[0]);
        const v3 seg = sub(p, p_prev);
        const double sx = dot(seg, e1), sy = dot(seg, e2);
        ++i;
        if (i > 1) total += atan2(prev_x * sy - prev_y * sx, prev_x * sx + prev_y * sy);
        prev_x = sx;
        prev_y = sy;
        p_prev = p;
    }
    *out = fabs(total);
    return 0;
}

double orc_conserved_energy(double u, double w, double mass) { /* geodesic.cpp:272-275 */
    return w * w + u * u - 2.0 * mass * u * u * u;
}

/* ------------------------------------------------------------------ */
/* RK4 — the reference test oracle (tests/oracles.hpp:19-55)            */
/* ------------------------------------------------------------------ */
static inline void rk4_rhs(double u, double w, double mass, double* ku, double* kw) {
    *ku = w;
    *kw = 3.0 * mass * u * u - u; /* oracles.hpp:19-21 */
}
void orc_rk4_step(double u, double w, double h, double mass, double out[2]) { /* oracles.hpp:23-30 */
    double k1u, k1w, k2u, k2w, k3u, k3w, k4u, k4w;
    rk4_rhs(u, w, mass, &k1u, &k1w);
    rk4_rhs(u + 0.5 * h * k1u, w + 0.5 * h * k1w, mass, &k2u, &k2w);
    rk4_rhs(u + 0.5 * h * k2u, w + 0.5 * h * k2w, mass, &k3u, &k3w);
    rk4_rhs(u + h * k3u, w + h * k3w, mass, &k4u, &k4w);
    out[0] = u + h / 6.0 * (k1u + 2.0 * k2u + 2.0 * k3u + k4u);
    out[1] = w + h / 6.0 * (k1w + 2.0 * k2w + 2.0 * k3w + k4w);
}
int orc_classify(double u, double w, double mass, double escape_radius, double phi_budget,
                 double h) { /* oracles.hpp:42-55 */
    const double u_capture = mass > 0.0 ? 1.0 / (2.0 * mass) : 1e300;
    const double u_escape = 1.0 / escape_radius;
    double phi = 0.0;
    while (phi < phi_budget) {
        if (u >= u_capture) return 0;
        if (u <= u_escape && w < 0.0) return 1;
        double o[2];
        orc_rk4_step(u, w, h, mass, o);
        u = o[0];
        w = o[1];
        phi += h;
    }
    return 2;
}

/* ------------------------------------------------------------------ */
/* RKF45 (no reference counterpart — control         */
/* structure after geodesic.cpp:104-160)                                */
/* ------------------------------------------------------------------ */
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

#define QMIN (-64)
#define QN 96
static double g_grow[QN], g_shrink[QN];
static pthread_once_t g_tables_once = PTHREAD_ONCE_INIT;
static void make_tables(void) {
    for (int i = 0; i < QN; ++i) {
        const int q = QMIN + i;
        const double f = 0.9 * pow(2.0, -(double)(q + 1) / 20.0);
        g_grow[i] = clampd(f, 0.2, 5.0);
        g_shrink[i] = clampd(f, 0.1, 0.9);
    }
}
void orc_rkf45_factor_tables(double* grow, double* shrink, int* qmin, int* n) {
    pthread_once(&g_tables_once, make_tables);
    if (grow) memcpy(grow, g_grow, sizeof g_grow);
    if (shrink) memcpy(shrink, g_shrink, sizeof g_shrink);
    if (qmin) *qmin = QMIN;
    if (n) *n = QN;
}

static inline int32_t hiword(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    return (int32_t)(b >> 32);
}

static inline double g_of(double U, double M3) { return U * fma(M3, U, -1.0); }

/* Returns 1 on accept. Operation order is normative (mirrored by the CUDA
 * kernel): every fma() below is one fused op, everything else separate. */
static int rkf45_step(double u, double w, double h, double M3, double rtol, double atol,
                      double hmax, double* un, double* wn, double* hn) {
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
    /* 5th-order solution (local extrapolation) */
    su = G1 * ku1; su = fma(G3, ku3, su); su = fma(G4, ku4, su); su = fma(G5, ku5, su);
    su = fma(G6, ku6, su);
    sw = G1 * kw1; sw = fma(G3, kw3, sw); sw = fma(G4, kw4, sw); sw = fma(G5, kw5, sw);
    sw = fma(G6, kw6, sw);
    const double u_new = fma(h, su, u), w_new = fma(h, sw, w);
    /* embedded error estimate (5th minus 4th) */
    su = H1 * ku1; su = fma(H3, ku3, su); su = fma(H4, ku4, su); su = fma(H5, ku5, su);
    su = fma(H6, ku6, su);
    sw = H1 * kw1; sw = fma(H3, kw3, sw); sw = fma(H4, kw4, sw); sw = fma(H5, kw5, sw);
    sw = fma(H6, kw6, sw);
    const double eu = fabs(h * su), ew = fabs(h * sw);
    /* max/min by compare-select (dmax/dmin: the first operand on NaN) */
    const double du = fma(rtol, dmax(fabs(u), fabs(u_new)), atol);
    const double dw = fma(rtol, dmax(fabs(w), fabs(w_new)), atol);
    /* error test, plus a geometric guard: one step may at most double r
     * (u_new >= u/2), so steps never overshoot past u = 0 on near-radial
     * outgoing rays (the reference's epsilon windows bound chords the same
     * way, geodesic.cpp:76-80). */
    const int err_ok = (eu <= du) && (ew <= dw);
    const int geo_ok = u_new >= 0.5 * u;
    const int accept = err_ok && geo_ok;
    /* Controller: q ~ floor(4*log2(E)) from the binary64 high words (Mitchell). */
    const int32_t du_ = hiword(eu) - hiword(du);
    const int32_t dw_ = hiword(ew) - hiword(dw);
    int32_t q = (du_ > dw_ ? du_ : dw_) >> 18;
    q = q < QMIN ? QMIN : (q > QMIN + QN - 1 ? QMIN + QN - 1 : q);
    if (accept) {
        *un = u_new;
        *wn = w_new;
        *hn = dmin(h * g_grow[q - QMIN], hmax);
    } else if (err_ok) {
        *hn = 0.5 * h;
    } else {
        *hn = h * g_shrink[q - QMIN];
    }
    return accept;
}

int orc_rkf45_step(double u, double w, double h, double mass, double rel_tol, double abs_tol,
                   double max_step, double out[2], double* hnext) {
    pthread_once(&g_tables_once, make_tables);
    out[0] = u;
    out[1] = w;
    return rkf45_step(u, w, h, 3.0 * mass, rel_tol, abs_tol, max_step, &out[0], &out[1], hnext);
}

/* ------------------------------------------------------------------ */
/* Scene modes: RK4 / RKF45 with disk + spheres     */
/* ------------------------------------------------------------------ */
#define MAXC 16

typedef struct {
    cam_t cam;
    double u_cap, u_esc, phi_max, M3;
    v3 light;
    v3 e1;     /* scene modes: normalized(camera - center), per frame */
    double u0; /* scene modes: 1 / |camera - center| */
    orc_table* table;  /* approximate mode: the b-table ... */
    double* psi0;      /* ... and each entry's inbound psi of the camera's u0 */
} prep_t;

static int prep_scene(const bhrt_scene* s, prep_t* p) {
    pthread_once(&g_tables_once, make_tables);
    const int st = cam_setup(s, &p->cam);
    if (st) return st;
    p->u_cap = s->mass > 0.0 ? 1.0 / (2.0 * s->mass) : INFINITY;
    p->u_esc = 1.0 / s->escape_radius;
    p->phi_max = 2.0 * PI * s->max_windings;
    p->M3 = 3.0 * s->mass;
    p->light = normalized(vld(s->light_dir));
    {   /* per-frame plane_basis / initial_conditions constants (geodesic.cpp:49-65) */
        const v3 v = sub(vld(s->cam_pos), vld(s->center));
        p->e1 = normalized(v);
        p->u0 = 1.0 / norm(v);
    }
    p->table = NULL;
    p->psi0 = NULL;
    return 0;
}

typedef struct {
    int k;             /* sphere index */
    double cx, cy, rho2;
    double lo, hi;     /* current angular window (unwrapped) */
} cand_t;

typedef struct {
    const bhrt_scene* s;
    v3 O, e1, e2, n;
    double next_disk;  /* +inf when no disk events */
    double disk_sigma; /* +1 / -1: which half of the disk line the next event is on */
    double disk_lx, disk_ly; /* unit disk line in plane coordinates */
    v3 disk_L;         /* unit disk line in world coordinates */
    int nc;            /* candidates (<= MAXC) or -1 = test all spheres every step */
    cand_t c[MAXC];
    double next_sph;
    /* result */
    int obj, sphere;
    v3 point;
} scene_ray_t;

static void sphere_window(double cx, double cy, double rho, double* lo, double* hi) {
    const double rc = sqrt(cx * cx + cy * cy);
    if (rc <= rho) { *lo = -INFINITY; *hi = INFINITY; return; }
    const double a = asin(rho / rc), pc = atan2(cy, cx);
    const double m = 1e-9; /* conservative culling margin; results never depend on it */
    *lo = pc - a - m;
    *hi = pc + a + m;
    if (*hi < 0.0) { *lo += 2.0 * PI; *hi += 2.0 * PI; }
}

/* atan2 for the disk-line angle of the scene modes: t =
 * min/max of |x|, |y| (one division), atan(t) = t + t s Q(s), s = t^2, with
 * Q a degree-19 Chebyshev fit (mpmath, |rel err| < 2.3e-16 on [0, 1])
 * evaluated by Estrin's scheme (8 dependent operations instead of 19 for
 * Horner), then the octant fix-up with two-part pi/2, pi. Normative op order
 * (oracle/bhrt_oracle.c atan2_est = device_common.cuh atan2_est). Finite
 * arguments, not both zero. */
static double atan2_est(double y, double x) {
    const double ax = fabs(x), ay = fabs(y);
    const double mx = ax < ay ? ay : ax, mn = ax < ay ? ax : ay;
    const double t = mn / mx;
    const double s = t * t, s2 = s * s, s4 = s2 * s2, s8 = s4 * s4, s16 = s8 * s8;
    const double b0 = fma(0x1.9999999999620p-3, s, -0x1.5555555555555p-2);
    const double b1 = fma(0x1.c71c71bb00a6cp-4, s, -0x1.24924924753ecp-3);
    const double b2 = fma(0x1.3b1399d1dcdc7p-4, s, -0x1.745d15ee35819p-4);
    const double b3 = fma(0x1.e1d0239d392a6p-5, s, -0x1.110fff599e4d2p-4);
    const double b4 = fma(0x1.841dcf603a209p-5, s, -0x1.aebbb1647a168p-5);
    const double b5 = fma(0x1.3328700bb8169p-5, s, -0x1.5d02278205cc7p-5);
    const double b6 = fma(0x1.843f4bca23369p-6, s, -0x1.00390504e9f2fp-5);
    const double b7 = fma(0x1.123baedb61abdp-7, s, -0x1.fd0e4de8fed90p-7);
    const double b8 = fma(0x1.1325b2f8964bep-10, s, -0x1.ca3677db66678p-9);
    const double b9 = fma(0x1.2f07811f9f6e9p-16, s, -0x1.a359b96a4eee4p-13);
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

static void ray_events_setup(scene_ray_t* R) {
    const bhrt_scene* s = R->s;
    R->next_disk = INFINITY;
    if (s->disk_enabled) {
        /* The disk plane (y = O.y) meets the orbital plane in the line
         * through O along L = n x (0,1,0); crossings are the phi-events
         * phi_L + k*pi. The hit direction alternates between +L^ and -L^. */
        /* L = n x (0,1,0) in plane coordinates: with n = e1 x e2 (unit,
         * orthonormal), L.e1 = -e2.y and L.e2 = e1.y exactly in real
         * arithmetic, so they are taken as such; |L|^2 = lx^2 + ly^2 and the
         * world line is lx e1 + ly e2. */
        const double lx = -R->e2.y, ly = R->e1.y;
        const double nl2 = lx * lx + ly * ly;
        if (nl2 >= 1e-24) { /* |L| >= 1e-12 */
            const double nl = sqrt(nl2);
            const double pl = atan2_est(ly, lx);
            R->next_disk = pl > 0.0 ? pl : pl + PI;
            R->disk_sigma = pl > 0.0 ? 1.0 : -1.0;
            /* one reciprocal for the unit line (plane and world coordinates) */
            const double inl = 1.0 / nl;
            R->disk_lx = lx * inl;
            R->disk_ly = ly * inl;
            R->disk_L = scl(add(scl(R->e1, lx), scl(R->e2, ly)), inl);
        }
    }
    R->nc = 0;
    R->next_sph = INFINITY;
    for (int k = 0; k < s->n_spheres; ++k) {
        const bhrt_sphere* sp = &s->spheres[k];
        const v3 c = sub(vld(sp->center), R->O);
        const double dn = dot(c, R->n);
        if (!(fabs(dn) < sp->radius)) continue;
        if (R->nc == MAXC) { R->nc = -1; break; }
        cand_t* cd = &R->c[R->nc++];
        cd->k = k;
        cd->cx = dot(c, R->e1);
        cd->cy = dot(c, R->e2);
        cd->rho2 = sp->radius * sp->radius - dn * dn;
        sphere_window(cd->cx, cd->cy, sqrt(cd->rho2), &cd->lo, &cd->hi);
    }
    if (R->nc < 0) { R->next_sph = -INFINITY; return; }
    for (int i = 0; i < R->nc; ++i) R->next_sph = dmin(R->next_sph, R->c[i].lo);
}

/* Cubic Hermite interpolation of u over one step, t in [0,1]. */
/* Monomial coefficients of the cubic Hermite interpolant of u over a step of
 * size h (u(0)=ua, u'(0)=h*wa, u(1)=ub, u'(1)=h*wb), normative op order. */
static inline void hermite_coef(double h, double ua, double wa, double ub, double wb, double a[4]) {
    a[0] = ua;
    a[1] = h * wa;
    a[2] = 3.0 * (ub - ua) - h * (2.0 * wa + wb);
    a[3] = 2.0 * (ua - ub) + h * (wa + wb);
}
static inline double hermite_eval(const double a[4], double t) {
    return fma(fma(fma(a[3], t, a[2]), t, a[1]), t, a[0]);
}
static inline double hermite_deval(const double a[4], double t) { /* d/dt */
    return fma(fma(3.0 * a[3], t, 2.0 * a[2]), t, a[1]);
}
static inline double hermite(double t, double h, double ua, double wa, double ub, double wb) {
    double a[4];
    hermite_coef(h, ua, wa, ub, wb, a);
    return hermite_eval(a, t);
}

/* Scene-mode ray setup (RK4 / RKF45 / TABLE; DESIGN.md §2 "Scene-mode ray
 * setup"): the orbital frame straight from the camera's unnormalised
 * direction D. e1 = (o - O)/|o - O| and u0 = 1/|o - O| are per-frame
 * (geodesic.cpp:49-65 with o = the camera); with c = D.e1 and T = D - c e1,
 * e2 = T / |T| (one reciprocal) and u0' = -(c / |T|) u0, which is the
 * reference's -(v.d)/(r0 b) with v = r0 e1, d = D/|D|, b = r0 |T| / |D|
 * (geodesic.cpp:57-65). The ray is radial iff |T|^2 < 1e-24 |D|^2 (the
 * reference's |tangential| < 1e-12 for unit d, geodesic.cpp:53); only then
 * is D normalised (radial_scene needs a unit direction). */
typedef struct {
    int ok;
    v3 e2;
    double w;
} frame_t;

static frame_t scene_frame(v3 e1, double u0, v3 D) {
    frame_t f;
    const double c = dot(D, e1);
    const v3 T = sub(D, scl(e1, c));
    const double t2 = dot(T, T);
    f.ok = !(t2 < 1e-24 * dot(D, D));
    f.e2 = mk(0.0, 0.0, 0.0);
    f.w = 0.0;
    if (!f.ok) return f;
    const double inv = 1.0 / sqrt(t2);
    f.e2 = scl(T, inv);
    f.w = -((c * inv) * u0);
    return f;
}

/* Hit tests over one accepted step (pa, ua, wa) -> (pb, ub, wb), DESIGN.md §Events.
 *  - disk: exact phi-event; radius from the step's cubic Hermite interpolant of u;
 *  - spheres: the step's polyline of S = ceil(h / chord_dphi) equal-angle
 *    sub-chords (vertices: Hermite u, directions by a rotation recurrence),
 *    first entering chord/circle intersection;
 *  - both in one step: the one at the smaller orbital angle wins.
 * Returns 1 on hit. */
static int step_events(scene_ray_t* R, double pa, double ua, double wa, double pb, double ub,
                       double wb) {
    const bhrt_scene* s = R->s;
    const double h = pb - pa;
    int hit = 0;
    /* ---- disk */
    int disk_hit = 0;
    double r_ev = 0.0, dlx = 0.0, dly = 0.0;
    if (R->next_disk > pa && R->next_disk <= pb) {
        const double t = (R->next_disk - pa) / h;
        const double u_ev = hermite(t, h, ua, wa, ub, wb);
        if (u_ev > 0.0) {
            r_ev = 1.0 / u_ev;
            if (r_ev >= s->disk_r_in && r_ev <= s->disk_r_out) {
                disk_hit = 1;
                dlx = R->disk_sigma * R->disk_lx;
                dly = R->disk_sigma * R->disk_ly;
            }
        }
    }
    /* ---- spheres */
    int act[MAXC];
    int na = 0;
    cand_t all;
    const int test_all = R->nc < 0;
    if (!test_all)
        for (int i = 0; i < R->nc; ++i)
            if (R->c[i].lo <= pb && R->c[i].hi >= pa) act[na++] = i;
    int sph_hit = 0, bsph = -1;
    double bqx = 0.0, bqy = 0.0;
    if (na > 0 || test_all) {
        int S = 1;
        if (h > s->chord_dphi) S = (int)ceil(h / s->chord_dphi);
        const double dl = h / S;
        const double cd_ = cos(dl), sd_ = sin(dl);
        double cj = cos(pa), sj = sin(pa);
        double rj = 1.0 / ua;
        double xj = cj * rj, yj = sj * rj;
        for (int j = 0; j < S && !sph_hit; ++j) {
            const double ck = cj * cd_ - sj * sd_;
            const double sk = sj * cd_ + cj * sd_;
            const double uk = (j + 1 == S) ? ub : hermite((double)(j + 1) / S, h, ua, wa, ub, wb);
            const double rk = 1.0 / uk;
            const double xk = ck * rk, yk = sk * rk;
            const double dx = xk - xj, dy = yk - yj;
            double best = INFINITY;
            const int ncand = test_all ? s->n_spheres : na;
            for (int a = 0; a < ncand; ++a) {
                const cand_t* cd;
                if (test_all) {
                    const bhrt_sphere* sp = &s->spheres[a];
                    const v3 c = sub(vld(sp->center), R->O);
                    const double dn = dot(c, R->n);
                    if (!(fabs(dn) < sp->radius)) continue;
                    all.k = a; all.cx = dot(c, R->e1); all.cy = dot(c, R->e2);
                    all.rho2 = sp->radius * sp->radius - dn * dn;
                    cd = &all;
                } else {
                    cd = &R->c[act[a]];
                }
                const double mx = xj - cd->cx, my = yj - cd->cy;
                const double A = dx * dx + dy * dy;
                const double B = mx * dx + my * dy;
                const double C = mx * mx + my * my - cd->rho2;
                if (!(C > 0.0)) continue;           /* entering hits only */
                const double disc = B * B - A * C;
                if (disc < 0.0) continue;
                const double t = (-B - sqrt(disc)) / A;
                if (t >= 0.0 && t <= 1.0 && t < best) {
                    best = t; sph_hit = 1; bsph = cd->k;
                    bqx = xj + t * dx; bqy = yj + t * dy;
                }
            }
            cj = ck; sj = sk; xj = xk; yj = yk;
        }
    }
    if (sph_hit && disk_hit) {
        /* sphere point at a smaller angle than the disk line <=> cross(p, l) > 0 */
        if (bqx * dly - bqy * dlx > 0.0) disk_hit = 0; else sph_hit = 0;
    }
    if (disk_hit) {
        hit = 1;
        R->obj = BHRT_OBJ_DISK;
        R->sphere = -1;
        R->point = add(R->O, scl(R->disk_L, R->disk_sigma * r_ev));
    } else if (sph_hit) {
        hit = 1;
        R->obj = BHRT_OBJ_SPHERE;
        R->sphere = bsph;
        R->point = add(R->O, add(scl(R->e1, bqx), scl(R->e2, bqy)));
    }
    /* advance event state past pb */
    while (R->next_disk <= pb) { R->next_disk += PI; R->disk_sigma = -R->disk_sigma; }
    if (!test_all) {
        R->next_sph = INFINITY;
        for (int i = 0; i < R->nc; ++i) {
            while (R->c[i].hi < pb) { R->c[i].lo += 2.0 * PI; R->c[i].hi += 2.0 * PI; }
            R->next_sph = dmin(R->next_sph, R->c[i].lo);
        }
    }
    return hit;
}

/* Unit tangent of the exact solution at (phi, u, w), world space. */
static v3 tangent_dir(const scene_ray_t* R, double phi, double u, double w) {
    const double c = cos(phi), sn = sin(phi);
    const double tx = -u * sn - w * c, ty = u * c - w * sn;
    return unit_fast(add(scl(R->e1, tx), scl(R->e2, ty)));
}

/* d/dt of hermite() (t in [0,1]); h01' = -h00'. */
static inline double hermite_d(double t, double h, double ua, double wa, double ub, double wb) {
    double a[4];
    hermite_coef(h, ua, wa, ub, wb, a);
    return hermite_deval(a, t);
}

/* Escape direction: the tangent where the trajectory
 * crosses r = escape_radius inside the last step, located on the step's
 * Hermite interpolant (linear guess + 2 Newton iterations), so the
 * direction does not depend on how far the last step overshot. Without a
 * crossing step (ray starts beyond the escape radius) it is the tangent at
 * the current state. */
static v3 escape_dir(const scene_ray_t* R, int has_step, double pa, double ua, double wa, double pb,
                     double ub, double wb, double u_esc, double energy, double M2) {
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
    /* u' from the first integral u'^2 = E - u^2 + 2Mu^3 (geodesic.cpp:272-275),
     * outgoing branch: more accurate than the interpolant's derivative. */
    const double q = energy - us * us + M2 * us * us * us;
    const double ws = -sqrt(q > 0.0 ? q : 0.0);
    return tangent_dir(R, pa + h * t, us, ws);
}

/* Radial ray in a scene: straight segment (geodesic.cpp:175-187) with hit tests. */
static void radial_scene(scene_ray_t* R, v3 origin, v3 dir, double seg_len, int captured) {
    const bhrt_scene* s = R->s;
    double best = seg_len;
    int obj = captured ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY, sph = -1;
    if (s->disk_enabled && dir.y != 0.0) {
        const double t = (R->O.y - origin.y) / dir.y;
        if (t >= 0.0 && t <= best) {
            const v3 q = sub(add(origin, scl(dir, t)), R->O);
            const double rq = sqrt(q.x * q.x + q.z * q.z);
            if (rq >= s->disk_r_in && rq <= s->disk_r_out) { best = t; obj = BHRT_OBJ_DISK; }
        }
    }
    for (int k = 0; k < s->n_spheres; ++k) {
        const bhrt_sphere* sp = &s->spheres[k];
        const v3 m = sub(origin, vld(sp->center));
        const double B = dot(m, dir), C = dot(m, m) - sp->radius * sp->radius;
        if (!(C > 0.0)) continue;
        const double disc = B * B - C;
        if (disc < 0.0) continue;
        const double t = -B - sqrt(disc);
        if (t >= 0.0 && t < best) { best = t; obj = BHRT_OBJ_SPHERE; sph = k; }
    }
    R->obj = obj;
    R->sphere = sph;
    R->point = (obj == BHRT_OBJ_SKY) ? dir : add(origin, scl(dir, best));
}

static int trace_scene(const bhrt_scene* s, const prep_t* P, v3 origin, v3 dir, bhrt_ray_record* rec,
                       scene_ray_t* R) {
    R->s = s;
    R->O = vld(s->center);
    R->obj = BHRT_OBJ_NONE;
    R->sphere = -1;
    rec->steps = 0;
    rec->rejected = 0;
    rec->phi = 0.0;
    const frame_t F = scene_frame(P->e1, P->u0, dir); /* dir: the raw camera direction */
    if (!F.ok) {
        const v3 ud = normalized(dir);
        const v3 v = sub(origin, R->O);
        const double r0 = norm(v);
        const int cap = dot(ud, sub(R->O, origin)) > 0.0;
        radial_scene(R, origin, ud, cap ? r0 - 2.0 * s->mass : s->escape_radius, cap);
        return 0;
    }
    R->e1 = P->e1;
    R->e2 = F.e2;
    R->n = cross(R->e1, R->e2);
    ray_events_setup(R);
    double phi = 0.0, u = P->u0, w = F.w;
    double pp = 0.0, up = 0.0, wp = 0.0; /* state before the last accepted step */
    int has_step = 0;
    const double M2 = 2.0 * s->mass;
    const double energy = w * w + u * u - M2 * u * u * u; /* conserved_energy, geodesic.cpp:272-275 */
    if (s->integrator == BHRT_INTEGRATOR_RK4) {
        const double h = s->step;
        for (;;) { /* oracles.hpp:47-54 loop structure */
            if (!(phi < P->phi_max)) { R->obj = BHRT_OBJ_STALLED; break; }
            if (u >= P->u_cap) { R->obj = BHRT_OBJ_HORIZON; break; }
            if (u <= P->u_esc && w < 0.0) {
                R->obj = BHRT_OBJ_SKY;
                R->point = escape_dir(R, has_step, pp, up, wp, phi, u, w, P->u_esc, energy, M2);
                break;
            }
            double nx[2];
            orc_rk4_step(u, w, h, s->mass, nx);
            const double pn = phi + h;
            rec->steps++;
            if (pn >= dmin(R->next_disk, R->next_sph) && step_events(R, phi, u, w, pn, nx[0], nx[1])) {
                phi = pn;
                break;
            }
            pp = phi; up = u; wp = w; has_step = 1;
            phi = pn; u = nx[0]; w = nx[1];
            if (!(u > 0.0)) return BHRT_NUMERICAL;
        }
    } else { /* RKF45 */
        double h = s->step;
        for (;;) { /* geodesic.cpp:199-236 loop structure */
            if (u >= P->u_cap) { R->obj = BHRT_OBJ_HORIZON; break; }
            if (u <= P->u_esc && w < 0.0) {
                R->obj = BHRT_OBJ_SKY;
                R->point = escape_dir(R, has_step, pp, up, wp, phi, u, w, P->u_esc, energy, M2);
                break;
            }
            if (phi > P->phi_max) { R->obj = BHRT_OBJ_STALLED; break; }
            double un, wn, hn;
            const int acc = rkf45_step(u, w, h, P->M3, s->rel_tol, s->abs_tol, s->max_step, &un, &wn, &hn);
            if (acc) {
                const double pn = phi + h;
                rec->steps++;
                if (pn >= dmin(R->next_disk, R->next_sph) && step_events(R, phi, u, w, pn, un, wn)) {
                    phi = pn;
                    break;
                }
                pp = phi; up = u; wp = w; has_step = 1;
                phi = pn; u = un; w = wn;
                if (!(u > 0.0)) return BHRT_NUMERICAL;
            } else {
                rec->rejected++;
            }
            h = hn;
            if (h < 1e-14) { /* StepSizeUnderflow, geodesic.cpp:156-157,224-231 */
                if (s->mass > 0.0 && u >= P->u_cap) { R->obj = BHRT_OBJ_HORIZON; break; }
                return BHRT_NUMERICAL;
            }
        }
    }
    rec->phi = phi;
    return 0;
}

/* ------------------------------------------------------------------ */
/* Approximate mode: b-table of inbound orbits      */
/* ------------------------------------------------------------------ */
struct orc_table {
    int entries, ns;
    double b_max, dpsi, u_cap, u_esc;
    int* kind;
    int* n;
    double* ends; /* psi_end, u_end, w_end, psi_esc */
    double* smp;  /* entries * ns * 2 */
};

static inline double hermite_ddeval(const double a[4], double t) { return fma(6.0 * a[3], t, 2.0 * a[2]); }

/* Newton on H(t) = target (or H'(t) = 0 when deriv) from t0, 3 iterations, clamped. */
static double cubic_solve(const double a[4], double t, double target, int deriv) {
    for (int it = 0; it < 3; ++it) {
        const double f = deriv ? hermite_deval(a, t) : hermite_eval(a, t) - target;
        const double df = deriv ? hermite_ddeval(a, t) : hermite_deval(a, t);
        if (df != 0.0) t = t - f / df;
        t = clampd(t, 0.0, 1.0);
    }
    return t;
}

static void table_entry_build(const bhrt_scene* s, orc_table* T, int e) {
    const double b = T->b_max * e / (T->entries - 1);
    double* S = T->smp + (size_t)e * T->ns * 2;
    double* E = T->ends + 4 * (size_t)e;
    if (!(b > 0.0)) {
        T->kind[e] = 3;
        T->n[e] = 0;
        E[0] = E[1] = E[2] = 0.0;
        E[3] = -1.0;
        return;
    }
    const double M3 = 3.0 * s->mass;
    double u = 0.0, w = 1.0 / b, psi = 0.0, h = s->step;
    S[0] = u;
    S[1] = w;
    int cnt = 1, kind = 2;
    for (;;) {
        if (cnt >= T->ns) { E[0] = psi; E[1] = u; E[2] = w; break; }
        const double target = (double)cnt * T->dpsi;
        int done = 0;
        while (psi < target) {
            const double rem = target - psi;
            const int last = !(h < rem);
            const double ht = last ? rem : h;
            double un, wn, hn;
            const int acc = rkf45_step(u, w, ht, M3, s->rel_tol, s->abs_tol, s->max_step, &un, &wn, &hn);
            if (acc) {
                if (un >= T->u_cap || wn <= 0.0) {
                    double a[4];
                    hermite_coef(ht, u, w, un, wn, a);
                    if (un >= T->u_cap) { /* capture inside this step */
                        const double t = cubic_solve(a, (T->u_cap - u) / (un - u), T->u_cap, 0);
                        E[0] = psi + ht * t; E[1] = T->u_cap; E[2] = hermite_deval(a, t) / ht;
                        kind = 0;
                    } else { /* periapsis u' = 0 inside this step */
                        const double t = cubic_solve(a, w / (w - wn), 0.0, 1);
                        E[0] = psi + ht * t; E[1] = hermite_eval(a, t); E[2] = 0.0;
                        kind = 1;
                    }
                    done = 1;
                    break;
                }
                psi = last ? target : psi + ht;
                u = un;
                w = wn;
            }
            h = hn;
            if (h < 1e-14) { E[0] = psi; E[1] = u; E[2] = w; done = 1; break; }
        }
        if (done) break;
        S[2 * cnt] = u;
        S[2 * cnt + 1] = w;
        ++cnt;
    }
    T->kind[e] = kind;
    T->n[e] = cnt;
    E[3] = -1.0;
    E[3] = orc_table_inbound_psi(T, e, T->u_esc);
}

double orc_table_inbound_psi(const orc_table* T, int e, double target) {
    const int kind = T->kind[e], n = T->n[e];
    if (kind == 3 || n < 1) return -1.0;
    const double* S = T->smp + (size_t)e * T->ns * 2;
    const double* E = T->ends + 4 * (size_t)e;
    if (!(target > S[0])) return 0.0;
    int j;
    double h, ua, wa, ub, wb;
    if (!(S[2 * (n - 1)] > target)) { /* at or beyond the last sample: end segment */
        if (kind == 2 || E[1] < target) return -1.0;
        j = n - 1;
        h = E[0] - (double)j * T->dpsi;
        ua = S[2 * j]; wa = S[2 * j + 1]; ub = E[1]; wb = E[2];
        if (!(h > 0.0)) return E[0];
    } else {
        int lo = 0, hi = n - 1; /* u(lo) <= target < u(hi) */
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (S[2 * mid] <= target) lo = mid; else hi = mid;
        }
        j = lo;
        h = T->dpsi;
        ua = S[2 * j]; wa = S[2 * j + 1]; ub = S[2 * j + 2]; wb = S[2 * j + 3];
    }
    double a[4];
    hermite_coef(h, ua, wa, ub, wb, a);
    const double t0 = ub > ua ? (target - ua) / (ub - ua) : 0.0;
    const double t = cubic_solve(a, t0, target, 0);
    return (double)j * T->dpsi + h * t;
}

/* u on entry e at orbit angle psi (mirror beyond periapsis); -1 if undefined. */
static double table_u(const orc_table* T, int e, double psi) {
    const int kind = T->kind[e], n = T->n[e];
    const double* S = T->smp + (size_t)e * T->ns * 2;
    const double* E = T->ends + 4 * (size_t)e;
    if (kind == 1 && psi > E[0]) psi = 2.0 * E[0] - psi;
    if (psi < 0.0 || n < 1) return -1.0;
    int j = (int)floor(psi / T->dpsi);
    double h, ua, wa, ub, wb, pa;
    if (j >= n - 1) {
        if (kind == 2 || psi > E[0]) return -1.0;
        j = n - 1;
        pa = (double)j * T->dpsi;
        h = E[0] - pa;
        if (!(h > 0.0)) return E[1];
        ua = S[2 * j]; wa = S[2 * j + 1]; ub = E[1]; wb = E[2];
    } else {
        pa = (double)j * T->dpsi;
        h = T->dpsi;
        ua = S[2 * j]; wa = S[2 * j + 1]; ub = S[2 * j + 2]; wb = S[2 * j + 3];
    }
    double a[4];
    hermite_coef(h, ua, wa, ub, wb, a);
    return hermite_eval(a, (psi - pa) / h);
}

orc_table* orc_table_build(const bhrt_scene* s) {
    pthread_once(&g_tables_once, make_tables);
    if (s->table_entries < 2 || s->table_samples < 2 || !(s->table_b_max > 0.0) || !(s->table_dpsi > 0.0))
        return NULL;
    orc_table* T = (orc_table*)calloc(1, sizeof *T);
    T->entries = s->table_entries;
    T->ns = s->table_samples;
    T->b_max = s->table_b_max;
    T->dpsi = s->table_dpsi;
    T->u_cap = s->mass > 0.0 ? 1.0 / (2.0 * s->mass) : INFINITY;
    T->u_esc = 1.0 / s->escape_radius;
    T->kind = (int*)calloc((size_t)T->entries, sizeof(int));
    T->n = (int*)calloc((size_t)T->entries, sizeof(int));
    T->ends = (double*)calloc((size_t)T->entries * 4, sizeof(double));
    T->smp = (double*)calloc((size_t)T->entries * T->ns * 2, sizeof(double));
    for (int e = 0; e < T->entries; ++e) table_entry_build(s, T, e);
    return T;
}

void orc_table_free(orc_table* T) {
    if (!T) return;
    free(T->kind); free(T->n); free(T->ends); free(T->smp); free(T);
}

int orc_table_entry(const orc_table* T, int e, int* kind, int* n, double ends[4], double* samples, int cap) {
    if (!T || e < 0 || e >= T->entries) return BHRT_INVALID_ARGUMENT;
    *kind = T->kind[e];
    *n = T->n[e];
    memcpy(ends, T->ends + 4 * (size_t)e, 4 * sizeof(double));
    const int m = T->n[e] < cap ? T->n[e] : cap;
    if (samples) memcpy(samples, T->smp + (size_t)e * T->ns * 2, 2 * sizeof(double) * (size_t)m);
    return 0;
}

/* One entry's plan for a ray with camera-side inbound position psi0. */
static int table_plan(const orc_table* T, int e, double psi0, double w0, int* outcome, double* phi_end) {
    const int kind = T->kind[e];
    const double* E = T->ends + 4 * (size_t)e;
    if (kind == 3 || psi0 < 0.0) return 0;
    if (w0 >= 0.0) { /* moving inward along the orbit */
        if (kind == 0) { *outcome = BHRT_OBJ_HORIZON; *phi_end = E[0] - psi0; return 1; }
        if (kind == 2) { *outcome = BHRT_OBJ_STALLED; *phi_end = INFINITY; return 1; }
        if (E[3] < 0.0) return 0;
        *outcome = BHRT_OBJ_SKY;
        *phi_end = (2.0 * E[0] - E[3]) - psi0;
        return 1;
    }
    if (E[3] < 0.0) return 0; /* moving outward: straight back out along the inbound branch */
    *outcome = BHRT_OBJ_SKY;
    *phi_end = psi0 - E[3];
    return 1;
}

static int trace_table(const bhrt_scene* s, const prep_t* P, v3 origin, v3 dir, bhrt_ray_record* rec,
                       scene_ray_t* R) {
    const orc_table* T = P->table;
    R->s = s;
    R->O = vld(s->center);
    R->obj = BHRT_OBJ_NONE;
    R->sphere = -1;
    rec->steps = 0;
    rec->rejected = 0;
    rec->phi = 0.0;
    const frame_t F = scene_frame(P->e1, P->u0, dir); /* dir: the raw camera direction */
    if (!F.ok) {
        const v3 ud = normalized(dir);
        const double r0 = norm(sub(origin, R->O));
        const int cap = dot(ud, sub(R->O, origin)) > 0.0;
        radial_scene(R, origin, ud, cap ? r0 - 2.0 * s->mass : s->escape_radius, cap);
        return 0;
    }
    R->e1 = P->e1;
    R->e2 = F.e2;
    R->n = cross(R->e1, R->e2);
    const double u0 = P->u0, w0 = F.w;
    const double M2 = 2.0 * s->mass;
    const double energy = w0 * w0 + u0 * u0 - M2 * u0 * u0 * u0;
    /* The orbit's impact parameter is fixed by its first integral
     * u'^2 + u^2 - 2Mu^3 = 1/b^2 (geodesic.cpp:272-275), not by |v x d|: the
     * initial conditions (geodesic.cpp:57-65) are flat-space ones. */
    if (!(energy > 0.0)) { R->obj = BHRT_OBJ_STALLED; return 0; } /* never reaches infinity */
    const double b = 1.0 / sqrt(energy);
    ray_events_setup(R);
    const int N = T->entries;
    const double x = (b * (double)(N - 1)) / T->b_max;
    int i = (int)floor(x);
    if (i > N - 2) i = N - 2;
    double f = x - (double)i;
    if (T->kind[i] == 3) f = 1.0;
    int oi = 0, oj = 0;
    double pi_ = 0.0, pj = 0.0;
    const int vi = table_plan(T, i, P->psi0[i], w0, &oi, &pi_);
    const int vj = table_plan(T, i + 1, P->psi0[i + 1], w0, &oj, &pj);
    int outcome;
    double phi_end, wi, wj;
    if (vi && vj && oi == oj && f > 0.0 && f < 1.0) {
        outcome = oi;
        phi_end = outcome == BHRT_OBJ_STALLED ? INFINITY : (1.0 - f) * pi_ + f * pj;
        wi = 1.0 - f;
        wj = f;
    } else {
        int use_j = f >= 0.5;
        if (use_j && !vj) use_j = 0;
        if (!use_j && !vi) use_j = 1;
        if (use_j ? !vj : !vi) { R->obj = BHRT_OBJ_STALLED; return 0; }
        outcome = use_j ? oj : oi;
        phi_end = use_j ? pj : pi_;
        wi = use_j ? 0.0 : 1.0;
        wj = use_j ? 1.0 : 0.0;
    }
    if (phi_end > P->phi_max) outcome = BHRT_OBJ_STALLED;
    const double stop = outcome == BHRT_OBJ_STALLED ? P->phi_max : phi_end;
    const double sgn = w0 >= 0.0 ? 1.0 : -1.0;
    while (R->next_disk < stop) { /* disk events along the interpolated orbit */
        const double ph = R->next_disk;
        double ui = -1.0, uj = -1.0;
        if (wi > 0.0) ui = table_u(T, i, P->psi0[i] + sgn * ph);
        if (wj > 0.0) uj = table_u(T, i + 1, P->psi0[i + 1] + sgn * ph);
        double u_ev;
        if (wi > 0.0 && wj > 0.0 && ui >= 0.0 && uj >= 0.0) u_ev = wi * ui + wj * uj;
        else u_ev = ui >= 0.0 ? ui : uj;
        if (u_ev > 0.0) {
            const double r_ev = 1.0 / u_ev;
            if (r_ev >= s->disk_r_in && r_ev <= s->disk_r_out) {
                R->obj = BHRT_OBJ_DISK;
                R->point = add(R->O, scl(R->disk_L, R->disk_sigma * r_ev));
                rec->phi = ph;
                return 0;
            }
        }
        R->next_disk += PI;
        R->disk_sigma = -R->disk_sigma;
    }
    R->obj = outcome;
    rec->phi = outcome == BHRT_OBJ_STALLED ? P->phi_max : phi_end;
    if (outcome == BHRT_OBJ_SKY) {
        const double ue = P->u_esc;
        const double q = energy - ue * ue + M2 * ue * ue * ue;
        R->point = tangent_dir(R, phi_end, ue, -sqrt(q > 0.0 ? q : 0.0));
    }
    return 0;
}

static void shade_object(const bhrt_scene* s, const prep_t* P, const scene_ray_t* R, double rgb[3]) {
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    switch (R->obj) {
        case BHRT_OBJ_SKY: sky(s, R->point, rgb); break;
        case BHRT_OBJ_DISK: {
            const v3 q = sub(R->point, R->O);
            const double r = sqrt(q.x * q.x + q.z * q.z);
            /* the ramp scale is one reciprocal per scene (the kernels take it from the host) */
            const double t = (r - s->disk_r_in) * (1.0 / (s->disk_r_out - s->disk_r_in));
            for (int c = 0; c < 3; ++c)
                rgb[c] = s->disk_color_in[c] + t * (s->disk_color_out[c] - s->disk_color_in[c]);
            break;
        }
        case BHRT_OBJ_SPHERE: {
            const bhrt_sphere* sp = &s->spheres[R->sphere];
            const v3 nrm = scl(sub(R->point, vld(sp->center)), 1.0 / sp->radius);
            const double lam = dmax(0.0, dot(nrm, P->light));
            const double k = s->ambient + (1.0 - s->ambient) * lam;
            for (int c = 0; c < 3; ++c) rgb[c] = sp->albedo[c] * k;
            break;
        }
        default: break;
    }
}

static int trace_sample_prepared(const bhrt_scene* s, const prep_t* P, int px, int py, int sample,
                                 bhrt_ray_record* rec, double rgb[3]) {
    const v3 origin = vld(s->cam_pos);
    /* mode R: the reference's unit ray; scene modes: the raw direction (scene_frame) */
    const v3 dir = s->integrator == BHRT_INTEGRATOR_REFERENCE ? cam_ray(s, &P->cam, px, py, sample)
                                                              : cam_dir_raw(s, &P->cam, px, py, sample);
    rec->sphere = -1;
    rec->point[0] = rec->point[1] = rec->point[2] = 0.0;
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    if (s->integrator == BHRT_INTEGRATOR_REFERENCE) {
        int kind, np, ns = 0, nr = 0;
        double dout[3], l2[6];
        const double o[3] = {origin.x, origin.y, origin.z}, d[3] = {dir.x, dir.y, dir.z};
        const int rc = orc_trace_reference(o, d, s->mass, s->center, s->epsilon, s->escape_radius,
                                           s->max_windings, s->rel_tol, s->abs_tol, &kind, dout, &np,
                                           l2, &ns, &nr);
        rec->steps = ns;
        rec->rejected = nr;
        rec->phi = 0.0;
        if (rc) return rc;
        rec->object = kind == 0 ? BHRT_OBJ_HORIZON : (kind == 1 ? BHRT_OBJ_SKY : BHRT_OBJ_STALLED);
        if (kind == 1) {
            memcpy(rec->point, dout, sizeof dout);
            orc_sample_direction(s->sky_rgb, s->sky_width, s->sky_height, dout, rgb);
        }
        return 0;
    }
    scene_ray_t R;
    const int rc = s->integrator == BHRT_INTEGRATOR_TABLE ? trace_table(s, P, origin, dir, rec, &R)
                                                          : trace_scene(s, P, origin, dir, rec, &R);
    if (rc) return rc;
    rec->object = R.obj;
    rec->sphere = R.sphere;
    if (R.obj == BHRT_OBJ_SKY || R.obj == BHRT_OBJ_DISK || R.obj == BHRT_OBJ_SPHERE)
        vst(rec->point, R.point);
    shade_object(s, P, &R, rgb);
    return 0;
}

/* The b-table depends only on these scene fields; the last one built is cached. */
static pthread_mutex_t g_table_mu = PTHREAD_MUTEX_INITIALIZER;
static orc_table* g_table = NULL;
static double g_table_key[10];

static int prep_table(const bhrt_scene* s, prep_t* P) {
    if (s->integrator != BHRT_INTEGRATOR_TABLE) return 0;
    const double key[10] = {s->mass, s->rel_tol, s->abs_tol, s->step, s->max_step,
                            (double)s->table_entries, (double)s->table_samples, s->table_b_max,
                            s->table_dpsi, s->escape_radius};
    pthread_mutex_lock(&g_table_mu);
    if (!g_table || memcmp(key, g_table_key, sizeof key) != 0) {
        orc_table_free(g_table);
        g_table = orc_table_build(s);
        memcpy(g_table_key, key, sizeof key);
    }
    P->table = g_table;
    pthread_mutex_unlock(&g_table_mu);
    if (!P->table) return BHRT_INVALID_ARGUMENT;
    /* bind the camera radius: each entry's inbound psi of u0 = 1/|cam - O| */
    const double u0 = 1.0 / norm(sub(vld(s->cam_pos), vld(s->center)));
    P->psi0 = (double*)malloc(sizeof(double) * (size_t)P->table->entries);
    for (int e = 0; e < P->table->entries; ++e) P->psi0[e] = orc_table_inbound_psi(P->table, e, u0);
    return 0;
}

static void prep_release(prep_t* P) {
    free(P->psi0);
    P->psi0 = NULL;
}

int orc_trace_sample(const bhrt_scene* s, int px, int py, int sample, bhrt_ray_record* rec,
                     double rgb[3]) {
    prep_t P;
    int st = prep_scene(s, &P);
    if (st) return st;
    st = prep_table(s, &P);
    if (st) return st;
    st = trace_sample_prepared(s, &P, px, py, sample, rec, rgb);
    prep_release(&P);
    return st;
}

static int shade_prepared(const bhrt_scene* s, const prep_t* P, int px, int py, uint8_t out[3],
                          bhrt_ray_record* recs) { /* render.cpp:22-49 */
    double acc[3] = {0.0, 0.0, 0.0};
    for (int sidx = 0; sidx < s->spp; ++sidx) {
        bhrt_ray_record tmp;
        bhrt_ray_record* rec = recs ? &recs[sidx] : &tmp;
        double c[3];
        const int rc = trace_sample_prepared(s, P, px, py, sidx, rec, c);
        if (rc) return rc;
        acc[0] += c[0];
        acc[1] += c[1];
        acc[2] += c[2];
    }
    const double inv = 1.0 / s->spp;
    for (int c = 0; c < 3; ++c) {
        const double scaled = round(acc[c] * inv * 255.0);
        out[c] = (uint8_t)clampd(scaled, 0.0, 255.0);
    }
    return 0;
}

int orc_shade_pixel(const bhrt_scene* s, int px, int py, uint8_t out[3], bhrt_ray_record* recs) {
    prep_t P;
    int st = prep_scene(s, &P);
    if (st) return st;
    st = prep_table(s, &P);
    if (st) return st;
    st = shade_prepared(s, &P, px, py, out, recs);
    prep_release(&P);
    return st;
}

void orc_scene_defaults(bhrt_scene* s) {
    memset(s, 0, sizeof *s);
    s->mass = 1.0;
    s->cam_pos[2] = -20.0;
    s->vertical_fov = 60.0 * PI / 180.0;
    s->width = 256;
    s->height = 256;
    s->spp = 1;
    s->max_windings = 10;
    s->seed = 1;
    s->epsilon = 0.05;
    s->escape_radius = 1e4;
    s->rel_tol = 1e-10;
    s->abs_tol = 1e-12;
    s->integrator = BHRT_INTEGRATOR_REFERENCE;
    s->sky_kind = BHRT_SKY_IMAGE;
    s->step = 1e-2;
    s->max_step = 0.1;
    s->chord_dphi = 0.01;
    s->checker_nu = 16;
    s->checker_nv = 8;
    s->checker_color_a[0] = 0.9; s->checker_color_a[1] = 0.9; s->checker_color_a[2] = 0.9;
    s->checker_color_b[0] = 0.1; s->checker_color_b[1] = 0.1; s->checker_color_b[2] = 0.15;
    s->disk_r_in = 6.0;
    s->disk_r_out = 20.0;
    s->disk_color_in[0] = 1.0; s->disk_color_in[1] = 0.95; s->disk_color_in[2] = 0.8;
    s->disk_color_out[0] = 0.8; s->disk_color_out[1] = 0.25; s->disk_color_out[2] = 0.05;
    s->light_dir[0] = 0.5; s->light_dir[1] = 1.0; s->light_dir[2] = -1.0;
    s->ambient = 0.1;
    s->table_entries = 100000;
    s->table_samples = 2048;
    s->table_b_max = 50.0;
    s->table_dpsi = 0.01;
}

static void set_info(bhrt_status_info* info, int code, int px, int py, const char* msg) {
    if (!info) return;
    info->code = code;
    info->px = px;
    info->py = py;
    snprintf(info->message, sizeof info->message, "%s", msg);
}

int orc_validate_scene(const bhrt_scene* s, bhrt_status_info* info) { /* render.cpp:11-20 */
    if (s->sky_kind == BHRT_SKY_IMAGE && (s->sky_rgb == NULL || s->sky_width < 1 || s->sky_height < 1)) {
        set_info(info, BHRT_USAGE, -1, -1, "scene: background image is required");
        return BHRT_USAGE;
    }
    if (s->width < 1 || s->height < 1) {
        set_info(info, BHRT_USAGE, -1, -1, "scene: image dimensions must be >= 1");
        return BHRT_USAGE;
    }
    if (s->spp < 1) { set_info(info, BHRT_USAGE, -1, -1, "scene: spp must be >= 1"); return BHRT_USAGE; }
    if (s->mass < 0.0) { set_info(info, BHRT_USAGE, -1, -1, "scene: mass must be >= 0"); return BHRT_USAGE; }
    const double d = norm(sub(vld(s->cam_pos), vld(s->center)));
    if (d <= 2.0 * s->mass) {
        set_info(info, BHRT_USAGE, -1, -1, "scene: camera must be outside the event horizon");
        return BHRT_USAGE;
    }
    return 0;
}

/* Trace-level validation the reference performs per ray (geodesic.cpp:19-27, camera.cpp:30-43). */
static int validate_trace(const bhrt_scene* s, bhrt_status_info* info) {
    if (!(s->epsilon > 0.0) || !(s->escape_radius > 0.0) || s->max_windings < 1 ||
        !(s->rel_tol > 0.0) || !(s->abs_tol > 0.0)) {
        set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: invalid parameter");
        return BHRT_INVALID_ARGUMENT;
    }
    if (s->integrator < 0 || s->integrator > BHRT_INTEGRATOR_TABLE ||
        (s->integrator != BHRT_INTEGRATOR_REFERENCE && !(s->step > 0.0)) ||
        (s->integrator == BHRT_INTEGRATOR_RKF45 && !(s->max_step > 0.0 && s->max_step < 1.0)) ||
        (s->integrator == BHRT_INTEGRATOR_REFERENCE && (s->disk_enabled || s->n_spheres > 0)) ||
        (s->integrator == BHRT_INTEGRATOR_TABLE &&
         (s->n_spheres > 0 || s->table_entries < 2 || s->table_samples < 2 || !(s->table_b_max > 0.0) ||
          !(s->table_dpsi > 0.0) || !(s->max_step > 0.0 && s->max_step < 1.0))) ||
        !(s->chord_dphi > 0.0) || (s->n_spheres > 0 && s->spheres == NULL) ||
        (s->sky_kind == BHRT_SKY_CHECKER && (s->checker_nu < 1 || s->checker_nv < 1))) {
        set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "scene extension: invalid parameter");
        return BHRT_INVALID_ARGUMENT;
    }
    double f[3], r[3], u[3];
    if (orc_camera_basis(s, f, r, u)) {
        set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "camera: degenerate orientation");
        return BHRT_INVALID_ARGUMENT;
    }
    return 0;
}

int orc_make_bands(int height, int workers, int* rs, int* re, int capacity, int* count) {
    if (height < 1 || workers < 1) return BHRT_INVALID_ARGUMENT; /* render.cpp:51-66 */
    const int n = height < workers ? height : workers;
    if (capacity < n) return BHRT_INVALID_ARGUMENT;
    const int base = height / n, extra = height % n;
    int row = 0;
    for (int i = 0; i < n; ++i) {
        const int rows = base + (i < extra ? 1 : 0);
        rs[i] = row;
        re[i] = row + rows;
        row += rows;
    }
    *count = n;
    return 0;
}

typedef struct {
    const bhrt_scene* s;
    const prep_t* P;
    int row_start, row_end;
    uint8_t* out;
    bhrt_ray_record* recs;
    int next;
    pthread_mutex_t mu;
    int fail_code, fail_px, fail_py; /* lowest failing (py, px) */
} job_t;

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    const int W = J->s->width;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int y = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (y >= J->row_end) return NULL;
        uint8_t* row = J->out + 3 * (size_t)(y - J->row_start) * W;
        for (int x = 0; x < W; ++x) {
            bhrt_ray_record* rr =
                J->recs ? J->recs + ((size_t)(y - J->row_start) * W + x) * J->s->spp : NULL;
            const int rc = shade_prepared(J->s, J->P, x, y, row + 3 * x, rr);
            if (rc) {
                pthread_mutex_lock(&J->mu);
                if (!J->fail_code || y < J->fail_py || (y == J->fail_py && x < J->fail_px)) {
                    J->fail_code = rc; J->fail_px = x; J->fail_py = y;
                }
                pthread_mutex_unlock(&J->mu);
                break; /* rest of this row is irrelevant: a lower pixel already failed */
            }
        }
    }
}

int orc_render_rows(const bhrt_scene* s, int row_start, int row_end, int threads, uint8_t* out,
                    bhrt_ray_record* records, bhrt_status_info* info) { /* render.cpp:68-119 */
    if (info) set_info(info, 0, -1, -1, "");
    int rc = orc_validate_scene(s, info);
    if (rc) return rc;
    if (threads < 1) { set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: threads must be >= 1"); return BHRT_INVALID_ARGUMENT; }
    if (row_start < 0 || row_end > s->height || row_start > row_end) {
        set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: row range out of bounds");
        return BHRT_INVALID_ARGUMENT;
    }
    if (row_end == row_start) return 0;
    rc = validate_trace(s, info);
    if (rc) return rc;
    prep_t P;
    prep_scene(s, &P);
    rc = prep_table(s, &P);
    if (rc) {
        set_info(info, rc, -1, -1, "table: invalid parameters");
        return rc;
    }
    job_t J = {s, &P, row_start, row_end, out, records, row_start, PTHREAD_MUTEX_INITIALIZER, 0, 0, 0};
    const int rows = row_end - row_start;
    const int pool = threads < rows ? threads : rows;
    if (pool == 1) {
        worker(&J);
    } else {
        pthread_t* ts = (pthread_t*)malloc(sizeof(pthread_t) * pool);
        for (int i = 0; i < pool; ++i) pthread_create(&ts[i], NULL, worker, &J);
        for (int i = 0; i < pool; ++i) pthread_join(ts[i], NULL);
        free(ts);
    }
    prep_release(&P);
    if (J.fail_code) {
        char msg[128];
        snprintf(msg, sizeof msg, "pixel (%d, %d): numerical failure", J.fail_px, J.fail_py);
        set_info(info, J.fail_code, J.fail_px, J.fail_py, msg);
        return J.fail_code;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Sphere field                                     */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t x; } sm_t;
static uint64_t sm_next(sm_t* g) {
    uint64_t z = (g->x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static double sm_unit(sm_t* g) { return (double)(sm_next(g) >> 11) * 0x1.0p-53; }

int orc_make_spheres(uint64_t seed, int n, const double center[3], double shell_min,
                     double shell_max, double radius_min, double radius_max, bhrt_sphere* out) {
    if (n < 0 || !(shell_min >= 0.0) || !(shell_max >= shell_min) || !(radius_min > 0.0) ||
        !(radius_max >= radius_min))
        return BHRT_INVALID_ARGUMENT;
    sm_t g = {seed};
    const double lo3 = shell_min * shell_min * shell_min;
    const double hi3 = shell_max * shell_max * shell_max;
    for (int i = 0; i < n; ++i) {
        const double cz = 2.0 * sm_unit(&g) - 1.0;
        const double th = 2.0 * PI * sm_unit(&g);
        const double rr = cbrt(lo3 + sm_unit(&g) * (hi3 - lo3));
        const double sxy = sqrt(1.0 - cz * cz);
        out[i].center[0] = center[0] + rr * (sxy * cos(th));
        out[i].center[1] = center[1] + rr * cz;
        out[i].center[2] = center[2] + rr * (sxy * sin(th));
        out[i].radius = radius_min + sm_unit(&g) * (radius_max - radius_min);
        out[i].albedo[0] = sm_unit(&g);
        out[i].albedo[1] = sm_unit(&g);
        out[i].albedo[2] = sm_unit(&g);
    }
    return 0;
}
