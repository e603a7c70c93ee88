// trace_reference.cu — mode R: the reference algorithm on the GPU.
//
// DOPRI5(4)+PI control inside epsilon-windows, window-end termination tests
// and last-chord escape direction, exactly as geodesic.cpp:84-238, one
// sample per thread. Compiled with --fmad=false (like the reference's x86-64
// build) and glibc's hypot restated, so window states are bit-identical to
// the reference; only pow() (step-hint only) and sin/cos (last chord) may
// differ by ulps (libdevice vs glibc).
// Shading out of line here too (1080p sky-only: 95.8 -> 95.2 ms).
#ifndef BHRT_INL_SHADE
#define BHRT_INL_SHADE __noinline__
#endif
#include "device_common.cuh"

namespace bhrt_b200 {

// ================================================================= mode R
// Dormand-Prince 5(4) tableau (geodesic.cpp:89-100), same constant expressions,
// in the constant bank: as literals every use was rematerialised by two UMOVs
// inside the window loop (64 per step); DMUL takes a constant-bank operand.
#ifndef BHRT_DOPRI_LITERALS
static __constant__ double kDopri[26] = {
    1.0 / 5.0,  // A21
    3.0 / 40.0,  // A31
    9.0 / 40.0,  // A32
    44.0 / 45.0,  // A41
    -56.0 / 15.0,  // A42
    32.0 / 9.0,  // A43
    19372.0 / 6561.0,  // A51
    -25360.0 / 2187.0,  // A52
    64448.0 / 6561.0,  // A53
    -212.0 / 729.0,  // A54
    9017.0 / 3168.0,  // A61
    -355.0 / 33.0,  // A62
    46732.0 / 5247.0,  // A63
    49.0 / 176.0,  // A64
    -5103.0 / 18656.0,  // A65
    35.0 / 384.0,  // B1
    500.0 / 1113.0,  // B3
    125.0 / 192.0,  // B4
    -2187.0 / 6784.0,  // B5
    11.0 / 84.0,  // B6
    71.0 / 57600.0,  // E1
    -71.0 / 16695.0,  // E3
    71.0 / 1920.0,  // E4
    -17253.0 / 339200.0,  // E5
    22.0 / 525.0,  // E6
    -1.0 / 40.0,  // E7
};
#define A21 (kDopri[0])
#define A31 (kDopri[1])
#define A32 (kDopri[2])
#define A41 (kDopri[3])
#define A42 (kDopri[4])
#define A43 (kDopri[5])
#define A51 (kDopri[6])
#define A52 (kDopri[7])
#define A53 (kDopri[8])
#define A54 (kDopri[9])
#define A61 (kDopri[10])
#define A62 (kDopri[11])
#define A63 (kDopri[12])
#define A64 (kDopri[13])
#define A65 (kDopri[14])
#define B1 (kDopri[15])
#define B3 (kDopri[16])
#define B4 (kDopri[17])
#define B5 (kDopri[18])
#define B6 (kDopri[19])
#define E1 (kDopri[20])
#define E3 (kDopri[21])
#define E4 (kDopri[22])
#define E5 (kDopri[23])
#define E6 (kDopri[24])
#define E7 (kDopri[25])
#else
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
#endif

__device__ __forceinline__ double rhs_w(double u, double mass) { return 3.0 * mass * u * u - u; }

// e / s of the error norm, bit-identical to the IEEE quotient. CUDA's double
// division leaves its inline fast path for a subroutine when the quotient is
// below ~2^-126 — including a zero numerator, which one of the two error
// components is on ~45% of far-field steps. A zero numerator gives +-0
// directly (s > 0); tiny ones are scaled by 2^900 first: a 2^900 is exact, its
// quotient takes the fast path and (>= 2^-940, normal for |a| >= 2^-900,
// s <= 2^40) scales back exactly, RN(a 2^900 / s) 2^-900 = RN(a / s)
// (tools/div_scale_check.c).
__device__ __forceinline__ double err_ratio(double e, double s) {
    const double ae = fabs(e);
    if (ae < 0x1p-120 && s > 0.0 && s <= 0x1p40) {
        if (ae == 0.0) return e;
        if (ae >= 0x1p-900) return ((e * 0x1p900) / s) * 0x1p-900;
    }
    return e / s;
}

// The reference's norm before its sqrt (geodesic.cpp:125-130), same operations.
__device__ __forceinline__ double exact_err2(double e0, double s0, double e1, double s1) {
    const double q0 = err_ratio(e0, s0), q1 = err_ratio(e1, s1);
    double err2 = 0.0;
    err2 += q0 * q0;
    err2 += q1 * q1;
    return err2 / 2.0;
}

// geodesic.cpp:84-162. Returns false on StepSizeUnderflow (phi/u/w then hold
// the failure state, as StepSizeUnderflow::state does).
// The step hint carried from one window to the next (geodesic.cpp:106,160):
// hint = h_try * clamp(0.9 * err^-0.14 * err_prev^0.08, 0.2, 5) of the
// window's last (accepted) step. It only matters when it is below the next
// window's dphi; it is kept as its inputs and evaluated lazily (below).
#ifdef BHRT_HINT_COUNT
__device__ unsigned long long g_hint_count[4];  // developer counters: exact hints, binding hints, multi-step windows
#endif
#ifndef BHRT_NO_LAZY_ERR
// (e0, s0, e1, s1) of a window's last step whose error norm was only bounded
// (hs.err2 = -1): the exact norm is formed from them if a hint needs it.
// One slot per thread of the 128-thread blocks of the mode-R kernels.
__shared__ double g_lazy_err[4][128];
#endif
__device__ __forceinline__ double exact_err2(double e0, double s0, double e1, double s1);

struct HintState {
    double h_try, err2, pprev;  // last accepted step, its squared error norm (see below), err_prev^0.08
    bool pending;               // false: no hint yet (hint = 0 in the reference)
};

// First step size of a window: min(hint, dphi), or dphi without a hint.
// A fp32 lower bound of the PI factor (|error| << the 0.1% margin) decides
// whether hint >= dphi for sure — then min(hint, dphi) = dphi exactly and
// the device pow is skipped; otherwise the exact double is formed.
__device__ __forceinline__ double window_h0(const HintState& hs, double dphi) {
    if (!hs.pending) return dphi;
    // err^2 <= 1e-12: err^-0.14 >= 6.9, pprev >= 1e-4^0.08 = 0.4786, so the
    // factor is >= 2.98 (or the clamp 5) and the hint >= 2.98 h_try; when
    // 2.9 h_try already covers dphi no pow is needed (most far-field windows)
    // A lazy norm (err2 = -1, see integrate_window) is known to be <= 2^-60.
    if (hs.err2 <= 1e-12 && 2.9 * hs.h_try >= dphi * 1.00001) return dphi;
    double err2 = hs.err2;
#ifndef BHRT_NO_LAZY_ERR
    if (err2 < 0.0) {
        const int t = threadIdx.x;
        err2 = exact_err2(g_lazy_err[0][t], g_lazy_err[1][t], g_lazy_err[2][t], g_lazy_err[3][t]);
    }
#endif
    if (err2 >= 0.0 && err2 <= 1.0 + 0x1p-52) {
        // err^2 <= 1e-30: err^-0.14 >= 126, pprev >= 1e-4^0.08 = 0.48, so the
        // factor is clamped to exactly 5 (also for err = 0: pow -> inf)
        float lo = 5.0f;
        if (err2 > 1e-30) {  // err^-0.14 = (err^2)^-0.07
            const float lf = 0.9f * exp2f(-0.07f * __log2f((float)err2)) * (float)hs.pprev;
            lo = fminf(fmaxf(lf * 0.999f, 0.2f), 5.0f);
        }
        if ((float)hs.h_try * lo >= (float)dphi * 1.00001f) return dphi;
    }
    const double factor = clampd(0.9 * pow(sqrt(err2), -0.7 / 5.0) * hs.pprev, 0.2, 5.0);
    const double hint = hs.h_try * factor;
#ifdef BHRT_HINT_COUNT
    atomicAdd(&g_hint_count[0], 1ull);
    if (hint < dphi) atomicAdd(&g_hint_count[1], 1ull);
#endif
    return hint > 0.0 ? dmin(hint, dphi) : dphi;
}

// geodesic.cpp:84-162. Returns false on StepSizeUnderflow (phi/u/w then hold
// the failure state, as StepSizeUnderflow::state does). pow_prev0 =
// pow(1e-4, 0.4 / 5) from the host libm: the err_prev factor of the first
// step of each window (err_prev starts at 1e-4) — the same double the
// reference multiplies by, without a device pow.
__device__ bool integrate_window(double& phi, double& u, double& w, double dphi, double mass,
                                 double rtol, double atol, HintState& hs, unsigned& nsteps,
                                 unsigned& nrej, double pow_prev0) {
    double y0 = u, y1 = w;
    double k10 = y1, k11 = rhs_w(y0, mass);
    double remaining = dphi;
    double h = window_h0(hs, dphi);
    double err_prev = 1e-4;
    double pprev = pow_prev0;  // pow(err_prev, 0.4 / 5)
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
        // err2 = the reference's err before its sqrt (geodesic.cpp:125-130);
        // err = sqrt(err2) is formed only where a pow needs it (rare). The
        // acceptance test err <= 1 is err2 <= 1 + 2^-52: RN(sqrt(x)) <= 1 iff
        // sqrt(x) <= 1 + 2^-53 (ties to even), i.e. x <= 1 + 2^-52 + 2^-106.
        double err2 = 0.0;
        bool lazy = false;
        const double tiny = 1e-42 * atol;
        if (fabs(e0) < tiny && fabs(e1) < tiny) {
            // s >= atol, so the norm is < 1e-42 < 1e-30. Every later use of
            // err is then independent of its value: the step is accepted, the
            // PI factor clamps to exactly 5 (err^-0.14 > 1.5e4, err_prev^0.08
            // >= 0.48), err_prev becomes 1e-4. 0 stands in for it, sparing
            // the divisions' and sqrt's denormal slow paths (frequent for
            // near-linear far-field windows). NaNs fail the test above.
#ifndef BHRT_NO_LAZY_ERR
        } else if (fabs(e0) <= s0 * 0x1p-30 && fabs(e1) <= s1 * 0x1p-30) {
            // both quotients <= 2^-30: err2 <= 2^-60, the step is accepted;
            // the exact norm is formed only where it is used (below, window_h0)
            lazy = true;
#endif
        } else {
            err2 = exact_err2(e0, s0, e1, s1);
        }
        if (lazy || err2 <= 1.0 + 0x1p-52) {
            y0 = n0;
            y1 = n1;
            k10 = k70;
            k11 = k71;
            remaining -= h_try;
            ++nsteps;
            if (!(remaining > 0.0)) {  // window done: the hint is formed lazily (window_h0)
#ifndef BHRT_NO_LAZY_ERR
                if (lazy) {
                    const int t = threadIdx.x;
                    g_lazy_err[0][t] = e0;
                    g_lazy_err[1][t] = s0;
                    g_lazy_err[2][t] = e1;
                    g_lazy_err[3][t] = s1;
                    hs = {h_try, -1.0, pprev, true};
                    break;
                }
#endif
                hs = {h_try, err2, pprev, true};
                break;
            }
            if (lazy) err2 = exact_err2(e0, s0, e1, s1);
            const double err = sqrt(err2);
#ifdef BHRT_HINT_COUNT
            atomicAdd(&g_hint_count[2], 1ull);
#endif
            h = h_try * clampd(0.9 * pow(err, -0.7 / 5.0) * pprev, 0.2, 5.0);
            err_prev = dmax(err, 1e-4);
            pprev = pow(err_prev, 0.4 / 5.0);
        } else {
            h = h_try * clampd(0.9 * pow(sqrt(err2), -0.2), 0.1, 0.9);
            ++nrej;
        }
        if (h < 1e-14 && remaining > 0.0) {
            phi = phi + (dphi - remaining);
            u = y0;
            w = y1;
            return false;
        }
    }
    phi = phi + dphi;
    u = y0;
    w = y1;
    return true;
}

// OrbitalPlaneBasis::point (geodesic.cpp:37-39)
__device__ __forceinline__ V3 plane_point(V3 origin, V3 e1, V3 e2, double r, double phi) {
    return add(origin, scl(add(scl(e1, cos(phi)), scl(e2, sin(phi))), r));
}

__device__ __forceinline__ void poly_put(double* pts, int cap, int k, V3 q) {
    if (k < cap) {
        pts[3 * k] = q.x;
        pts[3 * k + 1] = q.y;
        pts[3 * k + 2] = q.z;
    }
}

struct RResult {
    int obj;        // HORIZON / SKY / STALLED or -BHRT_NUMERICAL
    V3 edir;        // escape direction (SKY with at least one window)
    bool chord;     // edir is valid (else the ray escapes along its launch direction)
    double phi;     // phi at termination
    double defl;    // deflection_of_ray total (DEFL only)
};

// trace() window loop, geodesic.cpp:189-236, for a non-radial ray with
// orbital-plane basis (e1, e2) and initial state (u, w). Only (phi, u) of the
// last two window ends are kept; the escape direction is the normalised last
// chord of the polyline (geodesic.cpp:211-212). With DEFL the per-segment
// turning of deflection_of_ray (geodesic.cpp:248-260) is accumulated too.
// With POLY the polyline itself is written too (trace()'s RayPolyline::points,
// geodesic.cpp:195-236): pts[k] for k < cap (3 doubles each), the full point
// count in npoly (which may exceed cap: the caller re-runs with more room).
template <bool DEFL, bool POLY = false>
__device__ __forceinline__ RResult window_loop(const KParams& p, V3 origin, V3 center, V3 e1, V3 e2,
                                               double u, double w, unsigned& nsteps, unsigned& nrej,
                                               double* pts = nullptr, int cap = 0, int* npoly = nullptr,
                                               V3 ray_dir = {0.0, 0.0, 0.0}) {
    RResult R;
    R.obj = BHRT_OBJ_NONE;
    R.edir = mk(0.0, 0.0, 0.0);
    R.chord = false;
    R.defl = 0.0;
    double phi = 0.0;
    HintState hs{0.0, 0.0, 0.0, false};
    double prev_phi = 0.0, prev_u = 0.0, last_phi = 0.0, last_u = 0.0;
    int npts = 1;
    V3 p_prev = origin;
    double prev_x = 0.0, prev_y = 0.0;
    if (POLY) poly_put(pts, cap, 0, origin);
    for (;;) {
        if (u >= p.u_cap) { R.obj = BHRT_OBJ_HORIZON; break; }
        if (u <= p.u_esc && w < 0.0) {
            R.obj = BHRT_OBJ_SKY;
            const bool had_window = npts >= 2;
            if (POLY && !had_window)  // launched beyond the escape radius moving outward
                poly_put(pts, cap, npts++, add(origin, scl(ray_dir, p.escape_radius)));
            if (had_window) {
                const V3 last = plane_point(center, e1, e2, 1.0 / last_u, last_phi);
                const V3 prev = npts == 2 ? origin : plane_point(center, e1, e2, 1.0 / prev_u, prev_phi);
                R.edir = normalized(sub(last, prev));
                R.chord = true;
            }
            break;
        }
        if (phi > p.phi_max) { R.obj = BHRT_OBJ_STALLED; break; }
        // segment_dphi, geodesic.cpp:76-80
        const double hyp = glibc_hypot(u, w);
        const double dphi = clampd(p.epsilon * u * u / hyp, 1e-6, 0.1);
        if (!integrate_window(phi, u, w, dphi, p.mass, p.rel_tol, p.abs_tol, hs, nsteps, nrej,
                              p.ref_pow_prev0)) {
            if (p.mass > 0.0 && u >= p.u_cap) {
                if (POLY) {  // the underflow point, unless it repeats the last one (geodesic.cpp:222-224)
                    const V3 q = plane_point(center, e1, e2, 1.0 / u, phi);
                    const V3 last = npts == 1 ? origin : plane_point(center, e1, e2, 1.0 / last_u, last_phi);
                    if (norm(sub(q, last)) > 0.0) poly_put(pts, cap, npts++, q);
                }
                R.obj = BHRT_OBJ_HORIZON;
                break;
            }
            R.obj = -BHRT_NUMERICAL;
            R.edir = mk(u, 2.0, 0.0);  // StepSizeUnderflow at u (geodesic.cpp:157)
            break;
        }
        if (!(u > 0.0)) {  // geodesic.cpp:233-234
            R.obj = -BHRT_NUMERICAL;
            R.edir = mk(u, 1.0, 0.0);
            break;
        }
        prev_phi = last_phi;
        prev_u = last_u;
        last_phi = phi;
        last_u = u;
        if (POLY) poly_put(pts, cap, npts, plane_point(center, e1, e2, 1.0 / u, phi));
        ++npts;
        if (DEFL) {
            const V3 pt = plane_point(center, e1, e2, 1.0 / u, phi);
            const V3 seg = sub(pt, p_prev);
            const double sx = dot(seg, e1), sy = dot(seg, e2);
            if (npts > 2) R.defl += atan2(prev_x * sy - prev_y * sx, prev_x * sx + prev_y * sy);
            prev_x = sx;
            prev_y = sy;
            p_prev = pt;
        }
    }
    R.phi = phi;
    if (POLY) *npoly = npts;
    return R;
}

#ifndef BHRT_REF_MINB
#define BHRT_REF_MINB 8  // 64 regs, 32 warps/SM: 1/4/6/7/8/10 blocks -> 31.7/31.8/28.6/28.5/28.3/29.4 ms (960x540 mode R)
#endif
template <bool DIAG>  // DIAG: failed samples carry (u, kind) (bhrt_cuda.cu failure_text)
__global__ void __launch_bounds__(128, BHRT_REF_MINB) trace_reference_kernel(const __grid_constant__ KParams p) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned nsteps = 0, nrej = 0;
    const bool valid = i < n;
    const SampleId id = sample_of(p, valid ? i : 0);
    int obj = BHRT_OBJ_NONE;
    V3 edir = mk(0.0, 0.0, 0.0);
    double phi_end = 0.0;
    if (valid) {
        const V3 origin = vld(p.cam_pos), center = vld(p.center);
        const V3 dir = camera_ray(p, id.x, id.y, id.s);
        const Basis B = plane_basis(p, dir);
        edir = dir;
        if (!B.ok) {  // radial: geodesic.cpp:175-187
            obj = dot(dir, sub(center, origin)) > 0.0 ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY;
        } else {
            double u, w;
            initial_conditions(p, dir, u, w);
            const RResult R = window_loop<false>(p, origin, center, B.e1, B.e2, u, w, nsteps, nrej);
            obj = R.obj;
            if ((obj == BHRT_OBJ_SKY && R.chord) || (DIAG && obj < 0)) edir = R.edir;
            phi_end = R.phi;
        }
    }
    finish_sample(p, valid, id, obj, -1, edir, phi_end, nsteps, nrej);
    warp_add_stats(p.stats, nsteps, nrej, valid ? 1u : 0u);
}

// Ray batch (bhrt_cuda_trace_rays): the reference's
// trace() (geodesic.cpp:164-238) on caller rays {origin[3], dir[3]}, one
// record per ray; with defl != nullptr also deflection_of_ray
// (geodesic.cpp:240-262; NaN unless the ray escapes). The per-ray basis and
// initial state follow geodesic.cpp:49-65 (oracle orc_plane_basis /
// orc_initial_conditions, same operations). Origins inside the horizon are
// rejected on the host before launch.
// With POLY (bhrt_cuda_trace_polylines) each ray also writes its polyline:
// up to cap points at pts + 3 cap i, the full count at npoly[i].
template <bool DEFL, bool POLY>
__global__ void __launch_bounds__(128, BHRT_REF_MINB) trace_rays_kernel(const __grid_constant__ KParams p, const double* rays,
                                                         long long n, bhrt_ray_record* records, double* defl,
                                                         double* pts, int cap, int* npoly) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V3 origin = vld(rays + 6 * i), dir = vld(rays + 6 * i + 3), center = vld(p.center);
    unsigned nsteps = 0, nrej = 0;
    bhrt_ray_record rec;
    rec.sphere = -1;
    rec.phi = 0.0;
    V3 pt = mk(0.0, 0.0, 0.0);
    double d = 0.0;
    const V3 v = sub(origin, center);
    const V3 e1 = normalized(v);
    const V3 tangential = sub(dir, scl(e1, dot(dir, e1)));
    if (norm(tangential) < 1e-12) {  // radial: geodesic.cpp:175-187
        rec.object = dot(dir, sub(center, origin)) > 0.0 ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY;
        if (rec.object == BHRT_OBJ_SKY) pt = dir;
        if (POLY) {
            double* q = pts + (size_t)3 * cap * i;
            poly_put(q, cap, 0, origin);
            const double len = rec.object == BHRT_OBJ_SKY ? p.escape_radius : norm(v) - 2.0 * p.mass;
            poly_put(q, cap, 1, add(origin, scl(dir, len)));
            npoly[i] = 2;
        }
    } else {
        const V3 e2 = normalized(tangential);
        const double r0 = norm(v);
        const double b = norm(cross(v, dir));
        const double u = 1.0 / r0, w = -dot(v, dir) / (r0 * b);
        const RResult R = window_loop<DEFL, POLY>(p, origin, center, e1, e2, u, w, nsteps, nrej,
                                                  POLY ? pts + (size_t)3 * cap * i : nullptr, cap,
                                                  POLY ? npoly + i : nullptr, dir);
        rec.object = R.obj;
        if (R.obj == BHRT_OBJ_SKY) pt = R.chord ? R.edir : dir;
        rec.phi = R.phi;
        d = fabs(R.defl);
    }
    rec.steps = (int)nsteps;
    rec.rejected = (int)nrej;
    rec.point[0] = pt.x;
    rec.point[1] = pt.y;
    rec.point[2] = pt.z;
    records[i] = rec;
    if (DEFL) defl[i] = rec.object == BHRT_OBJ_SKY ? d : CUDART_NAN;
}

void launch_trace_rays(const KParams& p, const double* rays, long long n, bhrt_ray_record* records,
                       double* defl, cudaStream_t st) {
    const unsigned blocks = (unsigned)((n + 127) / 128);
    if (defl)
        trace_rays_kernel<true, false><<<blocks, 128, 0, st>>>(p, rays, n, records, defl, nullptr, 0, nullptr);
    else
        trace_rays_kernel<false, false><<<blocks, 128, 0, st>>>(p, rays, n, records, nullptr, nullptr, 0, nullptr);
}

void launch_trace_polylines(const KParams& p, const double* rays, long long n, bhrt_ray_record* records,
                            double* pts, int cap, int* npoly, cudaStream_t st) {
    const unsigned blocks = (unsigned)((n + 127) / 128);
    trace_rays_kernel<false, true><<<blocks, 128, 0, st>>>(p, rays, n, records, nullptr, pts, cap, npoly);
}

#ifdef BHRT_HINT_COUNT
extern "C" void bhrt_debug_hint_counts(unsigned long long out[4]) {
    cudaMemcpyFromSymbol(out, g_hint_count, sizeof(unsigned long long) * 4);
}
#endif

void launch_reference(const KParams& p, cudaStream_t st) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    if (p.diag)
        trace_reference_kernel<true><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(p);
    else
        trace_reference_kernel<false><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(p);
}

}  // namespace bhrt_b200
