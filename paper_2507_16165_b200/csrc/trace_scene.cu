// trace_scene.cu — RK4 / RKF45 renderers with disk + sphere hit tests.
//
// One sample per thread. The hot loop keeps only (phi, u, w, h), the state
// before the last step and the next event angle in registers; the ray's
// orbital-plane frame, disk line and sphere-candidate windows live in
// per-thread shared-memory slots (lane-major, conflict-free) that only setup,
// event steps and escape touch. Operation order mirrors the oracle
// (oracle/bhrt_oracle.c trace_scene / step_events / escape_dir), so records
// are bit-identical up to libdevice transcendentals outside the step.
// The shading and the escape direction are inlined in the RKF45
// instantiation (config 2: 5.79 -> 5.71 ms late in round 2; out of line won
// earlier, 7.72 -> 7.64, when the kernel held more state) and called out of
// line in the RK4 one (config 0: 1.20 vs 1.26 ms); the table kernel inlines.
#ifndef BHRT_INL_SHADE
#define BHRT_INL_SHADE __noinline__
#endif
// the escape direction out of line too (once per escaping ray): 7.27 -> 7.20 ms
#ifndef BHRT_INL_ESC
#define BHRT_INL_ESC __noinline__
#endif
#include "device_common.cuh"

namespace bhrt_b200 {


#ifndef BHRT_SCENE_BLOCK
#define BHRT_SCENE_BLOCK 128
#endif
constexpr int kBlock = BHRT_SCENE_BLOCK;
constexpr int kSlots = kCullSlots;
constexpr float kWinMargin = 5e-4f;  // fp32 window slack (rad); windows only cull
#ifndef BHRT_SCENE_MINB
// min resident blocks per SM (register cap 102): measured on B200, config 2:
// 3 -> 10.3, 4 -> 8.83, 5 -> 8.65, 6 -> 9.12 ms (5 spills only outside the step)
#define BHRT_SCENE_MINB 5
#endif
#ifndef BHRT_SCENE_MINB_RK4
// the RK4 instantiation (config 0: few long latency-bound rays) keeps more
// registers: 2 / 3 / 4 / 5 / 6 blocks per SM -> 1.21 / 1.21 / 1.22 / 1.34 / 1.48 ms
#define BHRT_SCENE_MINB_RK4 4
#endif

// Per-ray slots (lane-major: slot index = ray's position in the block, so
// a warp's 32 accesses hit 32 consecutive words — conflict-free).
template <int NS>
struct SceneSmT {
    static constexpr int kNS = NS;
    double e2[3][NS], n[3][NS];  // e1 is the per-frame KParams::cam_e1
    double sigma[NS], energy[NS], next_disk[NS];
    int list[NS];  // the ray's candidate list (KParams::cull record), read in place
    int nc[NS];
    float next_sph[NS];
};
using SceneSm = SceneSmT<kBlock>;

template <int NS>
__device__ __forceinline__ V3 ld3(const double (&a)[3][NS], int t) { return {a[0][t], a[1][t], a[2][t]}; }
template <int NS>
__device__ __forceinline__ void st3(double (&a)[3][NS], int t, V3 v) {
    a[0][t] = v.x;
    a[1][t] = v.y;
    a[2][t] = v.z;
}

// Sphere centre relative to the hole, in the oracle's order (center - O).
__device__ __forceinline__ V3 sphere_c(const KParams& p, int k) {
    const bhrt_sphere& s = p.spheres[k];
    return {__ldg(&s.center[0]) - p.center[0], __ldg(&s.center[1]) - p.center[1],
            __ldg(&s.center[2]) - p.center[2]};
}

// atan2 for culling only: odd minimax polynomial on [0, 1] after octant
// reduction, |error| < 2e-6 rad (checked in tests/test_abi.py against numpy);
// every caller widens by >= 5e-4 rad. About a third of atan2f's instructions.
__device__ __forceinline__ float atan2_cull(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float a = __fdividef(fminf(ax, ay), fmaxf(ax, ay));
    const float s = a * a;
    float r = fmaf(fmaf(fmaf(fmaf(fmaf(-0.01172120f, s, 0.05265332f), s, -0.11643287f), s, 0.19354346f), s,
                        -0.33262347f),
                   s, 0.99997726f) *
              a;
    if (ay > ax) r = 1.57079637f - r;
    if (x < 0.0f) r = 3.14159274f - r;
    return copysignf(r, y);
}

// A candidate window recurs every 2 pi of orbit angle (the circle is the
// same each winding). The occurrence in use at angle f is the first whose
// end is not before f; the lists keep the first occurrence and every ray
// derives its current one (fp32, k * 2 pi by one fma: within 1e-5 rad of
// repeated additions, far inside the windows' 1e-4 rad margins), so no
// per-ray window state is stored.
__device__ __forceinline__ float2 window_at(float4 w, float f) {
    if (w.y >= f) return make_float2(w.x, w.y);
    constexpr float k2pi = 2.0f * (float)PI_D;
    float kf = ceilf((f - w.y) * (1.0f / k2pi));
    float hi = fmaf(kf, k2pi, w.y);
    while (hi < f) {
        kf += 1.0f;
        hi = fmaf(kf, k2pi, w.y);
    }
    return make_float2(fmaf(kf, k2pi, w.x), hi);
}

__device__ __forceinline__ const CullList& cull_list(const KParams& p, int li) {
    return static_cast<const CullList*>(p.cull)[li];
}
__device__ __forceinline__ int cull_k(const CullList& L, int i) {
    return __ldg(reinterpret_cast<const unsigned char*>(L.k) + i);
}

// Disk line + sphere candidates (oracle ray_events_setup). Returns the first
// event angle.
template <class SM>
__device__ BHRT_INL_SETUP double events_setup(const KParams& p, SM& sm, int t, V3 e1, V3 e2, V3 n) {
    double next_disk = CUDART_INF;
    sm.sigma[t] = 1.0;
    if (p.disk_enabled) {
        // the disk line in plane coordinates: (L.e1, L.e2) = (-e2.y, e1.y)
        // (oracle ray_events_setup)
        const double lx = -e2.y, ly = e1.y;
        if (lx * lx + ly * ly >= 1e-24) {  // |L| >= 1e-12
            const double pl = atan2_est(ly, lx);
            next_disk = pl > 0.0 ? pl : pl + PI_D;
            sm.sigma[t] = pl > 0.0 ? 1.0 : -1.0;
            // the unit line (lx/nl, ly/nl) and L/nl are formed at hit time (disk_line)
        }
    }
#ifdef BHRT_EXPERIMENT_NODISKEV
    next_disk = CUDART_INF;  // timing experiment only: no disk events
#endif
    sm.next_disk[t] = next_disk;
    int nc = 0;
    float next_sph = CUDART_INF_F;
#ifdef BHRT_EXPERIMENT_NOCAND
    const int ns = 0;  // timing experiment only: no sphere candidates
#else
    const int ns = p.n_spheres;
#endif
    if (p.cull && ns > 0) {
        // plane-angle bin and orientation -> the frame's precomputed list of
        // conservative candidates with their windows (KParams::cull,
        // build_cull_lists_kernel), read in place
        const float na = (float)(n.x * p.cull_a[0] + n.y * p.cull_a[1] + n.z * p.cull_a[2]);
        const float nb = (float)(n.x * p.cull_b[0] + n.y * p.cull_b[1] + n.z * p.cull_b[2]);
        float th = atan2_cull(nb, na);  // lists cover +-1e-5 rad beyond their bin
        const bool flip = th < 0.0f;
        if (flip) th += (float)PI_D;
        int bin = (int)(th * (float)(p.cull_bins / PI_D));
        bin = bin < 0 ? 0 : (bin >= p.cull_bins ? p.cull_bins - 1 : bin);
        const int li = 2 * bin + (flip ? 1 : 0);
        // the ray reads its list's windows in place at event steps (window_at)
        const int2 hd = __ldg(reinterpret_cast<const int2*>(&cull_list(p, li)));
        nc = hd.x;
        if (nc > 0) next_sph = __int_as_float(hd.y);
        sm.list[t] = li;
    } else if (ns > 0) {
        nc = -1;  // no culling basis (never for a valid camera): every event step tests every sphere
    }
    if (nc < 0) next_sph = -CUDART_INF_F;
#ifdef BHRT_EXPERIMENT_NOSPHEREEVENTS
    nc = 0;  // timing experiment only: candidates computed, never tested
    next_sph = CUDART_INF_F;
#endif
#ifdef BHRT_COUNTERS
    atomicAdd(&p.stats[6], (unsigned long long)(nc < 0 ? 100 : nc));
#endif
    sm.nc[t] = nc;
    sm.next_sph[t] = next_sph;
    return dmin(next_disk, (double)next_sph);
}

struct Hit {
    int obj, sphere;
    V3 point;
};

// Unit disk line in plane coordinates and world space (oracle ray_events_setup
// values, same operations), formed only when a disk crossing lands in the annulus.
template <class SM>
__device__ __forceinline__ void disk_line(const KParams& p, const SM& sm, int t, double& dlx, double& dly, V3& Lw) {
    const V3 e1 = vld(p.cam_e1), e2 = ld3(sm.e2, t);
    const double lx = -e2.y, ly = e1.y;
    const double inl = 1.0 / sqrt(lx * lx + ly * ly);  // one reciprocal (oracle ray_events_setup)
    dlx = lx * inl;
    dly = ly * inl;
    Lw = scl(add(scl(e1, lx), scl(e2, ly)), inl);
}

// Sphere half of step_events(): first entering hit on the step's S
// equal-angle sub-chords among the candidates in act (all spheres when the
// candidate slots overflowed). Rare after radial culling (~0.04 per ray on
// config 2), so it is kept out of line: its registers do not count against
// the step loop's occupancy.
template <class SM>
__device__ BHRT_INL_SPH bool sphere_search(const KParams& p, const SM& sm, int t, double pa, double h,
                                           double ua, double ub, const Cubic cu, unsigned act, int nc,
                                           int& bsph, double& bqx, double& bqy) {
    const bool test_all = nc < 0;
    // Candidate-outer evaluation of the oracle's sub-chord-outer search:
    // each candidate scans only the sub-chords its (conservative) window
    // overlaps and stops at its first hit; the winner is the
    // lexicographic minimum of (sub-chord, chord parameter), ties to the
    // lower slot — the same hit the oracle finds.
    int S = 1;
    if (h > p.chord_dphi) S = (int)ceil(h / p.chord_dphi);
    const double dl = h / S;
    double cd_, sd_, c0, s0;
    if (dl <= 0.02) {
        // sub-chord rotation: Taylor series, truncation < 1e-20 for dl <= 0.02
        // (the oracle calls cos/sin; both are correctly rounded to ~1 ulp)
        const double d2 = dl * dl;
        cd_ = fma(fma(fma(fma(d2, -1.0 / 3628800.0, 1.0 / 40320.0), d2, -1.0 / 720.0), d2, 1.0 / 24.0),
                  d2 * d2, fma(d2, -0.5, 1.0));
        sd_ = fma(fma(fma(fma(d2, 1.0 / 362880.0, -1.0 / 5040.0), d2, 1.0 / 120.0), d2, -1.0 / 6.0),
                  d2 * dl, dl);
    } else {
        sincos(dl, &sd_, &cd_);
    }
    sincos(pa, &s0, &c0);
    const float fpa = (float)pa, rdl = 1.0f / (float)dl;  // conservative range only
    int best_j = S;
    double best_t = CUDART_INF;
    const int ncand = test_all ? p.n_spheres : nc;
    for (int a = 0; a < ncand; ++a) {
        int k, j0 = 0, j1 = S - 1;
        if (test_all) {
            k = a;
        } else {
            if (!(act & (1u << a))) continue;
            const CullList& L = cull_list(p, sm.list[t]);
            k = cull_k(L, a);
            BHRT_ASSERT(k < p.n_spheres);
            // the window occurrence step_events tested (at the step start)
            const float2 wn = window_at(__ldg(reinterpret_cast<const float4*>(L.win[a])), fpa);
            // clamp in float first: windows may be infinite
            const float fS = (float)S;
            j0 = (int)fminf(fmaxf(floorf((wn.x - fpa) * rdl) - 1.0f, 0.0f), fS);
            j1 = (int)fminf(fmaxf(floorf((wn.y - fpa) * rdl) + 1.0f, 0.0f), fS - 1.0f);
        }
        j1 = min(j1, best_j);
        if (j0 > j1) continue;
        const V3 e1 = vld(p.cam_e1), e2 = ld3(sm.e2, t), n = ld3(sm.n, t);
        const V3 c = sphere_c(p, k);
        const double r = __ldg(&p.spheres[k].radius);
        const double dn = dot(c, n);
        if (!(fabs(dn) < r)) continue;
        const double ccx = dot(c, e1), ccy = dot(c, e2);  // = the oracle's cand_t values
        const double rho2 = r * r - dn * dn;
        double cj = c0, sj = s0;
        for (int j = 0; j < j0; ++j) {  // same recurrence values as the sequential walk
            const double ck = cj * cd_ - sj * sd_;
            sj = sj * cd_ + cj * sd_;
            cj = ck;
        }
        const double uj = j0 == 0 ? ua : hermite_eval(cu, (double)j0 / S);
        const double rj = 1.0 / uj;
        double xj = cj * rj, yj = sj * rj;
        for (int j = j0; j <= j1; ++j) {
            const double ck = cj * cd_ - sj * sd_;
            const double sk = sj * cd_ + cj * sd_;
            const double uk = (j + 1 == S) ? ub : hermite_eval(cu, (double)(j + 1) / S);
            const double rk = 1.0 / uk;
            const double xk = ck * rk, yk = sk * rk;
            const double dx = xk - xj, dy = yk - yj;
            const double mx = xj - ccx, my = yj - ccy;
            const double A = dx * dx + dy * dy;
            const double Bq = mx * dx + my * dy;
            const double Cq = mx * mx + my * my - rho2;
            if (Cq > 0.0) {
                const double disc = Bq * Bq - A * Cq;
                if (!(disc < 0.0)) {
                    const double tq = (-Bq - sqrt(disc)) / A;
                    if (tq >= 0.0 && tq <= 1.0) {
                        if (j < best_j || tq < best_t) {
                            best_j = j;
                            best_t = tq;
                            bsph = k;
                            bqx = xj + tq * dx;
                            bqy = yj + tq * dy;
                        }
                        break;
                    }
                }
            }
            cj = ck;
            sj = sk;
            xj = xk;
            yj = yk;
        }
    }
    return best_j < S;
}

// Oracle step_events(): disk = exact phi-event on the step's Hermite
// interpolant; spheres = first entering hit on S equal-angle sub-chords.
// Returns true on hit; always advances the event state and next_ev.
template <class SM>
__device__ BHRT_INL_EVT bool step_events(const KParams& p, SM& sm, int t, double pa, double ua,
                                         double wa, double pb, double ub, double wb, double& next_ev,
                                         Hit& hit) {
    const double h = pb - pa;
    double next_disk = sm.next_disk[t];
#ifdef BHRT_COUNTERS
    atomicAdd(&p.stats[7], 1ull);
#endif
    const bool disk_in = next_disk > pa && next_disk <= pb;
    // ---- spheres
    const int nc = sm.nc[t];
    const bool test_all = nc < 0;
    // No window starts by pb (next_sph = the smallest window start, passed
    // windows already moved on): no candidate meets the step, none is passed,
    // so the sphere half is skipped entirely — disk-only event steps.
    const bool sph_here = test_all || sm.next_sph[t] <= (float)pb;
    unsigned act = 0;
    unsigned ang = 0;  // candidates whose angular window meets the step
    float next_sph = sm.next_sph[t];
    const CullList* L = nullptr;
    if (!test_all && sph_here) {
        // one pass over the list: the occurrence of each window in use at
        // the step start meets the step or not; the next window start after
        // the step is the first occurrence not ending before pb
        L = &cull_list(p, sm.list[t]);
        const float fa = (float)pa, fb = (float)pb;
        next_sph = CUDART_INF_F;
        for (int i = 0; i < nc; ++i) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(L->win[i]));
            const float2 wa_ = window_at(w, fa);
            if (wa_.x <= fb && wa_.y >= fa) ang |= 1u << i;
            next_sph = fminf(next_sph, wa_.y >= fb ? wa_.x : window_at(w, fb).x);
        }
    }
    // the step's Hermite interpolant, needed for a disk crossing, a window
    // meeting the step or the test-all search
    Cubic cu;
    if (disk_in || ang || test_all) cu = hermite_coef(h, ua, wa, ub, wb);
    // ---- disk (only the radius is kept across the sphere search; the disk
    // line is formed after it, so little stays live across that call)
    bool disk_hit = false;
    double r_ev;
    const double sigma = sm.sigma[t];
    if (disk_in) {
        const double tt = (next_disk - pa) / h;
        const double u_ev = hermite_eval(cu, tt);
        if (u_ev > 0.0) {
            r_ev = 1.0 / u_ev;
            disk_hit = r_ev >= p.disk_r_in && r_ev <= p.disk_r_out;
        }
    }
    if (ang) {
        // Conservative radial extent of the step's polyline. Its vertices lie
        // on the Hermite interpolant u(t), t in [0, 1]; u(t) minus the chord
        // between its end values is -t(1-t)(a2 + a3(1+t)), at most
        // (|a2| + 2|a3|)/4 in size (fp32, widened by 1e-5 of the coefficient
        // scale). A sub-chord of angle dl between radii r1, r2 stays within
        // [min(r1, r2) cos(dl), max(r1, r2)].
        float slo = 0.0f, shi = CUDART_INF_F;
        {
            const float a1 = (float)cu.a1, a2 = (float)cu.a2, a3 = (float)cu.a3, a0 = (float)ua;
            const float dev = 0.25f * (fabsf(a2) + 2.0f * fabsf(a3));
            float umin = fminf(a0, (float)ub) - dev, umax = fmaxf(a0, (float)ub) + dev;
            const float slack = 1e-5f * (fabsf(a0) + fabsf(a1) + fabsf(a2) + fabsf(a3));
            umin -= slack;
            umax += slack;
            const float dl = fminf((float)h, (float)p.chord_dphi);
            if (umax > 0.0f) slo = (1.0f / umax) * (1.0f - 0.5f * dl * dl) * (1.0f - 1e-5f);
            if (umin > 0.0f) shi = (1.0f / umin) * (1.0f + 1e-5f);
        }
        for (unsigned m = ang; m; m &= m - 1) {
            const int i = __ffs(m) - 1;
            const float2 r = __ldg(reinterpret_cast<const float2*>(L->win[i]) + 1);  // (rlo, rhi)
            if (r.x <= shi && r.y >= slo) act |= 1u << i;
        }
    }
    bool sph_hit = false;
    int bsph;          // outputs of sphere_search, read only when sph_hit
    double bqx, bqy;
    if (act || test_all) {
        sph_hit = sphere_search(p, sm, t, pa, h, ua, ub, cu, act, nc, bsph, bqx, bqy);
        if (sph_hit) {
            const V3 e1 = vld(p.cam_e1), e2 = ld3(sm.e2, t);
            hit.point = add(vld(p.center), add(scl(e1, bqx), scl(e2, bqy)));
        }
#ifdef BHRT_COUNTERS
        atomicAdd(&p.stats[4], 1ull);
        atomicAdd(&p.stats[5], (unsigned long long)__popc(act));
#endif
    }
    if (disk_hit) {
        double ux, uy;
        V3 Lw;
        disk_line(p, sm, t, ux, uy, Lw);
        if (sph_hit) {
            const double dlx = sigma * ux, dly = sigma * uy;
            if (bqx * dly - bqy * dlx > 0.0)
                disk_hit = false;
            else
                sph_hit = false;
        }
        if (disk_hit) hit.point = add(vld(p.center), scl(Lw, sigma * r_ev));
    }
    if (disk_hit) {
        hit.obj = BHRT_OBJ_DISK;
        hit.sphere = -1;
    } else if (sph_hit) {
        hit.obj = BHRT_OBJ_SPHERE;
        hit.sphere = bsph;
    }
    // advance the event state past pb
    if (next_disk <= pb) {
        double sg = sigma;
        while (next_disk <= pb) {
            next_disk += PI_D;
            sg = -sg;
        }
        sm.next_disk[t] = next_disk;
        sm.sigma[t] = sg;
    }
    if (!test_all && sph_here) sm.next_sph[t] = next_sph;
    next_ev = dmin(next_disk, (double)next_sph);
    return disk_hit || sph_hit;
}

__device__ __forceinline__ V3 tangent_dir(V3 e1, V3 e2, double phi, double u, double w) {
    double c, sn;
    sincos(phi, &sn, &c);
    const double tx = -u * sn - w * c, ty = u * c - w * sn;
    return unit_fast(add(scl(e1, tx), scl(e2, ty)));
}

// Oracle escape_dir(): tangent at the r = escape_radius crossing of the last
// step (Hermite + 2 Newton iterations, u' from the first integral).
template <class SM>
__device__ __forceinline__ V3 escape_dir_body(const KParams& p, SM& sm, int t, bool has_step, double pa,
                                      double ua, double wa, double pb, double ub, double wb) {
    const V3 e1 = vld(p.cam_e1), e2 = ld3(sm.e2, t);
#ifdef BHRT_EXPERIMENT_NOESC
    if (ua != -1.0) return e1;  // timing experiment only: no escape direction
#endif
    if (!has_step || !(ua > p.u_esc)) return tangent_dir(e1, e2, pb, ub, wb);
    const double u_esc = p.u_esc;
    const double h = pb - pa;
    const Cubic cu = hermite_coef(h, ua, wa, ub, wb);
    double tt = (ua - u_esc) / (ua - ub);
    for (int it = 0; it < 2; ++it) {
        const double f = hermite_eval(cu, tt) - u_esc;
        const double df = hermite_deval(cu, tt);
        if (df != 0.0) tt = tt - f / df;
        tt = clampd(tt, 0.0, 1.0);
    }
    const double us = hermite_eval(cu, tt);
    const double M2 = 2.0 * p.mass;
    const double q = sm.energy[t] - us * us + M2 * us * us * us;
    const double ws = -sqrt(q > 0.0 ? q : 0.0);
    return tangent_dir(e1, e2, pa + h * tt, us, ws);
}
// The RK4 instantiation calls it out of line (its registers stay off the
// step loop: config 0 1.20 vs 1.26 ms inlined); the RKF45 one inlines it
// with the shading (config 2 5.79 -> 5.71 ms).
template <class SM>
__device__ BHRT_INL_ESC V3 escape_dir(const KParams& p, SM& sm, int t, bool has_step, double pa,
                                      double ua, double wa, double pb, double ub, double wb) {
    return escape_dir_body(p, sm, t, has_step, pa, ua, wa, pb, ub, wb);
}

// Straight radial ray (geodesic.cpp:175-187) with scene hit tests.
__device__ __noinline__ Hit radial_scene(const KParams& p, V3 origin, V3 dir, double seg_len, bool captured) {
    const V3 O = vld(p.center);
    double best = seg_len;
    Hit H;
    H.obj = captured ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY;
    H.sphere = -1;
    if (p.disk_enabled && dir.y != 0.0) {
        const double tq = (O.y - origin.y) / dir.y;
        if (tq >= 0.0 && tq <= best) {
            const V3 q = sub(add(origin, scl(dir, tq)), O);
            const double rq = sqrt(q.x * q.x + q.z * q.z);
            if (rq >= p.disk_r_in && rq <= p.disk_r_out) {
                best = tq;
                H.obj = BHRT_OBJ_DISK;
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
        const double tq = -B - sqrt(disc);
        if (tq >= 0.0 && tq < best) {
            best = tq;
            H.obj = BHRT_OBJ_SPHERE;
            H.sphere = k;
        }
    }
    H.point = H.obj == BHRT_OBJ_SKY ? dir : add(origin, scl(dir, best));
    return H;
}

// DIAG (failure_text's re-trace only): failed samples also carry (u, kind)
// in their point for the host's failure text; the production instantiation
// keeps nothing extra alive on those exits.
template <int INTEG, bool DIAG>
__global__ void __launch_bounds__(kBlock, INTEG == BHRT_INTEGRATOR_RK4 ? BHRT_SCENE_MINB_RK4 : BHRT_SCENE_MINB)
    trace_scene_kernel(const __grid_constant__ KParams p) {
    __shared__ SceneSm sm;
    const int t = threadIdx.x;

    const long long n = (long long)p.n_rows * p.width * p.spp;
    const long long i = (long long)blockIdx.x * blockDim.x + t;
    unsigned nsteps = 0, nrej = 0;
    const bool valid = i < n;
    const SampleId id = sample_of(p, valid ? i : 0);
    Hit H;
    H.obj = BHRT_OBJ_NONE;
    H.sphere = -1;
    H.point = mk(0.0, 0.0, 0.0);
    double phi = 0.0;
    if (valid) {
        const V3 origin = vld(p.cam_pos), O = vld(p.center);
        const V3 D = camera_dir_raw(p, id.x, id.y, id.s);
        const Frame F = scene_frame(p, D);
        if (!F.ok) {
            const V3 dir = normalized(D);
            const double r0 = norm(sub(origin, O));
            const bool cap = dot(dir, sub(O, origin)) > 0.0;
            H = radial_scene(p, origin, dir, cap ? r0 - 2.0 * p.mass : p.escape_radius, cap);
        } else {
            const V3 e1 = vld(p.cam_e1);
            const V3 nrm = cross(e1, F.e2);
            st3(sm.e2, t, F.e2);
            st3(sm.n, t, nrm);
            double u = p.cam_u0, w = F.w;
            sm.energy[t] = w * w + u * u - (2.0 * p.mass) * u * u * u;
            double next_ev = events_setup(p, sm, t, e1, F.e2, nrm);
            double pp = 0.0, up = 0.0, wp = 0.0;  // RK4: state before the last accepted step
            bool has_step = false;
            if (INTEG == BHRT_INTEGRATOR_RK4) {
                const double h = p.step;
                // tests/oracles.hpp:47-54 loop structure (budget, capture and
                // escape tested before each step). The tests of the next trip
                // follow the step that produced the state; one combined test
                // (pn below the next event angle and phi_max, un strictly in
                // (u_esc, u_cap)) commits the common step, which none of them
                // can stop.
                if (!(phi < p.phi_max)) {
                    H.obj = BHRT_OBJ_STALLED;
                } else if (u >= p.u_cap) {
                    H.obj = BHRT_OBJ_HORIZON;
                } else if (u <= p.u_esc && w < 0.0) {
                    H.obj = BHRT_OBJ_SKY;
                } else {
                    double nev_eff = dmin(next_ev, p.phi_max);
                    for (;;) {
                        double un, wn;
                        rk4_step(u, w, h, p.mass, un, wn);
                        const double pn = phi + h;
                        ++nsteps;
                        if (pn < nev_eff && un > p.u_esc && un < p.u_cap) {
                            pp = phi;
                            up = u;
                            wp = w;
                            has_step = true;
                            phi = pn;
                            u = un;
                            w = wn;
                            continue;
                        }
                        if (pn >= next_ev && step_events(p, sm, t, phi, u, w, pn, un, wn, next_ev, H)) {
                            phi = pn;
                            break;
                        }
                        nev_eff = dmin(next_ev, p.phi_max);
                        pp = phi;
                        up = u;
                        wp = w;
                        has_step = true;
                        phi = pn;
                        u = un;
                        w = wn;
                        if (!(u > 0.0)) {
                            H.obj = -BHRT_NUMERICAL;
                            if (DIAG) H.point = mk(u, 1.0, 0.0);
                            break;
                        }
                        if (!(phi < p.phi_max)) { H.obj = BHRT_OBJ_STALLED; break; }
                        if (u >= p.u_cap) { H.obj = BHRT_OBJ_HORIZON; break; }
                        if (u <= p.u_esc && w < 0.0) { H.obj = BHRT_OBJ_SKY; break; }
                    }
                }
            } else {
                double h = p.step;
#ifdef BHRT_EXPERIMENT_NOLOOP
                H.obj = BHRT_OBJ_SKY;  // timing experiment only: setup + escape + shading
                if (u < 0.0)
#endif
                // geodesic.cpp:199-236 loop structure, with the capture and
                // escape tests of the next trip evaluated right after the
                // accepted step that produced the state (same tests, same
                // order: numerical, capture, escape, then stall at the top):
                // the escape direction then reads the step's end points from
                // registers instead of a saved previous state.
                if (u >= p.u_cap) {
                    H.obj = BHRT_OBJ_HORIZON;
                } else if (u <= p.u_esc && w < 0.0) {
                    H.obj = BHRT_OBJ_SKY;
                    H.point = escape_dir_body(p, sm, t, false, 0.0, 0.0, 0.0, phi, u, w);
                } else {
                    // One combined test per accepted step covers the common
                    // case — no event, capture, escape, numerical failure,
                    // underflow or stall can follow: pn below the next event
                    // angle and phi_max, un strictly inside (u_esc, u_cap)
                    // (so un > 0), hn >= 1e-14 — and commits the step. Any
                    // other outcome takes the exact tests in their original
                    // order below; the stall test of the next trip is
                    // evaluated at the end of this one (phi is unchanged by
                    // a rejection, and phi = 0 < phi_max on entry).
                    double nev_eff = dmin(next_ev, p.phi_max);
                    for (;;) {
                        double un, wn, hn;
                        // controller factors straight from the (L1-resident) global tables: measured
                        // faster than staging them in shared memory (8.21 -> 8.05 ms, config 2)
                        if (rkf45_step(u, w, h, p.M3, p.rel_tol, p.abs_tol, p.max_step, p.grow, p.shrink, un,
                                       wn, hn)) {
                            const double pn = phi + h;
                            ++nsteps;
                            // integer order tests (lt_pos): pn, hn > 0 and u_esc, u_cap >= 0
                            // (nev_eff may be negative: pn above it either way); a NaN un
                            // fails un < u_cap and takes the exact tests below
                            if (lt_pos(pn, nev_eff) & gt_pos(un, p.u_esc) & lt_pos(un, p.u_cap) &
                                ge_pos(hn, 1e-14)) {
                                phi = pn;
                                u = un;
                                w = wn;
                                h = hn;
                                continue;
                            }
                            if (pn >= next_ev && step_events(p, sm, t, phi, u, w, pn, un, wn, next_ev, H)) {
                                phi = pn;
                                break;
                            }
                            nev_eff = dmin(next_ev, p.phi_max);
                            if (!(un > 0.0)) {
                                H.obj = -BHRT_NUMERICAL;
                                if (DIAG) H.point = mk(un, 1.0, 0.0);
                                phi = pn;
                                u = un;
                                w = wn;
                                break;
                            }
                            if (un >= p.u_cap) {
                                H.obj = BHRT_OBJ_HORIZON;
                                phi = pn;
                                u = un;
                                break;
                            }
                            if (un <= p.u_esc && wn < 0.0) {
                                H.obj = BHRT_OBJ_SKY;
                                H.point = escape_dir_body(p, sm, t, true, phi, u, w, pn, un, wn);
                                phi = pn;
                                break;
                            }
                            phi = pn;
                            u = un;
                            w = wn;
                        } else {
                            ++nrej;
                        }
                        h = hn;
                        if (h < 1e-14) {
                            H.obj = (p.mass > 0.0 && u >= p.u_cap) ? BHRT_OBJ_HORIZON : -BHRT_NUMERICAL;
                            if (DIAG && H.obj < 0) H.point = mk(u, 2.0, 0.0);
                            break;
                        }
                        if (phi > p.phi_max) { H.obj = BHRT_OBJ_STALLED; break; }
                    }
                }
            }
            if (INTEG == BHRT_INTEGRATOR_RK4 && H.obj == BHRT_OBJ_SKY)
                H.point = escape_dir(p, sm, t, has_step, pp, up, wp, phi, u, w);
        }
    }
    finish_sample<INTEG == BHRT_INTEGRATOR_RKF45>(p, valid, id, H.obj, H.sphere, H.point, phi, nsteps, nrej);
    warp_add_stats(p.stats, nsteps, nrej, valid ? 1u : 0u);
}

// ----------------------------------------------------------------- culling lists
// One thread per (plane-angle bin, orientation): the conservative candidate
// list of EVERY orbital plane of the frame whose normal is
// s (cos t a + sin t b) with t in the bin widened by kCullEps (the ray's
// fp32 angle is within 3e-6 of its exact one) and s = +1 / -1. With
// f(t) = ca cos t + cb sin t and g(t) = ca sin t - cb cos t (c = centre - hole,
// ca = c.a, cb = c.b, cx = c.e1): c.n = s f, c.e2 = s g, and g is monotone on
// the bin unless f changes sign there (then g reaches +-|(ca, cb)|). A sphere
// is a candidate when min |f| < r; its window is the union over the bin of
// [atan2(cy, cx) -+ asin(rho / rc)] (rho <= sqrt(r^2 - min f^2), rc >= its
// minimum), infinite when the circle may contain the hole or straddle the
// atan2 cut; its radial extent [min rc - rho, max rc + rho]. All in double
// with relative slack, then rounded outward — culling only selects which
// exact fp64 tests run (sphere_search), so the lists cannot change results.
constexpr double kCullEps = 1e-5;
constexpr double kCullMargin = 1e-4;  // rad, beyond the exact union (fp32 rounding of the windows)

__global__ void __launch_bounds__(128) build_cull_lists_kernel(const __grid_constant__ KParams p, CullList* out) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= 2 * p.cull_bins) return;
    const int bin = id >> 1;
    const double sg = (id & 1) ? -1.0 : 1.0;
    const double bw = PI_D / p.cull_bins;
    double s0, c0, s1, c1;
    sincos(bin * bw - kCullEps, &s0, &c0);
    sincos((bin + 1) * bw + kCullEps, &s1, &c1);
    const V3 a = vld(p.cull_a), b = vld(p.cull_b), e1 = vld(p.cam_e1), O = vld(p.center);
    CullList L;
    L.n = 0;
    float next = CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < kCullSlots; ++i) {
        L.k[i] = 0;
        L.win[i][0] = L.win[i][1] = L.win[i][2] = L.win[i][3] = 0.0f;
    }
    for (int k = 0; k < p.n_spheres; ++k) {
        const V3 c = sub(vld(p.spheres[k].center), O);
        const double r = p.spheres[k].radius;
        const double ca = dot(c, a), cb = dot(c, b), cx = dot(c, e1);
        const double f0 = ca * c0 + cb * s0, f1 = ca * c1 + cb * s1;
        const double g0 = ca * s0 - cb * c0, g1 = ca * s1 - cb * c1;
        const double R = sqrt(ca * ca + cb * cb);
        const double slack = 1e-9 * (R + fabs(cx) + r) + 1e-12;
        const bool fcross = !(f0 > 0.0 && f1 > 0.0) && !(f0 < 0.0 && f1 < 0.0);
        const double fmn = fcross ? 0.0 : fmin(fabs(f0), fabs(f1));
        if (!(fmn < r + slack)) continue;  // no plane of the bin cuts the sphere
        if (L.n == kCullSlots) {
            L.n = -1;  // more than the slots: the rays of this list test every sphere
            break;
        }
        const double fl = fmn > slack ? fmn - slack : 0.0;
        const double rho = sqrt(fmax(r * r - fl * fl, 0.0)) * (1.0 + 1e-9) + slack;
        double glo = fmin(g0, g1), ghi = fmax(g0, g1);
        if (fcross) {
            if (g0 + g1 > 0.0) ghi = R; else glo = -R;
        }
        glo -= slack;
        ghi += slack;
        const double cylo = sg > 0.0 ? glo : -ghi, cyhi = sg > 0.0 ? ghi : -glo;
        const bool cy0 = cylo <= 0.0 && cyhi >= 0.0;
        const double cymin2 = cy0 ? 0.0 : fmin(cylo * cylo, cyhi * cyhi);
        const double cymax2 = fmax(cylo * cylo, cyhi * cyhi);
        const double rcmin = sqrt(cx * cx + cymin2), rcmax = sqrt(cx * cx + cymax2);
        float lo = -CUDART_INF_F, hi = CUDART_INF_F;
        if (rcmin > rho && !(cx < 0.0 && cy0)) {
            const double half = asin(fmin(1.0, rho / rcmin));
            const double pa = atan2(cylo, cx), pb = atan2(cyhi, cx);
            double l = fmin(pa, pb) - half - kCullMargin, h = fmax(pa, pb) + half + kCullMargin;
            if (h < 0.0) {
                l += 2.0 * PI_D;
                h += 2.0 * PI_D;
            }
            lo = (float)l;
            hi = (float)h;
        }
        const int i = L.n++;
        L.k[i] = (uint8_t)k;
        L.win[i][0] = lo;
        L.win[i][1] = hi;
        L.win[i][2] = (float)((rcmin - rho) * (1.0 - 1e-6) - 1e-6);
        L.win[i][3] = (float)((rcmax + rho) * (1.0 + 1e-6) + 1e-6);
        next = fminf(next, lo);
    }
    L.next_lo = next;
    out[id] = L;
}

void launch_cull_build(const KParams& p, CullList* out, cudaStream_t st) {
    const int n = 2 * p.cull_bins;
    build_cull_lists_kernel<<<(n + 127) / 128, 128, 0, st>>>(p, out);
}

void launch_scene(const KParams& p, cudaStream_t st) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    const unsigned blocks = (unsigned)((n + kBlock - 1) / kBlock);
    if (p.integrator == BHRT_INTEGRATOR_RK4) {
        if (p.diag)
            trace_scene_kernel<BHRT_INTEGRATOR_RK4, true><<<blocks, kBlock, 0, st>>>(p);
        else
            trace_scene_kernel<BHRT_INTEGRATOR_RK4, false><<<blocks, kBlock, 0, st>>>(p);
    } else {
        if (p.diag)
            trace_scene_kernel<BHRT_INTEGRATOR_RKF45, true><<<blocks, kBlock, 0, st>>>(p);
        else
            trace_scene_kernel<BHRT_INTEGRATOR_RKF45, false><<<blocks, kBlock, 0, st>>>(p);
    }
}

}  // namespace bhrt_b200
