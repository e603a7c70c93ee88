// table.cu — approximate mode (BASELINE.json configs[3]).
//
//   build_table_kernel : one thread per impact parameter b_e (100,000 uniform
//                        entries over [0, b_max]); RKF45 (scene tolerances) of
//                        the INBOUND null orbit u(psi), u(0) = 0, u'(0) = 1/b,
//                        sampled at psi_j = j*dpsi, ending at capture or
//                        periapsis (the orbit is fixed by b alone:
//                        u'^2 + u^2 - 2Mu^3 = 1/b^2, geodesic.cpp:272-275)
//   bind_table_kernel  : per frame, each entry's inbound psi of the camera's u0
//   trace_table_kernel : per sample, no integration: b from the ray's first
//                        integral, linear interpolation between entries
//                        floor(b) and floor(b)+1, disk events and escape angle
//                        from the interpolated orbit, fused shading.
// Normative text: oracle/bhrt_oracle.c (table_entry_build,
// orc_table_inbound_psi, table_u, table_plan, trace_table); same operation
// order, so GPU tables equal the oracle's bit for bit.
#include "device_common.cuh"

namespace bhrt_b200 {

__device__ __forceinline__ double hermite_ddeval(const Cubic& c, double t) {
    return fma(6.0 * c.a3, t, 2.0 * c.a2);
}

// Newton on H(t) = target (or H'(t) = 0), 3 iterations, clamped (oracle cubic_solve).
__device__ __forceinline__ double cubic_solve(const Cubic& c, double t, double target, bool deriv) {
    for (int it = 0; it < 3; ++it) {
        const double f = deriv ? hermite_deval(c, t) : hermite_eval(c, t) - target;
        const double df = deriv ? hermite_ddeval(c, t) : hermite_deval(c, t);
        if (df != 0.0) t = t - f / df;
        t = clampd(t, 0.0, 1.0);
    }
    return t;
}

struct TabView {
    const double* smp;
    const double* ends;
    const int32_t* kind;
    const int32_t* n;
    int ns;
    double dpsi, inv_dpsi;  // inv_dpsi = RN(1 / dpsi) from the host
};

// a / b from the host's y = RN(1/b): RN(a y) plus one Markstein fma
// correction, the IEEE quotient when a is 0 or in [2^-900, 2^900] and b is
// a normal constant (no intermediate under/overflow; tools/div_check.c),
// else the division.
__device__ __forceinline__ double div_by(double a, double b, double y) {
    const double m = fabs(a);
    if (m >= 0x1p-900 && m <= 0x1p900) {
        const double q0 = a * y;
        return fma(fma(-q0, b, a), y, q0);
    }
    return a / b;
}

// oracle orc_table_inbound_psi
__device__ double inbound_psi(const TabView& T, int e, double target) {
    const int kind = T.kind[e], n = T.n[e];
    if (kind == 3 || n < 1) return -1.0;
    const double* S = T.smp + (size_t)e * T.ns * 2;
    const double* E = T.ends + 4 * (size_t)e;
    if (!(target > S[0])) return 0.0;
    int j;
    double h, ua, wa, ub, wb;
    if (!(S[2 * (n - 1)] > target)) {
        if (kind == 2 || E[1] < target) return -1.0;
        j = n - 1;
        h = E[0] - (double)j * T.dpsi;
        ua = S[2 * j];
        wa = S[2 * j + 1];
        ub = E[1];
        wb = E[2];
        if (!(h > 0.0)) return E[0];
    } else {
        int lo = 0, hi = n - 1;
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (S[2 * mid] <= target)
                lo = mid;
            else
                hi = mid;
        }
        j = lo;
        h = T.dpsi;
        ua = S[2 * j];
        wa = S[2 * j + 1];
        ub = S[2 * j + 2];
        wb = S[2 * j + 3];
    }
    const Cubic c = hermite_coef(h, ua, wa, ub, wb);
    const double t0 = ub > ua ? (target - ua) / (ub - ua) : 0.0;
    const double t = cubic_solve(c, t0, target, false);
    return (double)j * T.dpsi + h * t;
}

// One entry's per-frame metadata, loaded together as soon as the entry index
// is known (independent loads: one memory latency instead of a chain).
struct TabEntry {
    int kind, n;
    double pend, pesc, psi0;  // ends[0], ends[3], the camera's inbound psi
};

// The frame's packed entry record (bind_table_kernel): (psi0, psi_end),
// (psi_esc, kind | n << 32) — two 16-byte loads per entry.
__device__ __forceinline__ TabEntry tab_entry(const double* meta, int e) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(meta + 4 * (size_t)e));
    const double2 b = __ldg(reinterpret_cast<const double2*>(meta + 4 * (size_t)e + 2));
    const long long kn = __double_as_longlong(b.y);
    return {(int)(kn & 0xffffffff), (int)(kn >> 32), a.y, b.x, a.x};
}

// oracle table_u: u on entry e at orbit angle psi (mirrored past periapsis).
__device__ double table_u(const TabView& T, int e, const TabEntry& M, double psi) {
    const int kind = M.kind, n = M.n;
    const double* S = T.smp + (size_t)e * T.ns * 2;
    const double* E = T.ends + 4 * (size_t)e;
    const double pend = M.pend;
    if (kind == 1 && psi > pend) psi = 2.0 * pend - psi;
    if (psi < 0.0 || n < 1) return -1.0;
    int j = (int)floor(div_by(psi, T.dpsi, T.inv_dpsi));
    double h, ua, wa, ub, wb, pa;
    if (j >= n - 1) {
        if (kind == 2 || psi > pend) return -1.0;
        j = n - 1;
        pa = (double)j * T.dpsi;
        h = pend - pa;
        if (!(h > 0.0)) return __ldg(&E[1]);
        ua = __ldg(&S[2 * j]);
        wa = __ldg(&S[2 * j + 1]);
        ub = __ldg(&E[1]);
        wb = __ldg(&E[2]);
    } else {
        pa = (double)j * T.dpsi;
        h = T.dpsi;
        const double2 a = __ldg(reinterpret_cast<const double2*>(S + 2 * j));
        const double2 b = __ldg(reinterpret_cast<const double2*>(S + 2 * j + 2));
        ua = a.x;
        wa = a.y;
        ub = b.x;
        wb = b.y;
    }
    const Cubic c = hermite_coef(h, ua, wa, ub, wb);
    return hermite_eval(c, (psi - pa) / h);
}

// oracle table_entry_build
__global__ void __launch_bounds__(128) build_table_kernel(const __grid_constant__ KParams p, double* smp,
                                                           double* ends, int32_t* kind_out, int32_t* n_out) {
    __shared__ double grow[kQN], shrink[kQN];
    for (int k = threadIdx.x; k < kQN; k += blockDim.x) {
        grow[k] = p.grow[k];
        shrink[k] = p.shrink[k];
    }
    __syncthreads();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.table_entries) return;
    const double b = p.table_b_max * e / (p.table_entries - 1);
    double* S = smp + (size_t)e * p.table_ns * 2;
    double* E = ends + 4 * (size_t)e;
    if (!(b > 0.0)) {
        kind_out[e] = 3;
        n_out[e] = 0;
        E[0] = E[1] = E[2] = 0.0;
        E[3] = -1.0;
        return;
    }
    double u = 0.0, w = 1.0 / b, psi = 0.0, h = p.step;
    S[0] = u;
    S[1] = w;
    int cnt = 1, kind = 2;
    for (;;) {
        if (cnt >= p.table_ns) {
            E[0] = psi;
            E[1] = u;
            E[2] = w;
            break;
        }
        const double target = (double)cnt * p.table_dpsi;
        bool done = false;
        while (psi < target) {
            const double rem = target - psi;
            const bool last = !(h < rem);
            const double ht = last ? rem : h;
            double un, wn, hn;
            const bool acc = rkf45_step(u, w, ht, p.M3, p.rel_tol, p.abs_tol, p.max_step, grow, shrink, un, wn, hn);
            if (acc) {
                if (un >= p.u_cap || wn <= 0.0) {
                    const Cubic c = hermite_coef(ht, u, w, un, wn);
                    if (un >= p.u_cap) {
                        const double t = cubic_solve(c, (p.u_cap - u) / (un - u), p.u_cap, false);
                        E[0] = psi + ht * t;
                        E[1] = p.u_cap;
                        E[2] = hermite_deval(c, t) / ht;
                        kind = 0;
                    } else {
                        const double t = cubic_solve(c, w / (w - wn), 0.0, true);
                        E[0] = psi + ht * t;
                        E[1] = hermite_eval(c, t);
                        E[2] = 0.0;
                        kind = 1;
                    }
                    done = true;
                    break;
                }
                psi = last ? target : psi + ht;
                u = un;
                w = wn;
            }
            h = hn;
            if (h < 1e-14) {
                E[0] = psi;
                E[1] = u;
                E[2] = w;
                done = true;
                break;
            }
        }
        if (done) break;
        S[2 * cnt] = u;
        S[2 * cnt + 1] = w;
        ++cnt;
    }
    kind_out[e] = kind;
    n_out[e] = cnt;
    E[3] = -1.0;
}

// psi_esc per entry (needs the finished entry) and, per frame, psi0 of u0.
__global__ void bind_table_kernel(const __grid_constant__ KParams p, double* ends, double* meta,
                                  double u0, int with_esc) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.table_entries) return;
    TabView T{p.tab_smp, ends, p.tab_kind, p.tab_n, p.table_ns, p.table_dpsi, 1.0 / p.table_dpsi};
    if (with_esc) ends[4 * (size_t)e + 3] = inbound_psi(T, e, p.u_esc);
    if (meta) {  // the frame's packed record (tab_entry)
        const double* E = ends + 4 * (size_t)e;
        const long long kn = (long long)(uint32_t)T.kind[e] | ((long long)T.n[e] << 32);
        double* m = meta + 4 * (size_t)e;
        m[0] = inbound_psi(T, e, u0);
        m[1] = E[0];
        m[2] = E[3];
        m[3] = __longlong_as_double(kn);
    }
}

// oracle table_plan
__device__ __forceinline__ bool table_plan(const TabEntry& M, double w0, int& outcome, double& phi_end) {
    const int kind = M.kind;
    const double psi0 = M.psi0;
    if (kind == 3 || psi0 < 0.0) return false;
    const double pesc = M.pesc;
    if (w0 >= 0.0) {
        if (kind == 0) {
            outcome = BHRT_OBJ_HORIZON;
            phi_end = M.pend - psi0;
            return true;
        }
        if (kind == 2) {
            outcome = BHRT_OBJ_STALLED;
            phi_end = CUDART_INF;
            return true;
        }
        if (pesc < 0.0) return false;
        outcome = BHRT_OBJ_SKY;
        phi_end = (2.0 * M.pend - pesc) - psi0;
        return true;
    }
    if (pesc < 0.0) return false;
    outcome = BHRT_OBJ_SKY;
    phi_end = psi0 - pesc;
    return true;
}

#ifndef BHRT_TAB_MINB
#define BHRT_TAB_MINB 7  // 5/6/7/8/10/12 blocks -> 1.76/1.67/1.56/1.56/1.73/1.94 ms (config 3)
#endif
__global__ void __launch_bounds__(128, BHRT_TAB_MINB) trace_table_kernel(const __grid_constant__ KParams p) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const SampleId id = sample_of(p, valid ? i : 0);
    int obj = BHRT_OBJ_NONE;
    V3 point = mk(0.0, 0.0, 0.0);
    double phi_out = 0.0;
    unsigned nevals = 0;  // interpolated-orbit evaluations (the "steps" counter in table mode)
    if (valid) {
        const TabView T{p.tab_smp, p.tab_ends, p.tab_kind, p.tab_n, p.table_ns, p.table_dpsi, p.inv_table_dpsi};
        const V3 origin = vld(p.cam_pos), O = vld(p.center);
        const V3 D = camera_dir_raw(p, id.x, id.y, id.s);
        const Frame F = scene_frame(p, D);
        if (!F.ok) {  // radial: straight segment (geodesic.cpp:175-187); table mode has no spheres
            const V3 dir = normalized(D);
            const double r0 = norm(sub(origin, O));
            const bool cap = dot(dir, sub(O, origin)) > 0.0;
            const double seg = cap ? r0 - 2.0 * p.mass : p.escape_radius;
            obj = cap ? BHRT_OBJ_HORIZON : BHRT_OBJ_SKY;
            double best = seg;
            if (p.disk_enabled && dir.y != 0.0) {
                const double tq = (O.y - origin.y) / dir.y;
                if (tq >= 0.0 && tq <= best) {
                    const V3 q = sub(add(origin, scl(dir, tq)), O);
                    const double rq = sqrt(q.x * q.x + q.z * q.z);
                    if (rq >= p.disk_r_in && rq <= p.disk_r_out) {
                        best = tq;
                        obj = BHRT_OBJ_DISK;
                    }
                }
            }
            point = obj == BHRT_OBJ_SKY ? dir : add(origin, scl(dir, best));
        } else {
            const V3 e1 = vld(p.cam_e1), e2 = F.e2;
            const double u0 = p.cam_u0, w0 = F.w;
            const double M2 = 2.0 * p.mass;
            const double energy = w0 * w0 + u0 * u0 - M2 * u0 * u0 * u0;
#ifdef BHRT_EXPERIMENT_NOTAB
            if (energy != -12345.0) {  // timing experiment only: setup + shading, no table
                obj = BHRT_OBJ_SKY;
                point = unit_fast(D);
            } else if (!(energy > 0.0)) {
#else
            if (!(energy > 0.0)) {
#endif
                obj = BHRT_OBJ_STALLED;
            } else {
                const double b = 1.0 / sqrt(energy);
                // disk line (oracle ray_events_setup)
                double next_disk = CUDART_INF, sigma = 1.0;
                const double lx = -e2.y, ly = e1.y;  // (L.e1, L.e2), oracle ray_events_setup
                if (p.disk_enabled) {
                    const double nl2 = lx * lx + ly * ly;
                    if (nl2 >= 1e-24) {  // |L| >= 1e-12
                        const double pl = atan2_est(ly, lx);
                        next_disk = pl > 0.0 ? pl : pl + PI_D;
                        sigma = pl > 0.0 ? 1.0 : -1.0;
                        // the unit line L/|L| is formed only on a disk hit (below)
                    }
                }
                const int N = p.table_entries;
                const double x = div_by(b * (double)(N - 1), p.table_b_max, p.inv_table_b_max);
                int ie = (int)floor(x);
                if (ie > N - 2) ie = N - 2;
                BHRT_ASSERT(ie >= 0 && ie + 1 < N);
                const TabEntry Mi = tab_entry(p.tab_meta, ie), Mj = tab_entry(p.tab_meta, ie + 1);
                double f = x - (double)ie;
                if (Mi.kind == 3) f = 1.0;
                const double p0i = Mi.psi0, p0j = Mj.psi0;
                int oi = 0, oj = 0;
                double pi_ = 0.0, pj = 0.0;
                const bool vi = table_plan(Mi, w0, oi, pi_);
                const bool vj = table_plan(Mj, w0, oj, pj);
                int outcome = BHRT_OBJ_STALLED;
                double phi_end = 0.0, wi = 0.0, wj = 0.0;
                bool ok = true;
                if (vi && vj && oi == oj && f > 0.0 && f < 1.0) {
                    outcome = oi;
                    phi_end = outcome == BHRT_OBJ_STALLED ? CUDART_INF : (1.0 - f) * pi_ + f * pj;
                    wi = 1.0 - f;
                    wj = f;
                } else {
                    bool use_j = f >= 0.5;
                    if (use_j && !vj) use_j = false;
                    if (!use_j && !vi) use_j = true;
                    if (use_j ? !vj : !vi) {
                        ok = false;
                    } else {
                        outcome = use_j ? oj : oi;
                        phi_end = use_j ? pj : pi_;
                        wi = use_j ? 0.0 : 1.0;
                        wj = use_j ? 1.0 : 0.0;
                    }
                }
                if (!ok) {
                    obj = BHRT_OBJ_STALLED;
                } else {
                    if (phi_end > p.phi_max) outcome = BHRT_OBJ_STALLED;
                    const double stop = outcome == BHRT_OBJ_STALLED ? p.phi_max : phi_end;
                    const double sgn = w0 >= 0.0 ? 1.0 : -1.0;
                    bool hit = false;
                    while (next_disk < stop) {
                        const double ph = next_disk;
                        double ui = -1.0, uj = -1.0;
#ifdef BHRT_EXPERIMENT_NOTABU
                        // timing experiment only: no orbit-sample gathers
                        if (wi > 0.0) ui = 0.01 * (1.0 + ph);
                        if (wj > 0.0) uj = 0.01 * (1.0 + ph);
#else
                        if (wi > 0.0) ui = table_u(T, ie, Mi, p0i + sgn * ph);
                        if (wj > 0.0) uj = table_u(T, ie + 1, Mj, p0j + sgn * ph);
#endif
                        nevals += (wi > 0.0) + (wj > 0.0);
                        double u_ev;
                        if (wi > 0.0 && wj > 0.0 && ui >= 0.0 && uj >= 0.0)
                            u_ev = wi * ui + wj * uj;
                        else
                            u_ev = ui >= 0.0 ? ui : uj;
                        if (u_ev > 0.0) {
                            const double r_ev = 1.0 / u_ev;
                            if (r_ev >= p.disk_r_in && r_ev <= p.disk_r_out) {
                                obj = BHRT_OBJ_DISK;
                                const double inl = 1.0 / sqrt(lx * lx + ly * ly);  // oracle ray_events_setup
                                const V3 Lw = scl(add(scl(e1, lx), scl(e2, ly)), inl);
                                point = add(O, scl(Lw, sigma * r_ev));
                                phi_out = ph;
                                hit = true;
                                break;
                            }
                        }
                        next_disk += PI_D;
                        sigma = -sigma;
                    }
                    if (!hit) {
                        obj = outcome;
                        phi_out = outcome == BHRT_OBJ_STALLED ? p.phi_max : phi_end;
                        if (outcome == BHRT_OBJ_SKY) {
                            const double ue = p.u_esc;
                            const double q = energy - ue * ue + M2 * ue * ue * ue;
                            const double ws = -sqrt(q > 0.0 ? q : 0.0);
                            double c, sn;
                            sincos(phi_end, &sn, &c);  // one argument reduction (libdevice sin/cos values)
                            const double tx = -ue * sn - ws * c, ty = ue * c - ws * sn;
                            point = unit_fast(add(scl(e1, tx), scl(e2, ty)));
                        }
                    }
                }
            }
        }
    }
    finish_sample(p, valid, id, obj, -1, point, phi_out, 0u, 0u);
    warp_add_stats(p.stats, nevals, 0u, valid ? 1u : 0u);
}

void launch_table_build(const KParams& p, double* smp, double* ends, int32_t* kind, int32_t* n, cudaStream_t st) {
    const int blocks = (p.table_entries + 127) / 128;
    build_table_kernel<<<blocks, 128, 0, st>>>(p, smp, ends, kind, n);
    KParams q = p;
    q.tab_smp = smp;
    q.tab_kind = kind;
    q.tab_n = n;
    bind_table_kernel<<<(p.table_entries + 255) / 256, 256, 0, st>>>(q, ends, nullptr, 0.0, 1);
}

void launch_table_bind(const KParams& p, double* ends, double* meta, double u0, cudaStream_t st) {
    bind_table_kernel<<<(p.table_entries + 255) / 256, 256, 0, st>>>(p, ends, meta, u0, 0);
}

void launch_table_trace(const KParams& p, cudaStream_t st) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    trace_table_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(p);
}

}  // namespace bhrt_b200
