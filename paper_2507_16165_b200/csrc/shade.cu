// shade.cu — per-pixel shading of the per-sample records (render.cpp:22-49):
// sky (image.cpp:131-169 or checker), disk ramp, Lambertian spheres; sample-
// order accumulation, round-half-away quantisation; kernel launch wrapper.
#include "device_common.cuh"

namespace bhrt_b200 {

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
__global__ void __launch_bounds__(256) shade_kernel(const __grid_constant__ KParams p) {
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
void launch_reference(const KParams& p, cudaStream_t st);
void launch_scene(const KParams& p, cudaStream_t st);

int launch_trace(const KParams& p, cudaStream_t st, int* launches, cudaEvent_t* ev) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    if (n <= 0) return 0;
    if (p.integrator != BHRT_INTEGRATOR_REFERENCE && p.integrator != BHRT_INTEGRATOR_RK4 &&
        p.integrator != BHRT_INTEGRATOR_RKF45)
        return -1;
    if (ev) cudaEventRecord(ev[0], st);
    if (p.integrator == BHRT_INTEGRATOR_REFERENCE)
        launch_reference(p, st);
    else
        launch_scene(p, st);
    ++*launches;
    if (ev) cudaEventRecord(ev[1], st);
    const long long npix = (long long)p.n_rows * p.width;
    shade_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(p);
    ++*launches;
    if (ev) cudaEventRecord(ev[2], st);
    return 0;
}

}  // namespace bhrt_b200
