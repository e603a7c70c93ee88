// bhrt_cuda.cu — host side of the C ABI (include/bhrt_cuda.h).
//
// Owns device state (bhrt_ctx), validates scenes with the reference's rules
// and error taxonomy (render.cpp:11-20,68-75; geodesic.cpp:19-27;
// camera.cpp:30-43), hoists the per-frame camera math the reference redoes
// per ray, and launches the kernels in trace.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "bhrt_kernel_params.h"

namespace bhrt_b200 {

int launch_trace(const KParams& p, cudaStream_t st, int* launches, cudaEvent_t* ev);
void launch_table_build(const KParams& p, double* smp, double* ends, int32_t* kind, int32_t* n, cudaStream_t st);
void launch_table_bind(const KParams& p, double* ends, double* meta, double u0, cudaStream_t st);
void launch_trace_polylines(const KParams& p, const double* rays, long long n, bhrt_ray_record* records,
                            double* pts, int cap, int* npoly, cudaStream_t st);
void launch_trace_rays(const KParams& p, const double* rays, long long n, bhrt_ray_record* records,
                       double* defl, cudaStream_t st);
void launch_cull_build(const KParams& p, CullList* out, cudaStream_t st);

namespace {

constexpr double kPi = 3.141592653589793;
constexpr size_t kStatBytes = kStatWords * sizeof(unsigned long long);  // all counter slots

struct HV3 {
    double x, y, z;
};
HV3 hv(const double* a) { return {a[0], a[1], a[2]}; }
HV3 hsub(HV3 a, HV3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double hdot(HV3 a, HV3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
HV3 hcross(HV3 a, HV3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double hnorm(HV3 a) { return std::sqrt(hdot(a, a)); }
HV3 hnormalized(HV3 a) {
    const double n = hnorm(a);
    return {a.x / n, a.y / n, a.z / n};
}
void hput(double* d, HV3 a) { d[0] = a.x; d[1] = a.y; d[2] = a.z; }

int set_info(bhrt_status_info* info, int code, int px, int py, const char* msg) {
    if (info) {
        info->code = code;
        info->px = px;
        info->py = py;
        std::snprintf(info->message, sizeof info->message, "%s", msg);
    }
    return code;
}

int cuda_fail(bhrt_status_info* info, cudaError_t e, const char* where) {
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    return set_info(info, BHRT_DEVICE, -1, -1, buf);
}

#define CK(call)                                              \
    do {                                                      \
        const cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(info, e_, #call); \
    } while (0)

// camera.cpp:30-43
bool camera_basis(const bhrt_scene* s, HV3& f, HV3& r, HV3& u) {
    const HV3 axis = hsub(hv(s->cam_look_at), hv(s->cam_pos));
    const double len = hnorm(axis);
    if (len == 0.0) return false;
    f = {axis.x / len, axis.y / len, axis.z / len};
    const HV3 rr = hcross(f, {0.0, 1.0, 0.0});
    if (hnorm(rr) < 1e-9) return false;
    r = hnormalized(rr);
    u = hcross(r, f);
    return true;
}

int validate_trace(const bhrt_scene* s, bhrt_status_info* info) {
    if (!(s->epsilon > 0.0) || !(s->escape_radius > 0.0) || s->max_windings < 1 ||
        !(s->rel_tol > 0.0) || !(s->abs_tol > 0.0))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: invalid parameter");
    if (s->integrator < 0 || s->integrator > BHRT_INTEGRATOR_TABLE ||
        (s->integrator != BHRT_INTEGRATOR_REFERENCE && !(s->step > 0.0)) ||
        (s->integrator == BHRT_INTEGRATOR_RKF45 && !(s->max_step > 0.0 && s->max_step < 1.0)) ||
        (s->integrator == BHRT_INTEGRATOR_REFERENCE && (s->disk_enabled || s->n_spheres > 0)) ||
        (s->integrator == BHRT_INTEGRATOR_TABLE &&
         (s->n_spheres > 0 || s->table_entries < 2 || s->table_samples < 2 || !(s->table_b_max > 0.0) ||
          !(s->table_dpsi > 0.0) || !(s->max_step > 0.0 && s->max_step < 1.0))) ||
        !(s->chord_dphi > 0.0) || (s->n_spheres > 0 && s->spheres == nullptr) ||
        s->n_spheres < 0 || s->n_spheres > kMaxSpheres ||
        (s->sky_kind == BHRT_SKY_CHECKER && (s->checker_nu < 1 || s->checker_nv < 1)))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "scene extension: invalid parameter");
    HV3 f, r, u;
    if (!camera_basis(s, f, r, u))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "camera: degenerate orientation");
    return 0;
}

// RKF45 controller tables: f_q = 0.9 * 2^(-(q+1)/20), clamped.
void factor_tables(double* grow, double* shrink) {
    for (int i = 0; i < kQN; ++i) {
        const int q = kQMin + i;
        const double f = 0.9 * std::pow(2.0, -static_cast<double>(q + 1) / 20.0);
        grow[i] = f < 0.2 ? 0.2 : (5.0 < f ? 5.0 : f);
        shrink[i] = f < 0.1 ? 0.1 : (0.9 < f ? 0.9 : f);
    }
}

// Plane-angle culling basis (KParams::cull_a/b): every orbital plane of the
// frame contains the camera-hole axis v, so its normal is
// s (cos t a + sin t b) for unit a, b perpendicular to v. The per-bin
// candidate lists themselves are built on the device (trace_scene.cu
// build_cull_lists_kernel). Returns false when culling is not applicable.
constexpr int kCullBins = 4096;

bool cull_basis(const bhrt_scene* s, KParams& k) {
    if (s->integrator != BHRT_INTEGRATOR_RK4 && s->integrator != BHRT_INTEGRATOR_RKF45) return false;
    const HV3 v = hsub(hv(s->cam_pos), hv(s->center));
    if (hnorm(v) == 0.0) return false;
    const HV3 vh = hnormalized(v);
    // a: unit vector perpendicular to v, from the coordinate axis least aligned with it
    HV3 axis = {1.0, 0.0, 0.0};
    if (std::fabs(vh.y) < std::fabs(vh.x) && std::fabs(vh.y) <= std::fabs(vh.z)) axis = {0.0, 1.0, 0.0};
    else if (std::fabs(vh.z) < std::fabs(vh.x)) axis = {0.0, 0.0, 1.0};
    const HV3 a = hnormalized(hcross(vh, axis));
    const HV3 b = hcross(vh, a);
    hput(k.cull_a, a);
    hput(k.cull_b, b);
    k.cull_bins = kCullBins;
    return true;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    int ensure(size_t n) {
        if (n <= cap) return 0;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1));
        if (e != cudaSuccess) return -1;
        cap = n;
        return 0;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Per-sample records for unfused shading (spp not dividing 32). Renders of one frame may run concurrently on several
// streams, so each render takes a slot whose previous user has finished
// (event), growing the pool up to kRecSlots; past that it waits on a slot.
struct RecSlot {
    DevBuf<bhrt_ray_record> buf;
    cudaEvent_t done = nullptr;
};
constexpr size_t kRecSlots = 4;

}  // namespace
}  // namespace bhrt_b200

using namespace bhrt_b200;

struct bhrt_ctx {
    int device = 0;
    bool has_scene = false;
    KParams kp{};
    bhrt_scene scene{};
    DevBuf<uint8_t> sky;
    DevBuf<bhrt_sphere> spheres;
    DevBuf<double> tables;
    DevBuf<bhrt_ray_record> records;  // trace_rays / render_rows record outputs
    std::vector<RecSlot*> rec_pool;   // unfused-shading scratch (RecSlot)
    size_t rec_rr = 0;
    DevBuf<double> rays, defl;  // bhrt_cuda_trace_rays
    DevBuf<double> poly_pts;    // bhrt_cuda_trace_polylines
    DevBuf<int32_t> poly_n;
    DevBuf<double> checker;     // checker cell boundaries (KParams::checker_tab)
    DevBuf<uint8_t> out;
    DevBuf<unsigned long long> stats;
    DevBuf<CullList> cull;  // KParams::cull, 2 * kCullBins lists
    DevBuf<double> tab_smp, tab_ends, tab_meta;
    DevBuf<int32_t> tab_kind, tab_n;
    bool has_table = false;
    double table_key[10] = {0};
    cudaStream_t last_stream = nullptr;
    int launches = 0;
    int pending = 0;
    int32_t last_rows = 0;
    // pinned: [0..7] last render's counters (async D2H), [8..15] their reset pattern
    // pinned: [0, kStatWords) the last render's counter slots (async D2H),
    // [kStatWords, 2 kStatWords) their reset pattern; folded into stats_sum
    unsigned long long* host_slots = nullptr;
    unsigned long long stats_sum[8] = {0, 0, 0, ULLONG_MAX, 0, 0, 0, 0};
    bool in_frame = false;  // bhrt_ctx_frame_begin .. bhrt_ctx_finish: counters accumulate
    int32_t out_image = 0;  // bhrt_ctx_set_output_layout
    // scene uploads: pinned staging -> device on a private non-blocking stream;
    // renders wait on up_done, so set_scene does not stall other contexts
    cudaStream_t up_stream = nullptr;
    cudaEvent_t up_done = nullptr;
    cudaEvent_t render_done = nullptr;  // after the last render's counters copy
    std::vector<cudaEvent_t> frame_ev;  // one per render of the open frame (any streams)
    size_t frame_nev = 0;
    unsigned char* staging = nullptr;
    size_t staging_cap = 0;
    bool timing = false;
    bool timed = false;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    uint64_t upload_bytes = 0;  // host->device bytes staged by the last set_scene
    // one-shot host-buffer path (bhrt_cuda_render_rows): row bands alternate
    // between two render streams; each band's rows go device->pinned staging
    // on a copy stream while later bands render; the host then places them
    // in the caller's buffer as they land
    cudaStream_t band_stream[2] = {nullptr, nullptr};
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> band_ev;  // [2b] band b rendered, [2b+1] band b on the host
    unsigned char* host_out = nullptr;
    size_t host_out_cap = 0;
};

extern "C" {

int32_t bhrt_cuda_abi_version(void) { return BHRT_CUDA_ABI_VERSION; }

void bhrt_scene_defaults(bhrt_scene* s) {
    std::memset(s, 0, sizeof *s);
    s->mass = 1.0;
    s->cam_pos[2] = -20.0;
    s->vertical_fov = 60.0 * kPi / 180.0;
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
    const double ca[3] = {0.9, 0.9, 0.9}, cb[3] = {0.1, 0.1, 0.15};
    const double di[3] = {1.0, 0.95, 0.8}, dout[3] = {0.8, 0.25, 0.05};
    const double l[3] = {0.5, 1.0, -1.0};
    std::memcpy(s->checker_color_a, ca, sizeof ca);
    std::memcpy(s->checker_color_b, cb, sizeof cb);
    s->disk_r_in = 6.0;
    s->disk_r_out = 20.0;
    std::memcpy(s->disk_color_in, di, sizeof di);
    std::memcpy(s->disk_color_out, dout, sizeof dout);
    std::memcpy(s->light_dir, l, sizeof l);
    s->ambient = 0.1;
    s->table_entries = 100000;
    s->table_samples = 2048;
    s->table_b_max = 50.0;
    s->table_dpsi = 0.01;
}

int bhrt_validate_scene(const bhrt_scene* s, bhrt_status_info* info) {  // render.cpp:11-20
    set_info(info, 0, -1, -1, "");
    if (!s) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "scene is NULL");
    if (s->sky_kind == BHRT_SKY_IMAGE && (s->sky_rgb == nullptr || s->sky_width < 1 || s->sky_height < 1))
        return set_info(info, BHRT_USAGE, -1, -1, "scene: background image is required");
    if (s->width < 1 || s->height < 1)
        return set_info(info, BHRT_USAGE, -1, -1, "scene: image dimensions must be >= 1");
    if (s->spp < 1) return set_info(info, BHRT_USAGE, -1, -1, "scene: spp must be >= 1");
    if (s->mass < 0.0) return set_info(info, BHRT_USAGE, -1, -1, "scene: mass must be >= 0");
    const double d = hnorm(hsub(hv(s->cam_pos), hv(s->center)));
    if (d <= 2.0 * s->mass)
        return set_info(info, BHRT_USAGE, -1, -1, "scene: camera must be outside the event horizon");
    return 0;
}

int bhrt_make_spheres(uint64_t seed, int32_t n, const double center[3], double shell_min,
                      double shell_max, double radius_min, double radius_max, bhrt_sphere* out) {
    if (n < 0 || !(shell_min >= 0.0) || !(shell_max >= shell_min) || !(radius_min > 0.0) ||
        !(radius_max >= radius_min))
        return BHRT_INVALID_ARGUMENT;
    uint64_t x = seed;
    const auto next = [&x]() {
        uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    const auto unit = [&]() { return static_cast<double>(next() >> 11) * 0x1.0p-53; };
    const double lo3 = shell_min * shell_min * shell_min;
    const double hi3 = shell_max * shell_max * shell_max;
    for (int i = 0; i < n; ++i) {
        const double cz = 2.0 * unit() - 1.0;
        const double th = 2.0 * kPi * unit();
        const double rr = std::cbrt(lo3 + unit() * (hi3 - lo3));
        const double sxy = std::sqrt(1.0 - cz * cz);
        out[i].center[0] = center[0] + rr * (sxy * std::cos(th));
        out[i].center[1] = center[1] + rr * cz;
        out[i].center[2] = center[2] + rr * (sxy * std::sin(th));
        out[i].radius = radius_min + unit() * (radius_max - radius_min);
        out[i].albedo[0] = unit();
        out[i].albedo[1] = unit();
        out[i].albedo[2] = unit();
    }
    return 0;
}

int bhrt_make_bands(int32_t height, int32_t workers, int32_t* rs, int32_t* re, int32_t cap,
                    int32_t* count) {  // render.cpp:51-66
    if (height < 1 || workers < 1) return BHRT_INVALID_ARGUMENT;
    const int n = std::min(height, workers);
    if (cap < n) return BHRT_INVALID_ARGUMENT;
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

int32_t bhrt_tile_row_count(int32_t row_start, int32_t row_end, int32_t tile_rows,
                            int32_t tile_stride, int32_t tile_offset) {
    if (tile_rows < 1 || tile_stride < 1 || tile_offset < 0 || tile_offset >= tile_stride ||
        row_end < row_start)
        return -1;
    const int rows = row_end - row_start;
    const int full_tiles = rows / tile_rows, rem = rows % tile_rows;
    const int ntiles = full_tiles + (rem ? 1 : 0);
    int count = 0;
    for (int t = tile_offset; t < ntiles; t += tile_stride) count += (t < full_tiles) ? tile_rows : rem;
    return count;
}

double bhrt_flops_per_step(int32_t integrator) {
    // Algorithmic FP64 flops per accepted step, fma = 2.
    switch (integrator) {
        case BHRT_INTEGRATOR_REFERENCE: return 152.0;  // 110 stages + 38 error + 4 controller
        case BHRT_INTEGRATOR_RK4: return 39.0;         // tests/oracles.hpp:23-30, invariants hoisted
        case BHRT_INTEGRATOR_RKF45: return 137.0;      // DESIGN.md §Roofline op count
        default: return 0.0;
    }
}

int bhrt_ctx_create(int32_t device, bhrt_ctx** out, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "bhrt_ctx_create: bad device");
    CK(cudaSetDevice(device));
    std::unique_ptr<bhrt_ctx> c(new bhrt_ctx());
    c->device = device;
    if (c->stats.ensure(kStatWords) || c->tables.ensure(2 * kQN))
        return set_info(info, BHRT_DEVICE, -1, -1, "bhrt_ctx_create: cudaMalloc failed");
    CK(cudaMallocHost(&c->host_slots, 2 * kStatWords * sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&c->up_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->up_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->render_done, cudaEventDisableTiming));
    CK(cudaEventRecord(c->up_done, c->up_stream));
    for (int i = 0; i < 2 * kStatWords; ++i) c->host_slots[i] = 0;
    c->host_slots[3] = c->host_slots[kStatWords + 3] = ULLONG_MAX;
    double tb[2 * kQN];
    factor_tables(tb, tb + kQN);
    CK(cudaMemcpy(c->tables.p, tb, sizeof tb, cudaMemcpyHostToDevice));
    *out = c.release();
    return 0;
}

int bhrt_ctx_set_timing(bhrt_ctx* c, int32_t enable) {
    if (!c) return BHRT_INVALID_ARGUMENT;
    bhrt_status_info* info = nullptr;
    CK(cudaSetDevice(c->device));
    if (enable && !c->ev[0])
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
    c->timing = enable != 0;
    return 0;
}

int bhrt_ctx_kernel_ms(bhrt_ctx* c, float* trace_ms, float* shade_ms) {
    if (!c || !c->timed || c->pending) return BHRT_INVALID_ARGUMENT;
    bhrt_status_info* info = nullptr;
    CK(cudaSetDevice(c->device));
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, c->ev[0], c->ev[1]));
    CK(cudaEventElapsedTime(&b, c->ev[1], c->ev[2]));
    if (trace_ms) *trace_ms = a;
    if (shade_ms) *shade_ms = b;
    return 0;
}

void bhrt_ctx_destroy(bhrt_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    c->sky.release();
    c->spheres.release();
    c->tables.release();
    c->records.release();
    for (RecSlot* r : c->rec_pool) {
        r->buf.release();
        if (r->done) cudaEventDestroy(r->done);
        delete r;
    }
    c->rec_pool.clear();
    c->out.release();
    c->stats.release();
    c->cull.release();
    c->checker.release();
    c->rays.release();
    c->defl.release();
    c->poly_pts.release();
    c->poly_n.release();
    if (c->host_slots) cudaFreeHost(c->host_slots);
    if (c->staging) cudaFreeHost(c->staging);
    if (c->up_done) cudaEventDestroy(c->up_done);
    if (c->render_done) cudaEventDestroy(c->render_done);
    for (auto e : c->frame_ev) cudaEventDestroy(e);
    if (c->up_stream) cudaStreamDestroy(c->up_stream);
    for (auto st : c->band_stream)
        if (st) cudaStreamDestroy(st);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto e : c->band_ev) cudaEventDestroy(e);
    if (c->host_out) cudaFreeHost(c->host_out);
    c->tab_smp.release();
    c->tab_ends.release();
    c->tab_meta.release();
    c->tab_kind.release();
    c->tab_n.release();
    delete c;
}

int bhrt_ctx_set_scene(bhrt_ctx* c, const bhrt_scene* s, bhrt_status_info* info) {
    int rc = bhrt_validate_scene(s, info);
    if (rc) return rc;
    rc = validate_trace(s, info);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    // only this context's own work can still read its buffers: its last
    // render and its previous uploads (other contexts keep running)
    if (c->pending) CK(cudaEventSynchronize(c->render_done));
    CK(cudaStreamSynchronize(c->up_stream));
    // the parameters below are rebuilt in place: until every step of the
    // upload has succeeded the context holds no renderable scene (a failed
    // allocation/copy must not leave a half-built KParams behind)
    c->has_scene = false;
    KParams& k = c->kp;
    std::memset(&k, 0, sizeof k);
    k.mass = s->mass;
    k.M3 = 3.0 * s->mass;
    std::memcpy(k.center, s->center, sizeof k.center);
    k.u_cap = s->mass > 0.0 ? 1.0 / (2.0 * s->mass) : INFINITY;
    k.u_esc = 1.0 / s->escape_radius;
    k.escape_radius = s->escape_radius;
    k.phi_max = 2.0 * kPi * s->max_windings;
    k.max_windings = s->max_windings;
    k.integrator = s->integrator;
    std::memcpy(k.cam_pos, s->cam_pos, sizeof k.cam_pos);
    {  // per-frame constants of plane_basis / initial_conditions (geodesic.cpp:49-65)
        const HV3 v = hsub(hv(s->cam_pos), hv(s->center));
        hput(k.cam_v, v);
        hput(k.cam_e1, hnormalized(v));
        k.cam_r0 = hnorm(v);
        k.cam_u0 = 1.0 / k.cam_r0;
    }
    HV3 f, r, u;
    camera_basis(s, f, r, u);
    hput(k.forward, f);
    hput(k.right, r);
    hput(k.up, u);
    k.tan_half_y = std::tan(s->vertical_fov / 2.0);  // camera.cpp:46-48
    const double aspect = static_cast<double>(s->width) / s->height;
    k.tan_half_x = k.tan_half_y * aspect;
    k.inv_width = 1.0 / s->width;  // camera_ray: (px + sx) / width by reciprocal + fma correction
    k.inv_height = 1.0 / s->height;
    k.inv_spp = 1.0 / s->spp;
    k.div_magic = s->width >= 2 ? ~0ull / static_cast<unsigned long long>(s->width) + 1ull : 0ull;
    k.width = s->width;
    k.height = s->height;
    k.spp = s->spp;
    k.seed = s->seed;
    {  // camera.cpp:12-17 splitmix64 of the seed (hash_counter's first round)
        uint64_t x = s->seed + 0x9e3779b97f4a7c15ULL;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
        k.seed_mix = x ^ (x >> 31);
    }
    k.epsilon = s->epsilon;
    k.rel_tol = s->rel_tol;
    k.abs_tol = s->abs_tol;
    k.ref_pow_prev0 = std::pow(1e-4, 0.4 / 5.0);  // host libm, as the reference
    k.step = s->step;
    k.max_step = s->max_step;
    k.chord_dphi = s->chord_dphi;
    k.sky_kind = s->sky_kind;
    k.checker_nu = s->checker_nu;
    k.checker_nv = s->checker_nv;
    double checker[3 * kCheckerMax];  // cell boundaries (shade_sample), uploaded below
    for (int i = 0; i < kCheckerMax; ++i) {
        const double th = -kPi + 2.0 * kPi * i / (s->checker_nu > 0 ? s->checker_nu : 1);
        checker[i] = std::cos(th);
        checker[kCheckerMax + i] = std::sin(th);
        checker[2 * kCheckerMax + i] = std::cos(kPi * i / (s->checker_nv > 0 ? s->checker_nv : 1));
    }
    std::memcpy(k.checker_a, s->checker_color_a, sizeof k.checker_a);
    std::memcpy(k.checker_b, s->checker_color_b, sizeof k.checker_b);
    k.disk_enabled = s->disk_enabled;
    k.disk_r_in = s->disk_r_in;
    k.disk_r_out = s->disk_r_out;
    k.disk_inv_width = 1.0 / (s->disk_r_out - s->disk_r_in);
    std::memcpy(k.disk_c_in, s->disk_color_in, sizeof k.disk_c_in);
    std::memcpy(k.disk_c_out, s->disk_color_out, sizeof k.disk_c_out);
    k.n_spheres = s->n_spheres;
    hput(k.light, hnormalized(hv(s->light_dir)));
    k.ambient = s->ambient;
    // host data -> pinned staging -> device (async on the upload stream)
    const size_t sky_bytes = s->sky_kind == BHRT_SKY_IMAGE ? 3ull * s->sky_width * s->sky_height : 0;
    const size_t sph_bytes = sizeof(bhrt_sphere) * static_cast<size_t>(s->n_spheres);
    const bool cull = s->n_spheres > 0 && cull_basis(s, k);
    const size_t chk_bytes = sizeof checker;
    const size_t need = chk_bytes + sky_bytes + sph_bytes;
    c->upload_bytes = need;
    if (need > c->staging_cap) {
        if (c->staging) CK(cudaFreeHost(c->staging));
        c->staging = nullptr;
        c->staging_cap = 0;
        CK(cudaMallocHost(&c->staging, need));
        c->staging_cap = need;
    }
    size_t off = 0;
    if (c->checker.ensure(3 * kCheckerMax)) return set_info(info, BHRT_DEVICE, -1, -1, "checker alloc failed");
    std::memcpy(c->staging + off, checker, chk_bytes);
    CK(cudaMemcpyAsync(c->checker.p, c->staging + off, chk_bytes, cudaMemcpyHostToDevice, c->up_stream));
    off += chk_bytes;
    k.checker_tab = c->checker.p;
    if (sky_bytes) {
        if (c->sky.ensure(sky_bytes)) return set_info(info, BHRT_DEVICE, -1, -1, "sky alloc failed");
        std::memcpy(c->staging + off, s->sky_rgb, sky_bytes);
        CK(cudaMemcpyAsync(c->sky.p, c->staging + off, sky_bytes, cudaMemcpyHostToDevice, c->up_stream));
        off += sky_bytes;
        k.sky = c->sky.p;
        k.sky_w = s->sky_width;
        k.sky_h = s->sky_height;
    }
    if (s->n_spheres > 0) {
        if (c->spheres.ensure(s->n_spheres)) return set_info(info, BHRT_DEVICE, -1, -1, "sphere alloc failed");
        std::memcpy(c->staging + off, s->spheres, sph_bytes);
        CK(cudaMemcpyAsync(c->spheres.p, c->staging + off, sph_bytes, cudaMemcpyHostToDevice, c->up_stream));
        off += sph_bytes;
        k.spheres = c->spheres.p;
        if (cull) {  // the candidate lists, from the spheres just uploaded
            if (c->cull.ensure(2 * static_cast<size_t>(kCullBins)))
                return set_info(info, BHRT_DEVICE, -1, -1, "cull alloc failed");
            k.cull = c->cull.p;
            launch_cull_build(k, c->cull.p, c->up_stream);
            CK(cudaGetLastError());
        }
    }
    k.fused_shade = (32 % s->spp) == 0 ? 1 : 0;
    k.grow = c->tables.p;
    k.shrink = c->tables.p + kQN;
    if (s->integrator == BHRT_INTEGRATOR_TABLE) {
        // The b-table depends only on these fields; rebuild only when they change.
        const double key[10] = {s->mass, s->rel_tol, s->abs_tol, s->step, s->max_step,
                                (double)s->table_entries, (double)s->table_samples, s->table_b_max,
                                s->table_dpsi, s->escape_radius};
        k.table_entries = s->table_entries;
        k.table_ns = s->table_samples;
        k.table_b_max = s->table_b_max;
        k.table_dpsi = s->table_dpsi;
        k.inv_table_b_max = 1.0 / s->table_b_max;
        k.inv_table_dpsi = 1.0 / s->table_dpsi;
        const size_t E = static_cast<size_t>(s->table_entries);
        if (!c->has_table || std::memcmp(key, c->table_key, sizeof key) != 0) {
            if (c->tab_smp.ensure(E * s->table_samples * 2) || c->tab_ends.ensure(E * 4) ||
                c->tab_kind.ensure(E) || c->tab_n.ensure(E) || c->tab_meta.ensure(4 * E))
                return set_info(info, BHRT_DEVICE, -1, -1, "table alloc failed");
            launch_table_build(k, c->tab_smp.p, c->tab_ends.p, c->tab_kind.p, c->tab_n.p, c->up_stream);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(c->up_stream));
            std::memcpy(c->table_key, key, sizeof key);
            c->has_table = true;
        }
        k.tab_smp = c->tab_smp.p;
        k.tab_ends = c->tab_ends.p;
        k.tab_kind = c->tab_kind.p;
        k.tab_n = c->tab_n.p;
        k.tab_meta = c->tab_meta.p;
        // bind the frame: each entry's inbound psi of the camera's u0 (oracle prep_table)
        const double u0 = 1.0 / hnorm(hsub(hv(s->cam_pos), hv(s->center)));
        launch_table_bind(k, c->tab_ends.p, c->tab_meta.p, u0, c->up_stream);
        CK(cudaGetLastError());
    }
    k.grow = c->tables.p;
    k.shrink = c->tables.p + kQN;
    CK(cudaEventRecord(c->up_done, c->up_stream));  // renders wait on this
    c->scene = *s;
    c->has_scene = true;
    return 0;
}

int bhrt_ctx_render_async(bhrt_ctx* c, int32_t row_start, int32_t row_end, int32_t tile_rows,
                          int32_t tile_stride, int32_t tile_offset, uint8_t* d_out,
                          bhrt_ray_record* d_records, void* stream, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    if (!c || !c->has_scene) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "context has no scene");
    if (row_start < 0 || row_end > c->scene.height || row_start > row_end)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: row range out of bounds");
    const int32_t rows = bhrt_tile_row_count(row_start, row_end, tile_rows, tile_stride, tile_offset);
    if (rows < 0) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: bad tiling");
    if (rows > 0 && d_out == nullptr) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: NULL output");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    KParams k = c->kp;
    k.row_start = row_start;
    k.row_end = row_end;
    k.tile_rows = tile_rows;
    k.tile_stride = tile_stride;
    k.tile_offset = tile_offset;
    k.n_rows = rows;
    const size_t nrec = static_cast<size_t>(rows) * k.width * k.spp;
    RecSlot* slot = nullptr;
    if (!d_records && !k.fused_shade && rows > 0) {  // unfused shading reads the records
        bool not_ready = false;
        for (RecSlot* r : c->rec_pool) {
            const cudaError_t q = cudaEventQuery(r->done);
            if (q == cudaSuccess) {
                slot = r;
                break;
            }
            not_ready = not_ready || q == cudaErrorNotReady;
        }
        if (not_ready) (void)cudaGetLastError();  // "not ready" is a status, not an error
        if (!slot && c->rec_pool.size() < kRecSlots) {
            slot = new RecSlot;
            c->rec_pool.push_back(slot);
            CK(cudaEventCreateWithFlags(&slot->done, cudaEventDisableTiming));
        }
        if (!slot) {
            slot = c->rec_pool[c->rec_rr++ % c->rec_pool.size()];
            CK(cudaStreamWaitEvent(st, slot->done, 0));
        }
        if (slot->buf.ensure(nrec)) return set_info(info, BHRT_DEVICE, -1, -1, "records alloc failed");
        d_records = slot->buf.p;
    }
    k.records = d_records;
    k.out = d_out;
    k.out_image = c->out_image;
    k.stats = c->stats.p;
    CK(cudaStreamWaitEvent(st, c->up_done, 0));  // the scene's uploads
    if (!c->in_frame) {  // counters + lowest failing pixel start fresh for this render
        CK(cudaMemcpyAsync(c->stats.p, c->host_slots + kStatWords, kStatBytes,
                           cudaMemcpyHostToDevice, st));
        c->launches = 0;
    }
    c->timed = c->timing && rows > 0;
    if (rows > 0 && launch_trace(k, st, &c->launches, c->timed ? c->ev : nullptr) != 0)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: unsupported integrator");
    CK(cudaGetLastError());
    if (slot) CK(cudaEventRecord(slot->done, st));
    if (c->in_frame) {
        // counters accumulate on the device; finish() reads them once after
        // every render of the frame (its renders may run on several streams)
        if (c->frame_nev == c->frame_ev.size()) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->frame_ev.push_back(e);
        }
        CK(cudaEventRecord(c->frame_ev[c->frame_nev++], st));
    } else {
        CK(cudaMemcpyAsync(c->host_slots, c->stats.p, kStatBytes, cudaMemcpyDeviceToHost,
                           st));
        CK(cudaEventRecord(c->render_done, st));
    }
    c->last_stream = st;
    c->pending = 1;
    c->last_rows = rows;
    c->kp.row_start = row_start;  // remembered for failure mapping
    c->kp.row_end = row_end;
    c->kp.tile_rows = tile_rows;
    c->kp.tile_stride = tile_stride;
    c->kp.tile_offset = tile_offset;
    c->kp.n_rows = rows;
    return 0;
}

int bhrt_ctx_set_output_layout(bhrt_ctx* c, int32_t image_layout) {
    if (!c || image_layout < 0 || image_layout > 1) return BHRT_INVALID_ARGUMENT;
    c->out_image = image_layout;
    return 0;
}

int bhrt_device_alloc(int32_t device, size_t bytes, void** d_ptr, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    if (!d_ptr) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "NULL output pointer");
    CK(cudaSetDevice(device));
    CK(cudaMalloc(d_ptr, bytes ? bytes : 1));
    return 0;
}

int bhrt_device_free(int32_t device, void* d_ptr) {
    bhrt_status_info* info = nullptr;
    CK(cudaSetDevice(device));
    CK(cudaFree(d_ptr));
    return 0;
}

int bhrt_ipc_export(int32_t device, void* d_ptr, uint8_t handle[64], bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, d_ptr));
    std::memcpy(handle, &h, sizeof h);
    return 0;
}

int bhrt_ipc_open(int32_t device, const uint8_t handle[64], void** d_ptr, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    CK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}

int bhrt_ipc_close(int32_t device, void* d_ptr) {
    bhrt_status_info* info = nullptr;
    CK(cudaSetDevice(device));
    CK(cudaIpcCloseMemHandle(d_ptr));
    return 0;
}

int bhrt_ctx_frame_begin(bhrt_ctx* c, void* stream, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    if (!c || !c->has_scene) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "context has no scene");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(cudaMemcpyAsync(c->stats.p, c->host_slots + kStatWords, kStatBytes, cudaMemcpyHostToDevice,
                       st));
    c->launches = 0;
    c->in_frame = true;
    c->frame_nev = 0;
    return 0;
}

// Counter slots (kStatSlots, kernel side warp_add_stats) -> the 8 counters:
// sums, except the lowest failing pixel (slot 0 only, atomicMin).
static void fold_stats(bhrt_ctx* c) {
    for (int w = 0; w < 8; ++w) c->stats_sum[w] = c->host_slots[w];
    for (int s = 1; s < kStatSlots; ++s)
        for (int w = 0; w < 8; ++w)
            if (w != 3) c->stats_sum[w] += c->host_slots[kStatStride * s + w];
}

// The reference's failure text for the lowest failing pixel (render.cpp:36-40
// forwards e.what(): geodesic.cpp:234 "trace: inverse radius left the
// positive domain", or StepSizeUnderflow's "adaptive step size underflow near
// u = <u>", geodesic.hpp:72-74). The frame's kernels only flag the pixel; on
// failure its row is traced once more with records (cold path), whose
// failing samples carry (u, kind) in point[0..1], and the first failing
// sample in sample order (shade_pixel's loop, render.cpp:25) names the error.
static void failure_text(bhrt_ctx* c, int px, int py, char* out, size_t cap) {
    std::snprintf(out, cap, "numerical failure");
    KParams k = c->kp;
    const size_t nrec = static_cast<size_t>(k.width) * k.spp;
    DevBuf<bhrt_ray_record> rec;
    DevBuf<uint8_t> img;
    if (rec.ensure(nrec) || img.ensure(3 * static_cast<size_t>(k.width))) {
        rec.release();
        img.release();
        (void)cudaGetLastError();
        return;
    }
    k.row_start = py;
    k.row_end = py + 1;
    k.tile_rows = 1;
    k.tile_stride = 1;
    k.tile_offset = 0;
    k.n_rows = 1;
    k.records = rec.p;
    k.out = img.p;
    k.out_image = 0;
    k.stats = c->stats.p;  // the frame's counters are already on the host
    k.diag = 1;            // the diagnostic kernel instantiations
    std::vector<bhrt_ray_record> h(k.spp);
    int launches = 0;
    bool ok = cudaMemcpyAsync(c->stats.p, c->host_slots + kStatWords, kStatBytes,
                              cudaMemcpyHostToDevice, c->up_stream) == cudaSuccess &&
              launch_trace(k, c->up_stream, &launches, nullptr) == 0 &&
              cudaMemcpyAsync(h.data(), rec.p + static_cast<size_t>(px) * k.spp,
                              sizeof(bhrt_ray_record) * k.spp, cudaMemcpyDeviceToHost,
                              c->up_stream) == cudaSuccess &&
              cudaStreamSynchronize(c->up_stream) == cudaSuccess;
    rec.release();
    img.release();
    if (!ok) {
        (void)cudaGetLastError();
        return;
    }
    for (const bhrt_ray_record& r : h) {
        if (r.object != -BHRT_NUMERICAL) continue;
        if (r.point[1] == 2.0)
            std::snprintf(out, cap, "adaptive step size underflow near u = %f", r.point[0]);
        else
            std::snprintf(out, cap, "trace: inverse radius left the positive domain");
        return;
    }
}

int bhrt_ctx_finish(bhrt_ctx* c, bhrt_status_info* info) {
    set_info(info, 0, -1, -1, "");
    if (!c) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "NULL context");
    CK(cudaSetDevice(c->device));
    if (c->in_frame && c->pending) {
        for (size_t i = 0; i < c->frame_nev; ++i) CK(cudaEventSynchronize(c->frame_ev[i]));
        CK(cudaMemcpyAsync(c->host_slots, c->stats.p, kStatBytes, cudaMemcpyDeviceToHost,
                           c->up_stream));
        CK(cudaStreamSynchronize(c->up_stream));
        CK(cudaEventRecord(c->render_done, c->up_stream));
    }
    c->frame_nev = 0;
    c->in_frame = false;
    if (!c->pending) return 0;
    CK(cudaEventSynchronize(c->render_done));  // this render only, not later work on the stream
    c->pending = 0;
    fold_stats(c);
    const unsigned long long fail = c->stats_sum[3];  // lowest failing y * width + x
    if (fail != ULLONG_MAX) {
        const int py = static_cast<int>(fail / c->kp.width);
        const int px = static_cast<int>(fail % c->kp.width);
        char what[96], msg[160];
        failure_text(c, px, py, what, sizeof what);
        std::snprintf(msg, sizeof msg, "pixel (%d, %d): %s", px, py, what);  // RenderError, render.hpp:43-46
        return set_info(info, BHRT_NUMERICAL, px, py, msg);
    }
    return 0;
}

int bhrt_ctx_upload_bytes(bhrt_ctx* c, uint64_t* staged, uint64_t* params_per_launch, uint64_t* counter_bytes) {
    if (!c) return BHRT_INVALID_ARGUMENT;
    if (staged) *staged = c->upload_bytes;
    if (params_per_launch) *params_per_launch = sizeof(KParams);
    if (counter_bytes) *counter_bytes = kStatBytes;
    return 0;
}

int bhrt_ctx_counters(bhrt_ctx* c, uint64_t out[8]) {
    if (!c) return BHRT_INVALID_ARGUMENT;
    for (int i = 0; i < 8; ++i) out[i] = c->stats_sum[i];
    return 0;
}

int bhrt_ctx_stats(bhrt_ctx* c, uint64_t* steps, uint64_t* rejected, uint64_t* rays, int32_t* launches) {
    if (!c) return BHRT_INVALID_ARGUMENT;
    if (steps) *steps = c->stats_sum[0];
    if (rejected) *rejected = c->stats_sum[1];
    if (rays) *rays = c->stats_sum[2];
    if (launches) *launches = c->launches;
    return 0;
}

}  // extern "C"

namespace {
std::mutex g_ctx_mu;
std::map<int, bhrt_ctx*> g_ctx;  // one cached context per device for the one-shot API

int cached_ctx(int dev, bhrt_ctx** out, bhrt_status_info* info) {
    auto it = g_ctx.find(dev);
    if (it != g_ctx.end()) {
        *out = it->second;
        return 0;
    }
    const int rc = bhrt_ctx_create(dev, out, info);
    if (rc == 0) g_ctx[dev] = *out;
    return rc;
}
}  // namespace

// The one-shot path without records (what render_rows callers use,
// render.cpp:68-119). Per device: the scene upload (async, pinned staging),
// then the device's cyclic rows of each of B row bands (edges on multiples of
// G rows, so a band's packed rows are a contiguous run of the whole range's
// packed order) rendered on alternating streams — a band's kernel fills the
// SMs while the previous band's longest blocks drain — and copied to pinned
// staging on a copy stream as soon as the band is done. The host places
// bands into the caller's buffer (unshuffling rows for G > 1) in band order
// while later bands still render/copy, so only the last band's copy and
// placement are exposed. Devices run concurrently; counters and the lowest
// failing pixel come from each context's frame (bhrt_ctx_frame_begin/finish).
static int render_rows_banded(const bhrt_scene* s, int32_t row_start, int32_t row_end, const std::vector<int>& devs,
                       uint8_t* out, bhrt_status_info* info) {
    const int G = static_cast<int>(devs.size());
    const int tile_rows = 1;  // cyclic rows across devices
    const int rows = row_end - row_start;
    const size_t row_bytes = 3ull * s->width;
    // bands: ~0.5 M samples or more each, at most 16 (4K x 4 spp: 16 bands)
    const long long samples = static_cast<long long>(rows) * s->width * s->spp;
    int B = static_cast<int>(std::min<long long>(16, std::max<long long>(1, samples / (1ll << 19))));
    B = std::min(B, std::max(1, rows / G));
    std::vector<int32_t> edge(B + 1);
    for (int b = 0; b <= B; ++b) {
        const long long e = static_cast<long long>(rows) * b / B;
        edge[b] = b == B ? row_end : row_start + static_cast<int32_t>(e - e % G);
    }
    std::vector<bhrt_ctx*> ctxs(G);
    std::vector<std::vector<int32_t>> boff(G, std::vector<int32_t>(B + 1, 0));  // packed row offsets
    for (int g = 0; g < G; ++g) {
        int rc = cached_ctx(devs[g], &ctxs[g], info);
        if (rc) return rc;
        bhrt_ctx* c = ctxs[g];
        rc = bhrt_ctx_set_scene(c, s, info);
        if (rc) return rc;
        CK(cudaSetDevice(c->device));
        if (!c->copy_stream) {
            for (auto& st : c->band_stream) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        }
        while (c->band_ev.size() < 2ull * B + 1) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->band_ev.push_back(e);
        }
        for (int b = 0; b < B; ++b)
            boff[g][b + 1] = boff[g][b] + bhrt_tile_row_count(edge[b], edge[b + 1], tile_rows, G, g);
        const size_t bytes = row_bytes * boff[g][B];
        if (c->out.ensure(bytes + 1)) return set_info(info, BHRT_DEVICE, -1, -1, "output alloc failed");
        if (bytes > c->host_out_cap) {
            if (c->host_out) CK(cudaFreeHost(c->host_out));
            c->host_out = nullptr;
            c->host_out_cap = 0;
            CK(cudaMallocHost(&c->host_out, bytes));
            c->host_out_cap = bytes;
        }
        rc = bhrt_ctx_frame_begin(c, c->band_stream[0], info);
        if (rc) return rc;
        CK(cudaEventRecord(c->band_ev[2 * B], c->band_stream[0]));  // the counters' reset
        CK(cudaStreamWaitEvent(c->band_stream[1], c->band_ev[2 * B], 0));
        for (int b = 0; b < B; ++b) {
            const int32_t nb = boff[g][b + 1] - boff[g][b];
            if (nb == 0) continue;
            cudaStream_t st = c->band_stream[b % 2];
            rc = bhrt_ctx_render_async(c, edge[b], edge[b + 1], tile_rows, G, g,
                                       c->out.p + row_bytes * boff[g][b], nullptr, st, info);
            if (rc) return rc;
            CK(cudaEventRecord(c->band_ev[2 * b], st));
            CK(cudaStreamWaitEvent(c->copy_stream, c->band_ev[2 * b], 0));
            CK(cudaMemcpyAsync(c->host_out + row_bytes * boff[g][b], c->out.p + row_bytes * boff[g][b],
                               row_bytes * nb, cudaMemcpyDeviceToHost, c->copy_stream));
            CK(cudaEventRecord(c->band_ev[2 * b + 1], c->copy_stream));
        }
    }
    // place the bands as they land (band-major, so every device's copy of a
    // band overlaps the placement of the previous one)
    for (int b = 0; b < B; ++b) {
        for (int g = 0; g < G; ++g) {
            bhrt_ctx* c = ctxs[g];
            const int32_t nb = boff[g][b + 1] - boff[g][b];
            if (nb == 0) continue;
            CK(cudaSetDevice(c->device));
            CK(cudaEventSynchronize(c->band_ev[2 * b + 1]));
            const unsigned char* src = c->host_out + row_bytes * boff[g][b];
            if (G == 1) {
                std::memcpy(out + row_bytes * (edge[b] - row_start), src, row_bytes * nb);
            } else {
                for (int j = 0; j < nb; ++j)  // band rows edge[b] + g + j G
                    std::memcpy(out + row_bytes * (edge[b] + g + static_cast<int64_t>(j) * G - row_start),
                                src + row_bytes * j, row_bytes);
            }
        }
    }
    int first_fail = 0;
    long long fail_key = LLONG_MAX;
    bhrt_status_info tmp;
    for (int g = 0; g < G; ++g) {
        const int r = bhrt_ctx_finish(ctxs[g], &tmp);
        if (r == BHRT_NUMERICAL) {
            const long long key = static_cast<long long>(tmp.py) * s->width + tmp.px;
            if (key < fail_key) {
                fail_key = key;
                if (info) *info = tmp;
                first_fail = r;
            }
        } else if (r) {
            if (info) *info = tmp;
            return r;
        }
    }
    return first_fail;
}

extern "C" int bhrt_cuda_render_rows(const bhrt_scene* s, int32_t row_start, int32_t row_end,
                                     const int32_t* devices, int32_t ndev, uint8_t* out,
                                     size_t out_len, bhrt_ray_record* records,
                                     bhrt_status_info* info) {
    // render.cpp:68-75 validation order: scene, then arguments.
    int rc = bhrt_validate_scene(s, info);
    if (rc) return rc;
    if (row_start < 0 || row_end > s->height || row_start > row_end)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: row range out of bounds");
    const size_t need = 3ull * static_cast<size_t>(row_end - row_start) * s->width;
    if (out_len < need || (need > 0 && out == nullptr))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: output buffer too small");
    if (row_end == row_start) return 0;
    rc = validate_trace(s, info);
    if (rc) return rc;

    std::lock_guard<std::mutex> lock(g_ctx_mu);
    std::vector<int> devs;
    if (!devices || ndev <= 0) {
        int d = 0;
        CK(cudaGetDevice(&d));
        devs.push_back(d);
    } else {
        devs.assign(devices, devices + ndev);
        for (int i = 0; i < ndev; ++i) {  // one cached context per device: each device once
            bool bad = devs[i] < 0;
            for (int j = 0; j < i; ++j) bad = bad || devs[i] == devs[j];
            if (bad) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "render: duplicate or negative device");
        }
    }
    const int G = static_cast<int>(devs.size());
    const int tile_rows = 1;  // cyclic rows (7.78x vs 6.35x for bands)
    std::vector<bhrt_ctx*> ctxs(G);
    std::vector<int32_t> nrows(G);
    if (!records) return render_rows_banded(s, row_start, row_end, devs, out, info);
    for (int g = 0; g < G; ++g) {
        rc = cached_ctx(devs[g], &ctxs[g], info);
        if (rc) return rc;
        rc = bhrt_ctx_set_scene(ctxs[g], s, info);
        if (rc) return rc;
        nrows[g] = bhrt_tile_row_count(row_start, row_end, tile_rows, G, g);
        if (ctxs[g]->out.ensure(3ull * nrows[g] * s->width + 1))
            return set_info(info, BHRT_DEVICE, -1, -1, "output alloc failed");
        bhrt_ray_record* d_rec = nullptr;
        if (records) {
            if (ctxs[g]->records.ensure(static_cast<size_t>(nrows[g]) * s->width * s->spp))
                return set_info(info, BHRT_DEVICE, -1, -1, "records alloc failed");
            d_rec = ctxs[g]->records.p;
        }
        rc = bhrt_ctx_render_async(ctxs[g], row_start, row_end, tile_rows, G, g, ctxs[g]->out.p,
                                   d_rec, nullptr, info);
        if (rc) return rc;
    }
    int first_fail = 0;
    long long fail_key = LLONG_MAX;
    bhrt_status_info tmp;
    for (int g = 0; g < G; ++g) {
        const int r = bhrt_ctx_finish(ctxs[g], &tmp);
        if (r == BHRT_NUMERICAL) {
            const long long key = static_cast<long long>(tmp.py) * s->width + tmp.px;
            if (key < fail_key) {
                fail_key = key;
                if (info) *info = tmp;
                first_fail = r;
            }
        } else if (r) {
            if (info) *info = tmp;
            return r;
        }
    }
    if (first_fail) return first_fail;
    const size_t row_bytes = 3ull * s->width;
    for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(devs[g]));
        if (G == 1) {
            CK(cudaMemcpy(out, ctxs[g]->out.p, row_bytes * nrows[g], cudaMemcpyDeviceToHost));
        } else {
            std::vector<uint8_t> stage(row_bytes * nrows[g]);
            CK(cudaMemcpy(stage.data(), ctxs[g]->out.p, stage.size(), cudaMemcpyDeviceToHost));
            for (int j = 0; j < nrows[g]; ++j) {
                const int y = packed_row_to_y(ctxs[g]->kp, j);
                std::memcpy(out + row_bytes * (y - row_start), stage.data() + row_bytes * j, row_bytes);
            }
        }
        if (records) {
            const size_t per_row = static_cast<size_t>(s->width) * s->spp;
            std::vector<bhrt_ray_record> stage(per_row * nrows[g]);
            CK(cudaMemcpy(stage.data(), ctxs[g]->records.p, sizeof(bhrt_ray_record) * stage.size(),
                          cudaMemcpyDeviceToHost));
            for (int j = 0; j < nrows[g]; ++j) {
                const int y = packed_row_to_y(ctxs[g]->kp, j);
                std::memcpy(records + per_row * (y - row_start), stage.data() + per_row * j,
                            sizeof(bhrt_ray_record) * per_row);
            }
        }
    }
    return 0;
}

// trace() / deflection_of_ray() for a batch of caller rays.
namespace {
int trace_batch_prepare(const bhrt_scene* s, const double* rays, int64_t n, bhrt_status_info* info) {
    // trace(): validate(cfg) (geodesic.cpp:19-27) then the mass (:167)
    if (!(s->epsilon > 0.0))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: epsilon must be > 0");
    if (!(s->escape_radius > 0.0))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: escape_radius must be > 0");
    if (s->max_windings < 1)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: max_windings must be >= 1");
    if (!(s->rel_tol > 0.0))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: rel_tol must be > 0");
    if (!(s->abs_tol > 0.0))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace config: abs_tol must be > 0");
    if (s->mass < 0.0) return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace: mass must be >= 0");
    if (s->integrator != BHRT_INTEGRATOR_REFERENCE)
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace_rays: integrator must be REFERENCE");
    for (int64_t i = 0; i < n; ++i) {  // geodesic.cpp:169-172
        const HV3 v = hsub(hv(rays + 6 * i), hv(s->center));
        if (s->mass > 0.0 && hnorm(v) <= 2.0 * s->mass)
            return set_info(info, BHRT_INVALID_ARGUMENT, static_cast<int>(i), -1,
                            "trace: ray origin is not outside the event horizon");
    }
    return 0;
}

KParams trace_batch_params(const bhrt_scene* s) {
    KParams k;
    std::memset(&k, 0, sizeof k);
    k.mass = s->mass;
    k.M3 = 3.0 * s->mass;
    std::memcpy(k.center, s->center, sizeof k.center);
    k.u_cap = s->mass > 0.0 ? 1.0 / (2.0 * s->mass) : INFINITY;
    k.u_esc = 1.0 / s->escape_radius;
    k.escape_radius = s->escape_radius;
    k.phi_max = 2.0 * kPi * s->max_windings;
    k.max_windings = s->max_windings;
    k.integrator = s->integrator;
    k.epsilon = s->epsilon;
    k.rel_tol = s->rel_tol;
    k.abs_tol = s->abs_tol;
    k.ref_pow_prev0 = std::pow(1e-4, 0.4 / 5.0);  // host libm, as the reference
    return k;
}

int trace_batch_failures(const bhrt_ray_record* records, int64_t n, bhrt_status_info* info) {
    for (int64_t i = 0; i < n; ++i)
        if (records[i].object == -BHRT_NUMERICAL)
            return set_info(info, BHRT_NUMERICAL, static_cast<int>(i), -1,
                            "trace: inverse radius left the positive domain or step underflow");
    return 0;
}
}  // namespace

extern "C" int bhrt_cuda_trace_rays(const bhrt_scene* s, const double* rays, int64_t n, int32_t device,
                                    bhrt_ray_record* records, double* deflection,
                                    bhrt_status_info* info) {
    if (!s || n < 0 || (n > 0 && (!rays || !records)))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace_rays: bad arguments");
    int rc = trace_batch_prepare(s, rays, n, info);
    if (rc) return rc;
    if (n == 0) return 0;
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    int dev = device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    bhrt_ctx* c = nullptr;
    rc = cached_ctx(dev, &c, info);
    if (rc) return rc;
    CK(cudaSetDevice(dev));
    if (c->rays.ensure(6 * static_cast<size_t>(n)) || c->records.ensure(static_cast<size_t>(n)) ||
        (deflection && c->defl.ensure(static_cast<size_t>(n))))
        return set_info(info, BHRT_DEVICE, -1, -1, "trace_rays: alloc failed");
    const KParams k = trace_batch_params(s);
    CK(cudaMemcpy(c->rays.p, rays, sizeof(double) * 6 * n, cudaMemcpyHostToDevice));
    launch_trace_rays(k, c->rays.p, n, c->records.p, deflection ? c->defl.p : nullptr, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(records, c->records.p, sizeof(bhrt_ray_record) * n, cudaMemcpyDeviceToHost));
    if (deflection) CK(cudaMemcpy(deflection, c->defl.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return trace_batch_failures(records, n, info);
}

// trace()'s RayPolyline for a batch of caller rays (geodesic.hpp:62-65,107-108).
extern "C" int bhrt_cuda_trace_polylines(const bhrt_scene* s, const double* rays, int64_t n, int32_t device,
                                         int32_t max_points, double* points, int32_t* npoints,
                                         bhrt_ray_record* records, bhrt_status_info* info) {
    if (!s || n < 0 || max_points < 0 || (n > 0 && (!rays || !records || !npoints)) ||
        (n > 0 && max_points > 0 && !points))
        return set_info(info, BHRT_INVALID_ARGUMENT, -1, -1, "trace_polylines: bad arguments");
    int rc = trace_batch_prepare(s, rays, n, info);
    if (rc) return rc;
    if (n == 0) return 0;
    const size_t npts = static_cast<size_t>(n) * static_cast<size_t>(max_points) * 3;
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    int dev = device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    bhrt_ctx* c = nullptr;
    rc = cached_ctx(dev, &c, info);
    if (rc) return rc;
    CK(cudaSetDevice(dev));
    if (c->rays.ensure(6 * static_cast<size_t>(n)) || c->records.ensure(static_cast<size_t>(n)) ||
        c->poly_n.ensure(static_cast<size_t>(n)) || (npts > 0 && c->poly_pts.ensure(npts)))
        return set_info(info, BHRT_DEVICE, -1, -1, "trace_polylines: alloc failed");
    const KParams k = trace_batch_params(s);
    CK(cudaMemcpy(c->rays.p, rays, sizeof(double) * 6 * n, cudaMemcpyHostToDevice));
    launch_trace_polylines(k, c->rays.p, n, c->records.p, npts > 0 ? c->poly_pts.p : nullptr, max_points,
                           c->poly_n.p, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(records, c->records.p, sizeof(bhrt_ray_record) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(npoints, c->poly_n.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    if (npts > 0) CK(cudaMemcpy(points, c->poly_pts.p, sizeof(double) * npts, cudaMemcpyDeviceToHost));
    return trace_batch_failures(records, n, info);
}
