// Kernel parameter block shared by host (bhrt_cuda.cu) and device (trace.cu).
// Everything per-frame that the reference recomputes per ray (camera basis,
// tan(fov/2): camera.cpp:46-48,67) is hoisted here once on the host with the
// reference's own operation order, so the device sees bit-identical values.
#pragma once

#include <cstddef>
#include <cstdint>

#include "bhrt_cuda.h"

namespace bhrt_b200 {

constexpr int kCullSlots = 8;  // candidate spheres kept per ray (more: test all)

// Candidate spheres of one (plane-angle bin, orientation): 144 bytes.
struct alignas(16) CullList {
    int32_t n;                  // candidates (<= kCullSlots); -1: more, test every sphere
    float next_lo;              // smallest window start
    uint8_t k[kCullSlots];      // sphere indices, increasing
    float win[kCullSlots][4];   // (lo, hi) unwrapped window angle, (rlo, rhi) radial extent
};
// the scene kernel reads (n, next_lo, k) as one int4 and the windows as float4s
static_assert(offsetof(CullList, k) == 8 && offsetof(CullList, win) == 16 && sizeof(CullList) == 144,
              "CullList layout");

// Render counters: kStatSlots copies of the 8 counter words, kStatStride
// words apart (own 128-byte line each). Warps add their steps / rejections /
// rays to slot blockIdx mod kStatSlots; the lowest failing pixel and the
// diagnostic counters live in slot 0; the host folds the slots after the
// render (one same-address atomic stream per warp cost config 3 a quarter of
// its time: 2.36 ms; 1.78 ms without counters, 1.84 ms with the slots).
#ifndef BHRT_STAT_SLOTS
#define BHRT_STAT_SLOTS 16  // 16 / 64 / 256 slots: 1.84 / 1.85 / 1.84 ms (config 3)
#endif
constexpr int kStatSlots = BHRT_STAT_SLOTS;
constexpr int kStatStride = 16;
constexpr int kStatWords = kStatSlots * kStatStride;

constexpr int kQMin = -64;  // RKF45 controller table range
constexpr int kQN = 96;
// Largest q with grow factor 0.9 * 2^(-(q+1)/20) >= 1 (checked against the
// host table by tests/test_abi.py): q + 1 <= -20 log2(1/0.9) = -3.04.
constexpr int kQGrowOne = -5;
constexpr int kMaxSpheres = 256;
constexpr int kMaxCand = 16;
constexpr int kCheckerMax = 64;  // checker cells resolved by threshold search (else atan2/asin)

struct KParams {
    // black hole + termination
    double mass, M3;
    double center[3];
    double u_cap, u_esc, phi_max, escape_radius;
    int32_t max_windings;
    int32_t integrator;
    // camera (hoisted): v = cam_pos - center, e1 = v/|v|, r0 = |v|, u0 = 1/r0
    double cam_v[3], cam_e1[3], cam_r0, cam_u0;
    double cam_pos[3];
    double forward[3], right[3], up[3];
    double tan_half_x, tan_half_y;
    double inv_width, inv_height;  // RN(1/width), RN(1/height)
    double inv_spp;                // 1.0 / spp (render.cpp:42)
    unsigned long long div_magic;  // floor(2^64 / width) + 1 for width >= 2, else 0 (sample_of row division)
    int32_t width, height, spp;
    int32_t diag;  // 1: failed samples carry (u, kind) in their record (bhrt_cuda.cu failure_text)
    uint64_t seed;
    uint64_t seed_mix;  // splitmix64(seed): hash_counter's first round (camera.cpp:21-28), per frame
    // integrator
    double epsilon, rel_tol, abs_tol, step, max_step, chord_dphi;
    // mode R: pow(1e-4, 0.4 / 5) with the HOST libm, i.e. the value the
    // reference's PI factor uses on the first step of every window, where
    // err_prev = 1e-4 (geodesic.cpp:107,144-151)
    double ref_pow_prev0;
    // rows: packed row j -> image row y (see bhrt_ctx_render_async)
    int32_t row_start, row_end, tile_rows, tile_stride, tile_offset, n_rows;
    // sky
    int32_t sky_kind, sky_w, sky_h, checker_nu, checker_nv;
    int32_t pad1;
    const uint8_t* sky;
    double checker_a[3], checker_b[3];
    // cell boundaries (device array, 3 x kCheckerMax): longitude k at
    // atan2 = -pi + 2 pi k / nu as cos [k], sin [kCheckerMax + k]; latitude k
    // at y = cos(pi k / nv) [2 kCheckerMax + k]. In global memory, not in the
    // parameter bank: the per-lane binary search indexes it divergently.
    const double* checker_tab;
    // disk
    int32_t disk_enabled;
    int32_t n_spheres;
    double disk_r_in, disk_r_out;
    double disk_inv_width;  // 1 / (disk_r_out - disk_r_in), the colour ramp's scale (oracle shade)
    double disk_c_in[3], disk_c_out[3];
    // spheres (device arrays)
    const bhrt_sphere* spheres;
    double light[3];
    double ambient;
    // RKF45 factor tables (device)
    const double* grow;
    const double* shrink;
    // Sphere culling by orbital-plane angle. Every orbital plane contains the
    // camera-hole axis v, so planes form a pencil n = s (cos t a + sin t b)
    // (a, b unit, perpendicular to v; s = +-1 the orientation). cull points
    // at 2 * cull_bins CullList records, [2 bin + (s < 0)], built on the
    // device per frame (build_cull_lists_kernel): the CONSERVATIVE candidate
    // spheres of every plane in the bin with their angular windows and
    // radial extents; the exact fp64 tests still decide.
    const void* cull;
    int32_t cull_bins;
    int32_t pad2;
    double cull_a[3], cull_b[3];
    // 1: shade inside the trace kernel (spp divides 32; the spp samples of a
    // pixel are adjacent lanes, summed in sample order by warp shuffles)
    int32_t fused_shade;
    // 0: `out` holds the rendered rows packed in order of y; 1: `out` is the
    // whole image and pixel (x, y) lands at 3 (y width + x) — e.g. a peer
    // GPU's image buffer mapped over NVLink (bhrt_ipc_open), so a rank's rows
    // need no gather
    int32_t out_image;
    // b-table (approximate mode): per entry kind/n, ends
    // {psi_end, u_end, w_end, psi_esc}, (u, u') samples at psi_j = j*dpsi with
    // a fixed stride of table_ns samples, and the frame's inbound psi of u0.
    const double* tab_smp;
    const double* tab_ends;
    const int32_t* tab_kind;
    const int32_t* tab_n;
    const double* tab_meta;  // per frame, 4 doubles per entry: psi0, psi_end, psi_esc, kind | n << 32
    int32_t table_entries, table_ns;
    double table_b_max, table_dpsi;
    double inv_table_b_max, inv_table_dpsi;  // RN(1/.) from the host (exact quotients: table.cu div_by)
    // outputs
    bhrt_ray_record* records;   // n_rows * width * spp
    uint8_t* out;               // n_rows * width * 3
    unsigned long long* stats;  // [0] steps, [1] rejected, [2] rays, [3] lowest failing y*width+x (ULLONG_MAX: none), [4..7] BHRT_COUNTERS
};

__host__ __device__ inline int packed_row_to_y(const KParams& p, int j) {
    if (p.tile_rows == 1) return p.row_start + j * p.tile_stride + p.tile_offset;  // no division
    const int tile = j / p.tile_rows;
    const int within = j - tile * p.tile_rows;
    return p.row_start + (tile * p.tile_stride + p.tile_offset) * p.tile_rows + within;
}

}  // namespace bhrt_b200
