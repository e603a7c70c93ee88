/*
 * bhrt_cuda.h — C ABI of the B200-native Schwarzschild ray-tracing hot path.
 *
 * This is the drop-in boundary for the reference's single choke point
 *
 *   std::vector<uint8_t> bhrt::render_rows(const SceneConfig&, int row_start,
 *                                          int row_end, int threads);
 *       (reference: proj/include/bhrt/render.hpp:60-61, proj/src/render.cpp:68-119)
 *
 * which every caller of the hot path goes through: render_image
 * (render.cpp:125-129), render_band (render.cpp:121-123), the network worker
 * (netrender.cpp:139-140) and the bench harness (bench.cpp:13-22).
 *
 * Rules:
 *   - plain C: PODs, pointers and sizes; no C++ or torch types cross;
 *   - the caller owns every buffer; calls are synchronous unless the name says
 *     `_async` (those enqueue on the caller's CUDA stream);
 *   - every entry point returns a bhrt_status code; failures also fill the
 *     optional bhrt_status_info (message, failing pixel);
 *   - a numerical failure reports the LOWEST (py, px) failing pixel, so the
 *     error is deterministic (the reference reports whichever thread lost the
 *     race first, render.cpp:100-104,117).
 */
#ifndef BHRT_CUDA_H
#define BHRT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BHRT_CUDA_ABI_VERSION 1

/* Status codes. 1..4 are the reference CLI exit codes (errors.hpp:8-9,
 * bhrt.cpp:338-356): UsageError=1, IoError=2, NumericalError=3,
 * ProtocolError=4. std::invalid_argument (render.cpp:71-73,
 * geodesic.cpp:19-27) gets its own code so the C++ shim can rethrow the
 * exact reference exception type. */
typedef enum bhrt_status {
    BHRT_OK = 0,
    BHRT_USAGE = 1,            /* bhrt::UsageError (validate_scene, render.cpp:11-20) */
    BHRT_IO = 2,               /* bhrt::IoError */
    BHRT_NUMERICAL = 3,        /* bhrt::RenderError : NumericalError (render.hpp:39-47) */
    BHRT_PROTOCOL = 4,         /* bhrt::ProtocolError (unused by the hot path) */
    BHRT_DEVICE = 5,           /* CUDA / NCCL failure (no reference counterpart) */
    BHRT_INVALID_ARGUMENT = 6  /* std::invalid_argument */
} bhrt_status;

typedef struct bhrt_status_info {
    int32_t code;       /* bhrt_status */
    int32_t px, py;     /* failing pixel for BHRT_NUMERICAL, else -1 */
    char message[256];
} bhrt_status_info;

/* Integrators. */
typedef enum bhrt_integrator {
    /* The reference algorithm: DOPRI5(4)+PI control inside epsilon-windows,
     * window-end termination tests, last-chord escape direction
     * (geodesic.cpp:84-162,164-238). Sky only (the reference has no disk or
     * spheres). Arithmetic follows the reference's non-FMA build. */
    BHRT_INTEGRATOR_REFERENCE = 0,
    /* Fixed-step classical RK4, the reference's test oracle
     * (tests/oracles.hpp:23-30,42-55), as a renderer. */
    BHRT_INTEGRATOR_RK4 = 1,
    /* Adaptive Runge-Kutta-Fehlberg 4(5), local extrapolation. */
    BHRT_INTEGRATOR_RKF45 = 2,
    /* Approximate mode: per-ray lookup in a deflection/trajectory table over
     * the impact parameter b, built by RKF45. */
    BHRT_INTEGRATOR_TABLE = 3
} bhrt_integrator;

typedef enum bhrt_sky_kind {
    BHRT_SKY_IMAGE = 0,   /* equirectangular RGB8 image, bilinear (image.cpp:131-169) */
    BHRT_SKY_CHECKER = 1  /* procedural lon/lat checkerboard */
} bhrt_sky_kind;

/* Opaque Lambertian sphere. */
typedef struct bhrt_sphere {
    double center[3];
    double radius;
    double albedo[3];
} bhrt_sphere;

/*
 * Scene. The first block restates the reference SceneConfig field by field
 * (render.hpp:16-22: BlackHole geodesic.hpp:14-19, Camera camera.hpp:12-18,
 * SampleSpec camera.hpp:30-33, TraceConfig geodesic.hpp:39-45, background
 * ImageBuffer image.hpp:31-57). The second block holds the north-star
 * extensions that have no reference counterpart; bhrt_scene_defaults()
 * fills them so that a scene built from reference fields alone renders
 * exactly what the reference renders.
 */
typedef struct bhrt_scene {
    /* --- reference SceneConfig --- */
    double mass;              /* BlackHole::mass (geometric units, >= 0) */
    double center[3];         /* BlackHole::center */
    double cam_pos[3];        /* Camera::position */
    double cam_look_at[3];    /* Camera::look_at */
    double vertical_fov;      /* Camera::vertical_fov, radians */
    int32_t width;            /* Camera::width */
    int32_t height;           /* Camera::height */
    int32_t spp;              /* SampleSpec::spp */
    int32_t max_windings;     /* TraceConfig::max_windings */
    uint64_t seed;            /* SampleSpec::seed */
    double epsilon;           /* TraceConfig::epsilon (reference integrator only) */
    double escape_radius;     /* TraceConfig::escape_radius */
    double rel_tol;           /* TraceConfig::rel_tol */
    double abs_tol;           /* TraceConfig::abs_tol */
    const uint8_t* sky_rgb;   /* SceneConfig::background pixels, RGB8, row 0 on top (borrowed) */
    int32_t sky_width;
    int32_t sky_height;

    /* --- extensions --- */
    int32_t integrator;       /* bhrt_integrator */
    int32_t sky_kind;         /* bhrt_sky_kind */
    double step;              /* RK4: fixed dphi; RKF45: initial dphi; TABLE: RKF45 initial dphi */
    double max_step;          /* RKF45: cap on dphi */
    double chord_dphi;        /* polyline refinement: max dphi of one chord in hit tests */
    int32_t checker_nu;       /* checkerboard cells in longitude */
    int32_t checker_nv;       /* checkerboard cells in latitude */
    double checker_color_a[3];
    double checker_color_b[3];
    int32_t disk_enabled;     /* equatorial thin disk in the plane y = center.y */
    int32_t n_spheres;
    double disk_r_in;
    double disk_r_out;
    double disk_color_in[3];  /* colour at r_in; linear ramp to disk_color_out at r_out */
    double disk_color_out[3];
    const bhrt_sphere* spheres; /* n_spheres entries (borrowed) */
    double light_dir[3];      /* direction TOWARD the light (normalised by the library) */
    double ambient;           /* Lambert: albedo * (ambient + (1-ambient) * max(0, n.l)) */
    int32_t table_entries;    /* TABLE: number of uniform b samples in [0, table_b_max] */
    int32_t table_samples;    /* TABLE: max trajectory samples per entry */
    double table_b_max;
    double table_dpsi;        /* TABLE: trajectory sample spacing in orbit angle */
} bhrt_scene;

/* Per-sample record for parity checks and flop accounting (optional). */
typedef enum bhrt_object {
    BHRT_OBJ_NONE = 0,
    BHRT_OBJ_HORIZON = 1,     /* captured */
    BHRT_OBJ_SKY = 2,         /* escaped */
    BHRT_OBJ_STALLED = 3,
    BHRT_OBJ_DISK = 4,
    BHRT_OBJ_SPHERE = 5       /* + sphere index in `sphere` */
} bhrt_object;

typedef struct bhrt_ray_record {
    int32_t object;           /* bhrt_object */
    int32_t sphere;           /* sphere index for BHRT_OBJ_SPHERE, else -1 */
    int32_t steps;            /* accepted integrator steps (windows for REFERENCE) */
    int32_t rejected;         /* rejected adaptive steps */
    double point[3];          /* hit point (disk/sphere), escape direction (sky), else 0 */
    double phi;               /* orbital-plane angle at termination */
} bhrt_ray_record;

/* Fills every field with the reference defaults (geodesic.hpp:39-45,
 * camera.hpp:12-33, bhrt.cpp:37-53) and the extension defaults
 * (integrator REFERENCE, image sky, no disk, no spheres). */
void bhrt_scene_defaults(bhrt_scene* scene);

/* Reference-equivalent scene validation (render.cpp:11-20 + trace
 * validation geodesic.cpp:19-27 + camera_basis camera.cpp:30-43). */
int bhrt_validate_scene(const bhrt_scene* scene, bhrt_status_info* info);

/* Seeded sphere field: centres volume-uniform in the shell [shell_min,
 * shell_max] about `center`, radii uniform in [radius_min, radius_max], albedo
 * uniform in [0,1]^3, all from one SplitMix64 stream. Host-side, so GPU and
 * oracle see identical spheres. */
int bhrt_make_spheres(uint64_t seed, int32_t n, const double center[3], double shell_min,
                      double shell_max, double radius_min, double radius_max, bhrt_sphere* out);

/* Contiguous scanline bands, identical to make_bands (render.cpp:51-66). */
int bhrt_make_bands(int32_t height, int32_t workers, int32_t* row_start, int32_t* row_end,
                    int32_t capacity, int32_t* count);

/* ---- one-shot render (host buffers; the drop-in for render_rows) ----
 * Renders rows [row_start, row_end) of the scene into `out` (caller-owned,
 * (row_end-row_start)*width*3 bytes, row-major RGB8). `devices`/`ndev` pick
 * GPUs (NULL/0 = current device); with ndev > 1 rows are split in cyclic
 * tiles across the listed devices from one host thread. `records`, when not
 * NULL, receives (row_end-row_start)*width*spp entries, index
 * ((py-row_start)*width + px)*spp + s. */
int bhrt_cuda_render_rows(const bhrt_scene* scene, int32_t row_start, int32_t row_end,
                          const int32_t* devices, int32_t ndev, uint8_t* out, size_t out_len,
                          bhrt_ray_record* records, bhrt_status_info* info);

/* Scene text: the reference's key=value scene format
 * (config.hpp parse_kv / serialize_scene / parse_scene, config.cpp:27-132)
 * extended with optional keys for the north-star features (integrator, step,
 * max-step, chord-dphi, sky, checker, checker-color-a/b, disk, disk-color-in/
 * out, spheres = count,seed[,shells..], sphere.<i> = cx,cy,cz,r,R,G,B,
 * light-dir, ambient, table-*; full list in csrc/scene_text.cpp).
 * parse: the fourteen reference keys are required, extension keys default to
 * bhrt_scene_defaults; errors are BHRT_USAGE with the reference's messages.
 * Spheres are written to `spheres` (capacity `cap`); *n_spheres receives the
 * count (BHRT_INVALID_ARGUMENT when cap is too small). The background image
 * is not part of the text (as in parse_scene): sky_rgb is left NULL.
 * format: reference keys in serialize_scene order and number format, then
 * only the extension keys that differ from the defaults, so a reference scene
 * formats byte-identically to serialize_scene. *len = text length without
 * the NUL; returns BHRT_INVALID_ARGUMENT when buf is NULL or cap <= *len. */
int bhrt_scene_parse_text(const char* text, bhrt_scene* scene, bhrt_sphere* spheres, int32_t cap,
                          int32_t* n_spheres, bhrt_status_info* info);
int bhrt_scene_format_text(const bhrt_scene* scene, char* buf, size_t cap, size_t* len);

/* Batch form of the reference's per-ray entry points:
 * trace() (geodesic.hpp:107-108, geodesic.cpp:164-238) and, when
 * `deflection` is not NULL, deflection_of_ray() (geodesic.hpp:110-113,
 * geodesic.cpp:240-262), for n caller rays. rays = n x {origin[3], dir[3]}
 * (host, row-major). Uses the scene's mass, center, epsilon, escape_radius,
 * max_windings, rel_tol, abs_tol; camera, samples and sky are ignored; the
 * integrator must be BHRT_INTEGRATOR_REFERENCE. Outcomes instead of
 * polylines: records[i].object = HORIZON (Captured) / SKY (Escaped; point =
 * unit escape direction, the normalised last chord) / STALLED, or
 * -BHRT_NUMERICAL; steps/rejected = DOPRI5 steps; phi = final phi.
 * deflection[i] = |total turning| for escaped rays, NaN otherwise (the
 * reference throws NumericalError there). Errors as the reference's: trace
 * config or mass invalid -> BHRT_INVALID_ARGUMENT; an origin inside the
 * horizon -> BHRT_INVALID_ARGUMENT with info->px = lowest such ray index;
 * numerical failures -> BHRT_NUMERICAL with info->px = lowest failing ray
 * (records are filled for every ray). device < 0: the current device. */
int bhrt_cuda_trace_rays(const bhrt_scene* scene, const double* rays, int64_t n, int32_t device,
                         bhrt_ray_record* records, double* deflection, bhrt_status_info* info);

/* The same batch, also returning each ray's polyline: the reference's
 * trace() RayPolyline::points (geodesic.hpp:62-65,107-108; geodesic.cpp:
 * 164-238): the origin, then every epsilon-window end; radial rays and rays
 * launched beyond the escape radius get the reference's two-point lines.
 * Ray i's first min(npoints[i], max_points) points land at
 * points + 3 * max_points * i (x, y, z doubles); npoints[i] is the full
 * count, so npoints[i] > max_points means truncated — call again with
 * max_points = max(npoints) (max_points = 0 only counts). Window ends are
 * bit-identical to the reference's; the world points use the device cos/sin
 * (within ulps of glibc's). Errors and records as bhrt_cuda_trace_rays. */
int bhrt_cuda_trace_polylines(const bhrt_scene* scene, const double* rays, int64_t n, int32_t device,
                              int32_t max_points, double* points, int32_t* npoints,
                              bhrt_ray_record* records, bhrt_status_info* info);

/* ---- persistent context: scene resident in HBM, async launches ---- */
typedef struct bhrt_ctx bhrt_ctx;

int bhrt_ctx_create(int32_t device, bhrt_ctx** out, bhrt_status_info* info);
void bhrt_ctx_destroy(bhrt_ctx* ctx);
/* Uploads the scene (constants, sky texels, spheres; builds the b-table for
 * BHRT_INTEGRATOR_TABLE). Synchronous. */
int bhrt_ctx_set_scene(bhrt_ctx* ctx, const bhrt_scene* scene, bhrt_status_info* info);
/* Enqueues the render of the rows selected by (row_start, row_end,
 * tile_rows, tile_stride, tile_offset) on `stream` (a cudaStream_t; NULL =
 * legacy default stream): row y is rendered iff row_start <= y < row_end and
 * ((y - row_start) / tile_rows) % tile_stride == tile_offset. Output rows are
 * packed in order of y into `d_out` (device pointer). `d_records`: optional
 * device array, as in bhrt_cuda_render_rows but packed like d_out.
 * Returns immediately. */
int bhrt_ctx_render_async(bhrt_ctx* ctx, int32_t row_start, int32_t row_end, int32_t tile_rows,
                          int32_t tile_stride, int32_t tile_offset, uint8_t* d_out,
                          bhrt_ray_record* d_records, void* stream, bhrt_status_info* info);
/* Opens a frame of several render_async calls (e.g. row bands enqueued back
 * to back so each band's copy-out overlaps the next band's kernel): counters
 * and the lowest failing pixel are reset once here on `stream` and then
 * accumulate over the frame's render_async calls — which may be issued on
 * different streams (e.g. alternating, so one band's kernel fills the SMs
 * while the previous band's last blocks finish) — until bhrt_ctx_finish,
 * which waits for all of them and reports the lowest failing pixel of the
 * whole frame. Without it every render_async starts fresh. */
int bhrt_ctx_frame_begin(bhrt_ctx* ctx, void* stream, bhrt_status_info* info);
/* Waits for the context's last render on its stream and reports the lowest
 * failing pixel, if any. */
int bhrt_ctx_finish(bhrt_ctx* ctx, bhrt_status_info* info);
/* Statistics of the last finished render: accepted steps, rejected steps,
 * rays, kernel launches. */
int bhrt_ctx_stats(bhrt_ctx* ctx, uint64_t* steps, uint64_t* rejected, uint64_t* rays,
                   int32_t* launches);
/* Raw device counters of the last finished render: [0] steps, [1] rejected,
 * [2] rays, [3] lowest failing pixel as y * width + x (UINT64_MAX: none), [4..7]
 * diagnostic counters of builds with -DBHRT_COUNTERS (0 otherwise). */
int bhrt_ctx_counters(bhrt_ctx* ctx, uint64_t out[8]);

/* Host->device bytes of the last bhrt_ctx_set_scene (pinned-staged uploads:
 * checker cell table, sky texels, spheres, sphere cull table), the size of
 * the kernel parameter block each launch carries, and the size of the render
 * counter block (reset host->device before, read device->host after each
 * render or frame). For e2e byte accounting. Any pointer may be NULL. */
int bhrt_ctx_upload_bytes(bhrt_ctx* ctx, uint64_t* staged, uint64_t* params_per_launch,
                          uint64_t* counter_bytes);
/* Per-kernel CUDA-event timing of subsequent renders (off by default).
 * After bhrt_ctx_finish, bhrt_ctx_kernel_ms returns the durations of the
 * last render's trace and shade kernels on the render stream. */
int bhrt_ctx_set_timing(bhrt_ctx* ctx, int32_t enable);
int bhrt_ctx_kernel_ms(bhrt_ctx* ctx, float* trace_ms, float* shade_ms);
/* Output layout of subsequent renders: 0 (default) = rows packed in order
 * of y into d_out; 1 = d_out is the whole image (height x width x 3) and each
 * rendered row lands at its image position — with d_out a peer GPU's image
 * buffer opened by bhrt_ipc_open, the ranks of a frame write their rows
 * straight into rank 0's image over NVLink and no gather follows. */
int bhrt_ctx_set_output_layout(bhrt_ctx* ctx, int32_t image_layout);

/* Device buffers shareable across processes (CUDA IPC over NVLink/NVSwitch
 * peer memory). bhrt_device_alloc: cudaMalloc on `device`; bhrt_ipc_export:
 * 64-byte handle of such a buffer; bhrt_ipc_open: map a peer process's buffer
 * on `device` (peer access enabled lazily); bhrt_ipc_close unmaps it. */
int bhrt_device_alloc(int32_t device, size_t bytes, void** d_ptr, bhrt_status_info* info);
int bhrt_device_free(int32_t device, void* d_ptr);
int bhrt_ipc_export(int32_t device, void* d_ptr, uint8_t handle[64], bhrt_status_info* info);
int bhrt_ipc_open(int32_t device, const uint8_t handle[64], void** d_ptr, bhrt_status_info* info);
int bhrt_ipc_close(int32_t device, void* d_ptr);

/* Number of rows selected by the tiling rule above. */
int32_t bhrt_tile_row_count(int32_t row_start, int32_t row_end, int32_t tile_rows,
                            int32_t tile_stride, int32_t tile_offset);

/* K0: measured FP64 FMA throughput of the current device (TFLOP/s). */
double bhrt_b200_fp64_peak_tflops(int iters, int reps, double* best_ms_out);

int32_t bhrt_cuda_abi_version(void);
/* Per-step algorithmic flop counts used for the roofline (fma = 2 flops). */
double bhrt_flops_per_step(int32_t integrator);

#ifdef __cplusplus
}
#endif

#endif /* BHRT_CUDA_H */
