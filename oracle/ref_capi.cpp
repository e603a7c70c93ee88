// ref_capi.cpp — C entry points over the COMPILED REFERENCE (oracle/_ref).
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile from the reference's own
// sources under /root/reference/proj (never copied into this repo) and used by
// tests/ to pin the oracle, by tests/golden/make_golden.py to produce the
// committed fixtures, and by bench.py's reference-arm / cpu_baseline legs.
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "bhrt/bench.hpp"
#include "bhrt/camera.hpp"
#include "bhrt/config.hpp"
#include "bhrt/geodesic.hpp"
#include "bhrt/image.hpp"
#include "bhrt/render.hpp"

#include "../include/bhrt_cuda.h"

using namespace bhrt;

namespace {

TraceConfig tcfg(double eps, double esc, int mw, double rt, double at) {
    TraceConfig c;
    c.epsilon = eps;
    c.escape_radius = esc;
    c.max_windings = mw;
    c.rel_tol = rt;
    c.abs_tol = at;
    return c;
}

Vec3 v(const double* a) { return {a[0], a[1], a[2]}; }
void put(double* a, const Vec3& x) { a[0] = x.x; a[1] = x.y; a[2] = x.z; }

SceneConfig to_scene(const bhrt_scene* s, ImageBuffer* bg) {
    SceneConfig sc;
    sc.hole = {s->mass, v(s->center)};
    sc.camera = {v(s->cam_pos), v(s->cam_look_at), s->vertical_fov, s->width, s->height};
    sc.samples = {s->spp, s->seed};
    sc.trace = tcfg(s->epsilon, s->escape_radius, s->max_windings, s->rel_tol, s->abs_tol);
    sc.background = bg;
    return sc;
}

ImageBuffer* make_bg(const bhrt_scene* s) {
    if (!s->sky_rgb) return nullptr;
    std::vector<std::uint8_t> px(s->sky_rgb, s->sky_rgb + 3 * static_cast<size_t>(s->sky_width) * s->sky_height);
    return new ImageBuffer(s->sky_width, s->sky_height, std::move(px));
}

int fill(bhrt_status_info* info, int code, int px, int py, const char* what) {
    if (info) {
        info->code = code;
        info->px = px;
        info->py = py;
        std::snprintf(info->message, sizeof info->message, "%s", what);
    }
    return code;
}

}  // namespace

extern "C" {

int ref_trace(const double* o, const double* d, double mass, const double* c, double eps, double esc,
              int mw, double rt, double at, int* kind, double* dir, int* npoints, double* last2) {
    try {
        const RayPolyline p = trace(v(o), v(d), BlackHole{mass, v(c)}, tcfg(eps, esc, mw, rt, at));
        *kind = static_cast<int>(p.outcome.kind);
        put(dir, p.outcome.escape_direction);
        *npoints = static_cast<int>(p.points.size());
        put(last2, p.points[p.points.size() >= 2 ? p.points.size() - 2 : 0]);
        put(last2 + 3, p.points.back());
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    } catch (const NumericalError&) {
        return BHRT_NUMERICAL;
    }
}

// Full polyline (for golden fixtures of the pointwise tests). Returns count or -code.
int ref_trace_points(const double* o, const double* d, double mass, const double* c, double eps,
                     double esc, int mw, double rt, double at, double* pts, int cap) {
    try {
        const RayPolyline p = trace(v(o), v(d), BlackHole{mass, v(c)}, tcfg(eps, esc, mw, rt, at));
        const int n = static_cast<int>(p.points.size());
        for (int i = 0; i < n && i < cap; ++i) put(pts + 3 * i, p.points[i]);
        return n;
    } catch (const std::invalid_argument&) {
        return -BHRT_INVALID_ARGUMENT;
    } catch (const NumericalError&) {
        return -BHRT_NUMERICAL;
    }
}

int ref_integrate_window(const double* st, double dphi, double mass, double rt, double at,
                         double* hint, double* out) {
    try {
        const GeodesicState s{st[0], st[1], st[2]};
        TraceConfig cfg = tcfg(0.05, 1e4, 10, rt, at);
        const GeodesicState r = integrate_window(s, dphi, mass, cfg, hint);
        out[0] = r.phi; out[1] = r.u; out[2] = r.du_dphi;
        return 0;
    } catch (const StepSizeUnderflow& e) {
        out[0] = e.state.phi; out[1] = e.state.u; out[2] = e.state.du_dphi;
        return 1;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    }
}

int ref_plane_basis(const double* o, const double* d, const double* c, double* e1, double* e2) {
    const auto b = plane_basis(v(o), v(d), BlackHole{1.0, v(c)});
    if (!b) return 0;
    put(e1, b->e1);
    put(e2, b->e2);
    return 1;
}

int ref_initial_conditions(const double* o, const double* d, const double* c, double* st) {
    try {
        const GeodesicState s = initial_conditions(v(o), v(d), BlackHole{1.0, v(c)});
        st[0] = s.phi; st[1] = s.u; st[2] = s.du_dphi;
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    }
}

double ref_step_dphi(double u, double eps) {
    return step_dphi({0.0, u, 0.0}, tcfg(eps, 1e4, 10, 1e-10, 1e-12));
}

int ref_deflection_angle(double b, double mass, double eps, double esc, double* out) {
    try {
        *out = deflection_angle(b, BlackHole{mass, {}}, tcfg(eps, esc, 10, 1e-10, 1e-12));
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    } catch (const NumericalError&) {
        return BHRT_NUMERICAL;
    }
}

int ref_deflection_of_ray(const double* o, const double* d, double mass, double eps, double esc,
                          double* out) {
    try {
        *out = deflection_of_ray(v(o), v(d), BlackHole{mass, {}}, tcfg(eps, esc, 10, 1e-10, 1e-12));
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    } catch (const NumericalError&) {
        return BHRT_NUMERICAL;
    }
}

uint64_t ref_hash_counter(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    return hash_counter(seed, a, b, c);
}

int ref_generate_ray(const bhrt_scene* s, int px, int py, int sample, double* origin, double* dir) {
    try {
        const SceneConfig sc = to_scene(s, nullptr);
        const Ray r = generate_ray(sc.camera, px, py, sample, sc.samples);
        put(origin, r.origin);
        put(dir, r.dir);
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    }
}

void ref_sample_direction(const uint8_t* rgb, int w, int h, const double* dir, double* out) {
    std::vector<std::uint8_t> px(rgb, rgb + 3 * static_cast<size_t>(w) * h);
    const ImageBuffer img(w, h, std::move(px));
    const Rgb c = sample_direction(img, v(dir));
    out[0] = c.r; out[1] = c.g; out[2] = c.b;
}

int ref_render_rows(const bhrt_scene* s, int row_start, int row_end, int threads, uint8_t* out,
                    bhrt_status_info* info) {
    ImageBuffer* bg = make_bg(s);
    int rc = 0;
    try {
        const SceneConfig sc = to_scene(s, bg);
        const std::vector<std::uint8_t> px = render_rows(sc, row_start, row_end, threads);
        std::memcpy(out, px.data(), px.size());
        fill(info, 0, -1, -1, "");
    } catch (const RenderError& e) {
        rc = fill(info, BHRT_NUMERICAL, e.px, e.py, e.what());
    } catch (const UsageError& e) {
        rc = fill(info, BHRT_USAGE, -1, -1, e.what());
    } catch (const std::invalid_argument& e) {
        rc = fill(info, BHRT_INVALID_ARGUMENT, -1, -1, e.what());
    } catch (const std::exception& e) {
        rc = fill(info, BHRT_IO, -1, -1, e.what());
    }
    delete bg;
    return rc;
}

int ref_make_bands(int height, int workers, int* rs, int* re, int cap, int* count) {
    try {
        const auto b = make_bands(height, workers);
        if (static_cast<int>(b.size()) > cap) return BHRT_INVALID_ARGUMENT;
        for (size_t i = 0; i < b.size(); ++i) { rs[i] = b[i].row_start; re[i] = b[i].row_end; }
        *count = static_cast<int>(b.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return BHRT_INVALID_ARGUMENT;
    }
}

// The reference's own timing harness (bench.cpp:13-22,59-73): mean wall
// seconds of `repeats` render_image runs at `threads`.
double ref_strong_scaling_mean(const bhrt_scene* s, int threads, int repeats) {
    ImageBuffer* bg = make_bg(s);
    double mean = -1.0;
    try {
        const SceneConfig sc = to_scene(s, bg);
        const auto recs = run_strong_scaling(sc, {threads}, repeats);
        mean = mean_wall_seconds(recs, threads);
    } catch (const std::exception&) {
        mean = -1.0;
    }
    delete bg;
    return mean;
}

// The reference's timing harness (run_strong_scaling, bench.cpp:59-73, timed
// at :13-22) with a RenderRunner (bench.hpp:32) that renders a SAMPLE of the
// frame's pixels — (px[i], py[i]), i < n — through the reference's own
// shade_pixel (render.cpp:22-49), pulled from a shared atomic counter by
// `threads` std::threads (render_rows' dynamic queue, render.cpp:80-115, at
// pixel granularity). Mean wall seconds of `repeats` runs; -1 on failure.
double ref_strong_scaling_pixels_mean(const bhrt_scene* s, int threads, int repeats, const int* px,
                                      const int* py, int n) {
    ImageBuffer* bg = make_bg(s);
    double mean = -1.0;
    try {
        const SceneConfig sc = to_scene(s, bg);
        const RenderRunner runner = [px, py, n](const SceneConfig& scene, int workers) {
            std::atomic<int> next{0};
            std::exception_ptr err;
            std::mutex mu;
            std::vector<std::thread> pool;
            for (int t = 0; t < workers; ++t)
                pool.emplace_back([&] {
                    try {
                        for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1))
                            (void)shade_pixel(scene, px[i], py[i]);
                    } catch (...) {  // first failure wins (render.cpp:100-104)
                        std::lock_guard<std::mutex> g(mu);
                        if (!err) err = std::current_exception();
                        next.store(n);
                    }
                });
            for (auto& th : pool) th.join();
            if (err) std::rethrow_exception(err);
        };
        const auto recs = run_strong_scaling(sc, {threads}, repeats, BenchMode::threads, runner);
        mean = mean_wall_seconds(recs, threads);
    } catch (const std::exception&) {
        mean = -1.0;
    }
    delete bg;
    return mean;
}

// image.cpp:107-113 save_ppm of a w x h RGB8 image. Returns the size;
// writes when cap is large enough.
size_t ref_save_ppm(int w, int h, const std::uint8_t* rgb, std::uint8_t* out, size_t cap) {
    std::vector<std::uint8_t> px(rgb, rgb + 3 * static_cast<size_t>(w) * h);
    const std::vector<std::uint8_t> b = save_ppm(ImageBuffer(w, h, std::move(px)));
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    return b.size();
}

// config.cpp:96-112 serialize_scene of the scene's reference fields.
// Returns the text length; writes when cap is large enough.
size_t ref_serialize_scene(const bhrt_scene* s, char* buf, size_t cap) {
    const std::string t = serialize_scene(to_scene(s, nullptr));
    if (buf && cap > t.size()) std::memcpy(buf, t.c_str(), t.size() + 1);
    return t.size();
}

// config.cpp:27-44,114-130 parse_scene(parse_kv(text)) into the reference
// fields of `out` (other fields untouched). BHRT_USAGE + message on error.
int ref_parse_scene(const char* text, bhrt_scene* out, bhrt_status_info* info) {
    try {
        const SceneConfig sc = parse_scene(parse_kv(text));
        out->mass = sc.hole.mass;
        put(out->center, sc.hole.center);
        put(out->cam_pos, sc.camera.position);
        put(out->cam_look_at, sc.camera.look_at);
        out->vertical_fov = sc.camera.vertical_fov;
        out->width = sc.camera.width;
        out->height = sc.camera.height;
        out->spp = sc.samples.spp;
        out->seed = sc.samples.seed;
        out->epsilon = sc.trace.epsilon;
        out->escape_radius = sc.trace.escape_radius;
        out->max_windings = sc.trace.max_windings;
        out->rel_tol = sc.trace.rel_tol;
        out->abs_tol = sc.trace.abs_tol;
        return 0;
    } catch (const UsageError& e) {
        return fill(info, BHRT_USAGE, -1, -1, e.what());
    }
}

}  // extern "C"
