// render_shim.cpp — drop-in replacement for the reference's proj/src/render.cpp.
//
// Implements the whole render.hpp surface (validate_scene, shade_pixel,
// make_bands, render_rows, render_band, render_image; render.hpp:26-66) with
// the reference's signatures, types and exception taxonomy, on top of the C
// ABI in include/bhrt_cuda.h. Compiled against the reference's OWN headers,
// so objects built from the reference (netrender.o, bench.o, the CLI, its
// acceptance suite) link to this file instead of render.o unchanged — every
// caller of the hot path (render.cpp:121-129, netrender.cpp:139-140,
// bench.cpp:13-22) then runs on the GPU.
//
// `threads` keeps its meaning as a validity check (render.cpp:71); the work
// runs on the devices in $BHRT_DEVICES (comma-separated ordinals; default:
// the current device). Output is byte-identical for every `threads` and
// every device split (cyclic rows), like render.hpp:58-59,65 requires.
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "bhrt/render.hpp"
#include "bhrt_cuda.h"

namespace bhrt {

namespace {

// The underlying failure text of a BHRT_NUMERICAL status: the part after
// "pixel (x, y): ", i.e. the e.what() the reference's RenderError wraps
// (render.cpp:36-40).
std::string failure_what(const bhrt_status_info& info) {
    const std::string m(info.message);
    const size_t k = m.find("): ");
    return k == std::string::npos ? m : m.substr(k + 3);
}


bhrt_scene to_abi(const SceneConfig& s) {
    bhrt_scene a;
    bhrt_scene_defaults(&a);  // extensions off: reference integrator, image sky
    a.mass = s.hole.mass;
    a.center[0] = s.hole.center.x;
    a.center[1] = s.hole.center.y;
    a.center[2] = s.hole.center.z;
    a.cam_pos[0] = s.camera.position.x;
    a.cam_pos[1] = s.camera.position.y;
    a.cam_pos[2] = s.camera.position.z;
    a.cam_look_at[0] = s.camera.look_at.x;
    a.cam_look_at[1] = s.camera.look_at.y;
    a.cam_look_at[2] = s.camera.look_at.z;
    a.vertical_fov = s.camera.vertical_fov;
    a.width = s.camera.width;
    a.height = s.camera.height;
    a.spp = s.samples.spp;
    a.seed = s.samples.seed;
    a.epsilon = s.trace.epsilon;
    a.escape_radius = s.trace.escape_radius;
    a.max_windings = s.trace.max_windings;
    a.rel_tol = s.trace.rel_tol;
    a.abs_tol = s.trace.abs_tol;
    if (s.background) {
        a.sky_rgb = s.background->bytes().data();
        a.sky_width = s.background->width();
        a.sky_height = s.background->height();
    } else {
        a.sky_rgb = nullptr;
        a.sky_width = a.sky_height = 0;
    }
    return a;
}

std::vector<int32_t> devices_from_env() {
    std::vector<int32_t> d;
    const char* e = std::getenv("BHRT_DEVICES");
    if (!e || !*e) return d;
    std::string s(e);
    size_t pos = 0;
    while (pos <= s.size()) {
        const size_t comma = s.find(',', pos);
        const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        if (!tok.empty()) d.push_back(static_cast<int32_t>(std::stoi(tok)));
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return d;
}

[[noreturn]] void rethrow(int code, const bhrt_status_info& info) {
    switch (code) {
        case BHRT_USAGE: throw UsageError(info.message);
        case BHRT_INVALID_ARGUMENT: throw std::invalid_argument(info.message);
        case BHRT_NUMERICAL: throw RenderError(info.px, info.py, failure_what(info));
        case BHRT_IO: throw IoError(info.message);
        default: throw std::runtime_error(std::string("bhrt_cuda: ") + info.message);
    }
}

}  // namespace

void validate_scene(const SceneConfig& scene) {  // render.cpp:11-20
    const bhrt_scene a = to_abi(scene);
    bhrt_status_info info;
    const int rc = bhrt_validate_scene(&a, &info);
    if (rc) rethrow(rc, info);
}

std::vector<std::uint8_t> render_rows(const SceneConfig& scene, int row_start, int row_end,
                                      int threads) {  // render.cpp:68-119
    validate_scene(scene);
    if (threads < 1) throw std::invalid_argument("render: threads must be >= 1");
    if (row_start < 0 || row_end > scene.camera.height || row_start > row_end)
        throw std::invalid_argument("render: row range out of bounds");
    const int rows = row_end - row_start;
    std::vector<std::uint8_t> out(3 * static_cast<std::size_t>(rows) * scene.camera.width);
    if (rows == 0) return out;
    const bhrt_scene a = to_abi(scene);
    const std::vector<int32_t> devs = devices_from_env();
    bhrt_status_info info;
    const int rc = bhrt_cuda_render_rows(&a, row_start, row_end, devs.empty() ? nullptr : devs.data(),
                                         static_cast<int32_t>(devs.size()), out.data(), out.size(),
                                         nullptr, &info);
    if (rc) rethrow(rc, info);
    return out;
}

std::array<std::uint8_t, 3> shade_pixel(const SceneConfig& scene, int px, int py) {  // render.cpp:22-49
    if (px < 0 || px >= scene.camera.width || py < 0 || py >= scene.camera.height)
        throw std::invalid_argument("shade_pixel: pixel out of range");
    const std::vector<std::uint8_t> row = render_rows(scene, py, py + 1, 1);
    return {row[3 * px], row[3 * px + 1], row[3 * px + 2]};
}

std::vector<BandAssignment> make_bands(int height, int workers) {  // render.cpp:51-66
    if (height < 1 || workers < 1)
        throw std::invalid_argument("make_bands: height and workers must be >= 1");
    const int n = height < workers ? height : workers;
    std::vector<int32_t> rs(n), re(n);
    int32_t count = 0;
    bhrt_make_bands(height, workers, rs.data(), re.data(), n, &count);
    std::vector<BandAssignment> bands;
    bands.reserve(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i) bands.push_back({i, rs[i], re[i]});
    return bands;
}

std::vector<std::uint8_t> render_band(const SceneConfig& scene, const BandAssignment& band) {
    return render_rows(scene, band.row_start, band.row_end, 1);  // render.cpp:121-123
}

ImageBuffer render_image(const SceneConfig& scene, int threads) {  // render.cpp:125-129
    std::vector<std::uint8_t> pixels = render_rows(scene, 0, scene.camera.height, threads);
    return ImageBuffer(scene.camera.width, scene.camera.height, std::move(pixels));
}

}  // namespace bhrt
