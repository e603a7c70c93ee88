// bench_main.cpp — the reference's timing harness driving the B200 path.
//
//   bhrt_bench_b200 bench --config SCENE --background PPM --output CSV
//                   [--sweep strong|weak] [--worker-counts 1,2,4]
//                   [--weak-pairs 1x128,2x256,4x512] [--repeats 5] [--warmup 1]
//
// The reference CLI's `bench` subcommand (tools/bhrt.cpp:246-275, flags at
// :306-313, exit codes at :338-356) without its CLI11 front end (not vendored
// in /root/reference). The sweep, the timing and the CSV are the reference's
// OWN code, linked unchanged: run_strong_scaling / run_weak_scaling
// (bench.cpp:59-92, each run timed around one RenderRunner call,
// bench.cpp:13-22) and emit_csv (bench.cpp:94-131, per-configuration means
// as run = -1 rows). What runs inside the timed call is the B200 path:
//   * a scene of reference keys only: the default RenderRunner, i.e.
//     render_image — which resolves to render_shim.cpp (the C ABI, mode R,
//     byte-identical to the reference's image);
//   * a scene with extension keys (integrator, disk, spheres, checker sky;
//     bhrt_scene_parse_text): a RenderRunner that renders the whole frame
//     through bhrt_cuda_render_rows with host buffers.
// `--config` takes a complete scene text (serialize_scene's keys, as in a
// coordinator JOB). `--warmup N` (default 1, a drop-in addition) renders N
// untimed frames first so the first timed run does not carry CUDA context
// creation. Devices: $BHRT_DEVICES (comma-separated ordinals), as the shim.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bhrt/bench.hpp"
#include "bhrt/config.hpp"
#include "bhrt/errors.hpp"
#include "bhrt/image.hpp"
#include "bhrt/render.hpp"
#include "bhrt_cuda.h"

namespace {

using bhrt::UsageError;

// The keys parse_scene reads (config.cpp parse_scene); anything else is an
// extension key of bhrt_scene_parse_text.
const std::set<std::string> kReferenceKeys = {
    "mass", "center", "cam-pos", "look-at", "fov-rad", "width", "height", "spp",
    "seed", "epsilon", "escape-radius", "max-windings", "rel-tol", "abs-tol"};

std::vector<int> parse_counts(const std::string& s, const char* flag) {
    std::vector<int> v;
    std::stringstream in(s);
    std::string item;
    while (std::getline(in, item, ','))
        v.push_back(static_cast<int>(bhrt::parse_int(item, flag)));
    if (v.empty()) throw UsageError(std::string("invalid ") + flag + ": empty list");
    return v;
}

std::vector<std::pair<int, int>> parse_pairs(const std::string& s, const char* flag) {
    std::vector<std::pair<int, int>> v;
    std::stringstream in(s);
    std::string item;
    while (std::getline(in, item, ',')) {
        const size_t x = item.find('x');
        if (x == std::string::npos) throw UsageError(std::string("invalid ") + flag + ": expected WORKERSxWIDTH");
        v.emplace_back(static_cast<int>(bhrt::parse_int(item.substr(0, x), flag)),
                       static_cast<int>(bhrt::parse_int(item.substr(x + 1), flag)));
    }
    if (v.empty()) throw UsageError(std::string("invalid ") + flag + ": empty list");
    return v;
}

std::string read_file(const std::string& path, const char* what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw bhrt::IoError(std::string("cannot open ") + what + " '" + path + "'");
    std::stringstream buf;
    buf << in.rdbuf();
    return buf.str();
}

std::vector<int32_t> devices_from_env() {
    std::vector<int32_t> d;
    const char* e = std::getenv("BHRT_DEVICES");
    for (const char* p = e; p && *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) break;
        d.push_back(static_cast<int32_t>(v));
        p = *end == ',' ? end + 1 : end;
    }
    return d;
}

// Extension scene: the parsed bhrt_scene and its storage.
struct ExtScene {
    bhrt_scene s{};
    std::vector<bhrt_sphere> spheres;
    std::unique_ptr<bhrt::ImageBuffer> sky;
};

void render_ext(const ExtScene& x, int width, std::vector<std::uint8_t>& pixels) {
    bhrt_scene s = x.s;
    s.width = width;
    pixels.resize(3ull * static_cast<size_t>(s.width) * static_cast<size_t>(s.height));
    const std::vector<int32_t> devs = devices_from_env();
    bhrt_status_info info;
    const int rc = bhrt_cuda_render_rows(&s, 0, s.height, devs.empty() ? nullptr : devs.data(),
                                         static_cast<int32_t>(devs.size()), pixels.data(), pixels.size(),
                                         nullptr, &info);
    if (rc == BHRT_NUMERICAL) {  // the underlying text after "pixel (x, y): " (render.cpp:36-40)
        const std::string m(info.message);
        const size_t k = m.find("): ");
        throw bhrt::RenderError(info.px, info.py, k == std::string::npos ? m : m.substr(k + 3));
    }
    if (rc == BHRT_USAGE) throw UsageError(info.message);
    if (rc == BHRT_INVALID_ARGUMENT) throw std::invalid_argument(info.message);
    if (rc) throw bhrt::IoError(std::string("bhrt_cuda: ") + info.message);
}

int cmd_bench(const std::map<std::string, std::string>& opt) {
    if (opt.at("config").empty()) throw UsageError("--config is required");
    const std::string output = opt.at("output");
    if (output.empty()) throw UsageError("--output is required");
    const std::string text = read_file(opt.at("config"), "config file");
    const std::string background = opt.at("background");
    const int repeats = static_cast<int>(bhrt::parse_int(opt.at("repeats"), "--repeats"));
    if (repeats < 1) throw UsageError("invalid --repeats: must be >= 1");
    const int warmup = static_cast<int>(bhrt::parse_int(opt.at("warmup"), "--warmup"));
    if (warmup < 0) throw UsageError("invalid --warmup: must be >= 0");

    bool reference_only = true;
    for (const auto& kv : bhrt::parse_kv(text))
        if (!kReferenceKeys.count(kv.first)) reference_only = false;

    bhrt::SceneConfig scene;
    std::unique_ptr<bhrt::ImageBuffer> bg;
    ExtScene ext;
    bhrt::RenderRunner runner;  // empty: the reference's default, render_image
    if (reference_only) {
        if (background.empty()) throw UsageError("--background is required");
        scene = bhrt::parse_scene(bhrt::parse_kv(text));
        bg = std::make_unique<bhrt::ImageBuffer>(bhrt::load_ppm_file(background));
        scene.background = bg.get();
        bhrt::validate_scene(scene);
    } else {
        bhrt_status_info info;
        int32_t nsph = 0;
        int rc = bhrt_scene_parse_text(text.c_str(), &ext.s, nullptr, 0, &nsph, &info);
        if (rc == BHRT_INVALID_ARGUMENT && nsph > 0) {
            ext.spheres.resize(static_cast<size_t>(nsph));
            rc = bhrt_scene_parse_text(text.c_str(), &ext.s, ext.spheres.data(), nsph, &nsph, &info);
        }
        if (rc) throw UsageError(info.message);
        if (ext.s.sky_kind == BHRT_SKY_IMAGE) {
            if (background.empty()) throw UsageError("--background is required");
            ext.sky = std::make_unique<bhrt::ImageBuffer>(bhrt::load_ppm_file(background));
            ext.s.sky_rgb = ext.sky->bytes().data();
            ext.s.sky_width = ext.sky->width();
            ext.s.sky_height = ext.sky->height();
        }
        if (bhrt_validate_scene(&ext.s, &info)) throw UsageError(info.message);
        // the record fields (bench.cpp make_record) of the extended scene
        scene.camera.width = ext.s.width;
        scene.camera.height = ext.s.height;
        scene.samples.spp = ext.s.spp;
        scene.trace.epsilon = ext.s.epsilon;
        runner = [&ext](const bhrt::SceneConfig& sc, int workers) {
            if (workers < 1) throw std::invalid_argument("render: threads must be >= 1");
            std::vector<std::uint8_t> pixels;
            render_ext(ext, sc.camera.width, pixels);
        };
    }

    const std::string sweep = opt.at("sweep");
    if (sweep != "strong" && sweep != "weak") throw UsageError("invalid --sweep: expected 'strong' or 'weak'");
    for (int i = 0; i < warmup; ++i) {  // untimed: CUDA context, module load, first scene upload
        if (runner)
            runner(scene, 1);
        else
            bhrt::render_image(scene, 1);
    }
    std::vector<bhrt::TimingRecord> records;
    if (sweep == "strong") {
        records = bhrt::run_strong_scaling(scene, parse_counts(opt.at("worker-counts"), "--worker-counts"),
                                           repeats, bhrt::BenchMode::threads, runner);
    } else {
        records = bhrt::run_weak_scaling(scene, parse_pairs(opt.at("weak-pairs"), "--weak-pairs"), repeats,
                                         bhrt::BenchMode::threads, runner);
    }
    const std::string csv = bhrt::emit_csv(records);
    std::ofstream out(output, std::ios::trunc);
    if (!out) throw bhrt::IoError("cannot open '" + output + "' for writing");
    out << csv;
    if (!out) throw bhrt::IoError("write failed for '" + output + "'");
    std::fprintf(stderr, "wrote %s (%zu runs)\n", output.c_str(), records.size());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    std::map<std::string, std::string> opt = {
        {"config", ""},       {"background", ""}, {"output", ""},      {"sweep", "strong"},
        {"worker-counts", "1,2,4"}, {"weak-pairs", "1x128,2x256,4x512"}, {"repeats", "5"}, {"warmup", "1"}};
    if (argc < 2 || std::strcmp(argv[1], "bench") != 0) {
        std::fprintf(stderr,
                     "usage: %s bench --config SCENE --background PPM --output CSV [--sweep strong|weak] "
                     "[--worker-counts L] [--weak-pairs L] [--repeats N] [--warmup N]\n",
                     argv[0]);
        return 1;
    }
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--", 0) != 0 || !opt.count(a.substr(2)) || i + 1 >= argc) {
            std::fprintf(stderr, "error: unknown or incomplete argument '%s'\n", a.c_str());
            return 1;
        }
        opt[a.substr(2)] = argv[++i];
    }
    try {
        return cmd_bench(opt);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const bhrt::NumericalError& e) {
        std::fprintf(stderr, "numerical error: %s\n", e.what());
        return 3;
    } catch (const bhrt::IoError& e) {
        std::fprintf(stderr, "i/o error: %s\n", e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
