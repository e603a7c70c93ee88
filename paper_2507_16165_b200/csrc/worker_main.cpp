// worker_main.cpp — GPU-backed network worker for the reference coordinator.
//
//   bhrt_worker_b200 worker --connect HOST:PORT [--threads N]
//
// The reference's `bhrt worker` subcommand (tools/bhrt.cpp:239-244) with the
// same flags and exit codes (bhrt.cpp:338-356). It speaks the unchanged BHRT
// wire protocol through the reference's own frame code (protocol.hpp
// read_frame / write_frame) and follows run_worker's exchange
// (netrender.cpp:107-165: HELLO, JOB, ROWS chunks of <= 64 rows, DONE; ERROR
// with codes 1 protocol / 2 io / 3 numerical before rethrowing). What differs
// is the scene: the JOB's key=value text is read by bhrt_scene_parse_text,
// which accepts the reference keys exactly as parse_scene does plus the
// extension keys (integrator, disk, spheres, checker sky, ...; SURVEY §8f
// rows 1-2), and the band is rendered by bhrt_cuda_render_rows on the B200
// (devices from $BHRT_DEVICES). A checker-sky scene may carry an empty PPM.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bhrt/errors.hpp"
#include "bhrt/image.hpp"
#include "bhrt/netrender.hpp"
#include "bhrt/protocol.hpp"
#include "bhrt/render.hpp"
#include "bhrt/stream.hpp"
#include "bhrt_cuda.h"

namespace {

// The underlying failure text of a BHRT_NUMERICAL status: the part after
// "pixel (x, y): ", i.e. the e.what() the reference's RenderError wraps
// (render.cpp:36-40).
std::string failure_what(const bhrt_status_info& info) {
    const std::string m(info.message);
    const size_t k = m.find("): ");
    return k == std::string::npos ? m : m.substr(k + 3);
}


constexpr std::uint32_t kErrProtocol = 1, kErrIo = 2, kErrNumerical = 3;  // netrender.cpp:14-16
constexpr int kRowsPerChunk = 64;                                        // netrender.cpp:18

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

void serve_job(bhrt::ByteStream& stream) {
    using namespace bhrt;
    write_frame(stream, HelloMsg{});
    const Message hello = read_frame(stream);
    const auto* h = std::get_if<HelloMsg>(&hello);
    if (h == nullptr) throw ProtocolError("expected HELLO from coordinator");
    if (h->version != kProtocolVersion)
        throw ProtocolError("unsupported coordinator version " + std::to_string(h->version));
    const Message job_msg = read_frame(stream);
    const auto* job = std::get_if<JobMsg>(&job_msg);
    if (job == nullptr) throw ProtocolError("expected JOB");

    bhrt_scene s;
    bhrt_status_info info;
    int32_t nsph = 0;
    std::vector<bhrt_sphere> spheres;
    int rc = bhrt_scene_parse_text(job->scene_text.c_str(), &s, nullptr, 0, &nsph, &info);
    if (rc == BHRT_INVALID_ARGUMENT && nsph > 0) {
        spheres.resize(static_cast<size_t>(nsph));
        rc = bhrt_scene_parse_text(job->scene_text.c_str(), &s, spheres.data(), nsph, &nsph, &info);
    }
    if (rc) throw UsageError(info.message);
    std::unique_ptr<ImageBuffer> background;
    if (s.sky_kind == BHRT_SKY_IMAGE || !job->background_ppm.empty()) {
        background = std::make_unique<ImageBuffer>(load_ppm(job->background_ppm));
        s.sky_rgb = background->bytes().data();
        s.sky_width = background->width();
        s.sky_height = background->height();
    }
    rc = bhrt_validate_scene(&s, &info);
    if (rc) throw UsageError(info.message);

    const BandAssignment band = job->band;
    if (band.row_start < 0 || band.row_end > s.height || band.row_start > band.row_end)
        throw ProtocolError("JOB band outside image bounds");
    const size_t row_bytes = 3ull * static_cast<size_t>(s.width);
    std::vector<std::uint8_t> pixels(row_bytes * static_cast<size_t>(band.row_end - band.row_start));
    if (!pixels.empty()) {
        const std::vector<int32_t> devs = devices_from_env();
        rc = bhrt_cuda_render_rows(&s, band.row_start, band.row_end, devs.empty() ? nullptr : devs.data(),
                                   static_cast<int32_t>(devs.size()), pixels.data(), pixels.size(), nullptr,
                                   &info);
        if (rc == BHRT_NUMERICAL) throw RenderError(info.px, info.py, failure_what(info));
        if (rc == BHRT_USAGE) throw UsageError(info.message);
        if (rc == BHRT_INVALID_ARGUMENT) throw std::invalid_argument(info.message);
        if (rc) throw IoError(std::string("bhrt_cuda: ") + info.message);
    }
    for (int row = band.row_start; row < band.row_end; row += kRowsPerChunk) {
        const int count = std::min(kRowsPerChunk, band.row_end - row);
        const auto first = pixels.begin() + static_cast<std::ptrdiff_t>(row_bytes * (row - band.row_start));
        write_frame(stream, RowsMsg{static_cast<std::uint32_t>(row), static_cast<std::uint32_t>(count),
                                    {first, first + static_cast<std::ptrdiff_t>(row_bytes * count)}});
    }
    write_frame(stream, DoneMsg{});
}

void run_gpu_worker(bhrt::ByteStream& stream) {
    const auto report = [&stream](std::uint32_t code, const std::string& text) {
        try {
            bhrt::write_frame(stream, bhrt::ErrorMsg{code, text});
        } catch (...) {  // coordinator gone; the original error still propagates
        }
    };
    try {
        serve_job(stream);
    } catch (const bhrt::ProtocolError& e) {
        report(kErrProtocol, e.what());
        throw;
    } catch (const bhrt::NumericalError& e) {
        report(kErrNumerical, e.what());
        throw;
    } catch (const std::exception& e) {
        report(kErrIo, e.what());
        throw;
    }
}

}  // namespace

int main(int argc, char** argv) {
    std::string endpoint = "127.0.0.1:4900";
    if (argc < 2 || std::strcmp(argv[1], "worker") != 0) {
        std::fprintf(stderr, "usage: %s worker --connect HOST:PORT [--threads N]\n", argv[0]);
        return 1;
    }
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--connect" && i + 1 < argc) {
            endpoint = argv[++i];
        } else if (a == "--threads" && i + 1 < argc) {
            if (std::atoi(argv[++i]) < 1) {  // render.cpp:71: threads must be >= 1
                std::fprintf(stderr, "error: --threads must be >= 1\n");
                return 1;
            }
        } else {
            std::fprintf(stderr, "error: unknown argument '%s'\n", a.c_str());
            return 1;
        }
    }
    try {
        const auto [host, port] = bhrt::parse_endpoint(endpoint);
        const std::unique_ptr<bhrt::FdStream> stream = bhrt::connect_tcp(host, port);
        run_gpu_worker(*stream);
        return 0;
    } catch (const bhrt::UsageError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const bhrt::ProtocolError& e) {
        std::fprintf(stderr, "protocol error: %s\n", e.what());
        return 4;
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
