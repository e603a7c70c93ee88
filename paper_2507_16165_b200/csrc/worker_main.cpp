// worker_main.cpp — GPU-backed network worker for the reference coordinator.
//
//   bhrt_worker_b200 worker --connect HOST:PORT [--threads N]
//
// The reference's `bhrt worker` subcommand (tools/bhrt.cpp:239-244) with the
// same flags and exit codes (bhrt.cpp:338-356), linked against render_shim.cpp
// instead of render.cpp: the unchanged BHRT wire protocol and run_worker
// (netrender.cpp:107-165) serve the coordinator's JOB, and the band itself
// is rendered by the B200 kernels.
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "bhrt/errors.hpp"
#include "bhrt/netrender.hpp"
#include "bhrt/stream.hpp"

int main(int argc, char** argv) {
    std::string endpoint = "127.0.0.1:4900";
    int threads = 1;
    if (argc < 2 || std::strcmp(argv[1], "worker") != 0) {
        std::fprintf(stderr, "usage: %s worker --connect HOST:PORT [--threads N]\n", argv[0]);
        return 1;
    }
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--connect" && i + 1 < argc) {
            endpoint = argv[++i];
        } else if (a == "--threads" && i + 1 < argc) {
            threads = std::atoi(argv[++i]);
            if (threads <= 0) threads = 1;
        } else {
            std::fprintf(stderr, "error: unknown argument '%s'\n", a.c_str());
            return 1;
        }
    }
    try {
        const auto [host, port] = bhrt::parse_endpoint(endpoint);
        const std::unique_ptr<bhrt::FdStream> stream = bhrt::connect_tcp(host, port);
        bhrt::run_worker(*stream, threads);
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
