// K0: FP64 FMA throughput microbenchmark (roofline denominator).
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the ray tracer is
// FP64-pipe bound, so its roofline denominator is measured here: every
// thread runs kChains independent DFMA dependency chains, so the FP64 pipe
// (not DFMA latency) is the limit. flops = threads * iters * kChains * 2.
#include <cuda_runtime.h>
#include <cstdint>

namespace bhrt_b200 {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep live, never true
}

// Returns achieved FP64 TFLOP/s (best of `reps`), or a negative CUDA error code.
extern "C" double bhrt_b200_fp64_peak_tflops(int iters, int reps, double* best_ms_out) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * blocks * threads) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp64_peak_kernel<<<blocks, threads>>>(out, iters / 10 + 1, 0.999999, 1e-9);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        fp64_peak_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return -2.0;
    if (best_ms_out) *best_ms_out = best;
    const double flops = 2.0 * kChains * static_cast<double>(iters) * blocks * threads;
    return flops / (best * 1e-3) / 1e12;
}

}  // namespace bhrt_b200
