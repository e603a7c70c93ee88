// Microbenchmark: DFMA throughput per SM vs resident warps and per-thread ILP
// (how much independent FP64 work the B200 scheduler needs to hide latency).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int c = 0; c < ILP; ++c) x[c] = threadIdx.x * 1e-7 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < ILP; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < ILP; ++c) s += x[c];
    if (s == 1.2345) out[0] = s;
}
template <int ILP>
void run(int warps_per_sm, int sms, double* out) {
    const int iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<ILP><<<sms, 32 * warps_per_sm>>>(out, 100, 0.9999, 1e-9);
    cudaEventRecord(e0);
    k<ILP><<<sms, 32 * warps_per_sm>>>(out, iters, 0.9999, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dfma_per_sm_per_ns = (double)iters * ILP * 32 * warps_per_sm / (ms * 1e6);
    // cycles per dependent DFMA for one warp = ms*1e6*clk / iters  (clk ~1.965 GHz)
    printf("ILP %d warps/SM %2d: %7.2f DFMA lanes/SM/ns  (%.1f cyc per chain step)\n", ILP, warps_per_sm,
           dfma_per_sm_per_ns, ms * 1e6 * 1.965 / iters);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    for (int w : {1, 2, 4, 8, 12, 16, 24, 32}) run<1>(w, sms, out);
    for (int w : {1, 2, 4, 8, 16}) run<2>(w, sms, out);
    for (int w : {1, 4, 8, 16}) run<4>(w, sms, out);
    return 0;
}
