// shade.cu — per-pixel shading pass for spp values that do not divide the
// warp (fused shading handles spp in {1,2,4,8,16,32} inside the trace
// kernels): reads the per-sample records, shades (device_common.cuh
// shade_sample), accumulates in sample order and quantises (render.cpp:22-49).
// Also the launch wrapper for a render.
#include "device_common.cuh"

namespace bhrt_b200 {

__global__ void __launch_bounds__(256) shade_kernel(const __grid_constant__ KParams p) {
    const long long npix = (long long)p.n_rows * p.width;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    double acc[3] = {0.0, 0.0, 0.0};
    bool failed = false;
    for (int s = 0; s < p.spp; ++s) {
        const bhrt_ray_record r = p.records[i * p.spp + s];
        if (r.object < 0) {
            failed = true;
            break;
        }
        double c[3];
        shade_sample(p, r.object, r.sphere, vld(r.point), c);
        acc[0] += c[0];
        acc[1] += c[1];
        acc[2] += c[2];
    }
    const long long jrow = i / p.width;
    uint8_t* o = p.out + 3 * (p.out_image ? (long long)packed_row_to_y(p, (int)jrow) * p.width +
                                                (i - jrow * p.width)
                                          : i);
    if (failed) {
        // lowest failing pixel in image order (y * width + x)
        const long long j = i / p.width;
        atomicMin(&p.stats[3], (unsigned long long)packed_row_to_y(p, (int)j) * p.width + (i - j * p.width));
        o[0] = o[1] = o[2] = 0;
        return;
    }
    store_pixel(o, acc, p.inv_spp);
}

void launch_reference(const KParams& p, cudaStream_t st);
void launch_scene(const KParams& p, cudaStream_t st);
void launch_table_trace(const KParams& p, cudaStream_t st);

int launch_trace(const KParams& p, cudaStream_t st, int* launches, cudaEvent_t* ev) {
    const long long n = (long long)p.n_rows * p.width * p.spp;
    if (n <= 0) return 0;
    if (p.integrator < BHRT_INTEGRATOR_REFERENCE || p.integrator > BHRT_INTEGRATOR_TABLE) return -1;
    if (!p.fused_shade && !p.records) return -1;
    if (ev) cudaEventRecord(ev[0], st);
    if (p.integrator == BHRT_INTEGRATOR_REFERENCE)
        launch_reference(p, st);
    else if (p.integrator == BHRT_INTEGRATOR_TABLE)
        launch_table_trace(p, st);
    else
        launch_scene(p, st);
    ++*launches;
    if (ev) cudaEventRecord(ev[1], st);
    if (!p.fused_shade) {
        const long long npix = (long long)p.n_rows * p.width;
        shade_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(p);
        ++*launches;
    }
    if (ev) cudaEventRecord(ev[2], st);
    return 0;
}

}  // namespace bhrt_b200
