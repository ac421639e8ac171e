// Measured FP32 FFMA peak of this device (ks_peak_ffma, include/ks.h): the
// denominator of the "alu" roofline of the FP32 CUDA-core KS kernels
// ("measure once per box ... an FFMA loop for FP32").  Not on the
// KS path.  Every thread runs 8 independent FMA chains (enough ILP to cover
// the 4-cycle FMA latency at 4 warps per SM sub-partition); 2 CTAs x 512
// threads per SM; flops = 2 x threads x 8 x iterations / event-timed duration.
#include "ks_internal.h"

namespace {

constexpr int PEAK_CHAINS = 8;
constexpr int PEAK_ITERS = 4096;

__global__ void __launch_bounds__(512, 2) ks_peak_ffma_kernel(float* out, float b, float c) {
    float v[PEAK_CHAINS];
#pragma unroll
    for (int q = 0; q < PEAK_CHAINS; ++q) v[q] = (float)(threadIdx.x + q) * 1e-3f;
#pragma unroll 16
    for (int it = 0; it < PEAK_ITERS; ++it)
#pragma unroll
        for (int q = 0; q < PEAK_CHAINS; ++q) v[q] = fmaf(v[q], b, c);
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < PEAK_CHAINS; ++q) s += v[q];
    if (s == 12345.678f) out[0] = s;        // keeps the chains live; never true for these inputs
}

}  // namespace

extern "C" ks_status_t ks_peak_ffma(ks_stream_t stream, double* tflops) {
    if (!tflops) return KS_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return KS_ERR_CUDA;
    const int sms = ks::num_sms(dev);
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return KS_ERR_OOM;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const dim3 grid(sms * 2 * 4), block(512);              // 4 waves of 2 CTAs per SM
    ks_peak_ffma_kernel<<<grid, block, 0, s>>>(out, 0.999f, 1e-4f);   // warm-up (clocks, icache)
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, s);
        ks_peak_ffma_kernel<<<grid, block, 0, s>>>(out, 0.999f, 1e-4f);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return KS_ERR_CUDA;
    const double flops = 2.0 * (double)grid.x * block.x * PEAK_CHAINS * PEAK_ITERS;
    *tflops = flops / (best * 1e-3) / 1e12;
    return KS_OK;
}
