// Probe: FP32 FMA throughput of FFMA vs FFMA2 (fma.rn.f32x2, sm_100a), 8
// independent chains per thread, 1024 threads per SM; prints TFLOP/s.
// Also checks FFMA2 is bit-identical to two FFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_ffma2 scripts/probe_ffma2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <bool PAIR>
__global__ void __launch_bounds__(1024) peak(float* out, int iters, float s) {
    float x = threadIdx.x * 1e-6f, y = s;
    if constexpr (!PAIR) {
        float acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = q * 1e-3f;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = fmaf(x, y, acc[q]);
        float t = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) t += acc[q];
        out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    } else {
        uint64_t acc[8];
        const uint64_t xx = f2(x, x), yy = f2(y, y);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = f2(q * 1e-3f, q * 2e-3f);
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = fma2(xx, yy, acc[q]);
        float t = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += __uint_as_float((uint32_t)acc[q]) + __uint_as_float((uint32_t)(acc[q] >> 32));
        out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    }
}

__global__ void exact(int* bad) {
    // FFMA2 lanes vs scalar fmaf on awkward values
    uint32_t seed = 12345u + threadIdx.x * 7919u;
    for (int i = 0; i < 4096; ++i) {
        seed = seed * 1664525u + 1013904223u; float a = __uint_as_float((seed >> 9) | 0x3f000000u) - 0.75f;
        seed = seed * 1664525u + 1013904223u; float b = __uint_as_float((seed >> 9) | 0x40000000u) - 3.0f;
        seed = seed * 1664525u + 1013904223u; float c = __uint_as_float((seed >> 9) | 0x3e000000u) * 1e-3f;
        seed = seed * 1664525u + 1013904223u; float d = __uint_as_float((seed >> 9) | 0x3f800000u) * 0.37f;
        uint64_t r = fma2(f2(a, d), f2(b, a), f2(c, b));
        float lo = __uint_as_float((uint32_t)r), hi = __uint_as_float((uint32_t)(r >> 32));
        if (__float_as_uint(lo) != __float_as_uint(fmaf(a, b, c)) || __float_as_uint(hi) != __float_as_uint(fmaf(d, a, b)))
            atomicAdd(bad, 1);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* o;
    cudaMalloc(&o, sizeof(float) * sms * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int pass = 0; pass < 2; ++pass) {
        for (int pair = 0; pair < 2; ++pair) {
            cudaEventRecord(a);
            if (pair) peak<true><<<sms, 1024>>>(o, iters, 1.0001f);
            else peak<false><<<sms, 1024>>>(o, iters, 1.0001f);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double flops = 2.0 * 16 * iters * 1024.0 * sms;
            if (pass) printf("%s: %.1f TFLOP/s\n", pair ? "FFMA2" : "FFMA ", flops / ms / 1e9);
        }
    }
    int* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    exact<<<64, 256>>>(bad);
    int h = -1;
    cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    printf("FFMA2 vs fmaf mismatches: %d of %d\n", h, 64 * 256 * 4096 * 2);
    return 0;
}
