// Probe: issue rate of back-to-back tcgen05.mma (cta_group::1, M = 128, operands
// K-major SWIZZLE_128B in shared memory, accumulator in TMEM) for kind::tf32
// and kind::f16 (BF16) at several N, one CTA per SM.  Prints MAC / clock / SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pmr scripts/probe_mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// K-major SWIZZLE_64B / SWIZZLE_32B (rows of 64 / 32 bytes; SBO = 8 rows)
template <int RB>
__device__ __forceinline__ uint64_t swdesc(uint32_t addr) {
    if constexpr (RB == 128) return sw128(addr);
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((8 * RB) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(RB == 64 ? 4 : 6) << 61;
    return d;
}

template <int KIND>   // 0 = tf32, 1 = f16 (bf16 operands)
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// NST stages of (A, B) tiles: the MMAs cycle through them (fresh operands per MMA
// group, as in a pipelined kernel) instead of re-reading one tile.
template <int KIND, int N, int NST = 1>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t STAGE = (128 + N) * 128;
    const uint32_t sA0 = su32(base);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < NST * (128 + N) * 32; i += blockDim.x) ((float*)base)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t fmt = KIND == 0 ? 2u : 1u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t sA = sA0 + (uint32_t)(it % NST) * STAGE, sB = sA + 128 * 128;
#pragma unroll
            for (int s = 0; s < 4; ++s)          // 4 MMAs cover the 128-byte rows (32 bytes of K each)
                mma<KIND>(tmem + (uint32_t)((it & 1) * N), sw128(sA + 32 * s), sw128(sB + 32 * s), idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n"
                     ::"r"(su32(&bar)));
        unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N, int NST = 1>
void run(const char* name, int sms) {
    unsigned long long* d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    const int smem = NST * (128 + N) * 128 + 1024;
    cudaFuncSetAttribute(rate<KIND, N, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    rate<KIND, N, NST><<<sms, 128, smem>>>(iters, d);
    rate<KIND, N, NST><<<sms, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double kper = KIND == 0 ? 8 : 16;
    const double macs = (double)iters * 4 * 128 * N * kper;
    printf("%-10s st=%d N=%3d: %s  cycles/MMA %.1f  MAC/clk/SM %.0f\n", name, NST, N, cudaGetErrorString(e), mx / (iters * 4.0),
           macs / mx);
    cudaFree(d);
}

// RB-byte operand rows (RB/32 MMAs per stage), NST stages; NLD extra warps stream
// LDS.128 over a separate 64 KB region meanwhile (transposer / epilogue traffic).
template <int N, int RB, int NST, int NLD>
__global__ void __launch_bounds__(32 * (1 + NLD), 1) rate_rb(int iters, unsigned long long* cyc, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t STAGE = (128 + N) * RB;
    const uint32_t sA0 = su32(base);
    const uint32_t ld0 = sA0 + NST * STAGE;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < (NST * (128 + N) * RB + 65536) / 4; i += blockDim.x) ((float*)base)[i] = 0.f;
    if (threadIdx.x == 0) {
        done = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t sA = sA0 + (uint32_t)(it % NST) * STAGE, sB = sA + 128 * RB;
#pragma unroll
            for (int s = 0; s < RB / 32; ++s)
                mma<0>(tmem + (uint32_t)((it & 1) * N), swdesc<RB>(sA + 32 * s), swdesc<RB>(sB + 32 * s), idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n"
                     ::"r"(su32(&bar)));
        unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
        done = 1;
    } else if (threadIdx.x >= 32) {
        float acc = 0.f;
        const uint32_t t = threadIdx.x - 32;
        while (!done) {
#pragma unroll 8
            for (int q = 0; q < 32; ++q) {
                float4 v;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "r"(ld0 + ((t * 16 + q * 16 * 32 * NLD) & 65535)));
                acc += v.x + v.w;
            }
        }
        if (acc == 12345.f) sink[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int RB, int NST, int NLD>
void run_rb(int sms) {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    cudaMalloc(&sink, 4);
    const int smem = NST * (128 + N) * RB + 65536 + 1024;
    cudaFuncSetAttribute(rate_rb<N, RB, NST, NLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4000 * 128 / (RB * 4);
    rate_rb<N, RB, NST, NLD><<<sms, 32 * (1 + NLD), smem>>>(iters, d, sink);
    rate_rb<N, RB, NST, NLD><<<sms, 32 * (1 + NLD), smem>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double macs = (double)iters * (RB / 32) * 128 * N * 8;
    printf("tf32 RB=%3d N=%3d st=%d ldwarps=%d: %s  MAC/clk/SM %.0f\n", RB, N, NST, NLD, cudaGetErrorString(e), macs / mx);
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    if (getenv("PROBE_RB")) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        run_rb<256, 128, 2, 0>(sms); run_rb<256, 64, 2, 0>(sms); run_rb<256, 32, 2, 0>(sms);
        run_rb<128, 128, 2, 0>(sms); run_rb<128, 64, 2, 0>(sms); run_rb<128, 32, 2, 0>(sms);
        run_rb<64, 128, 2, 0>(sms); run_rb<64, 32, 2, 0>(sms);
        run_rb<256, 128, 2, 4>(sms); run_rb<256, 128, 2, 8>(sms); run_rb<256, 32, 2, 4>(sms); run_rb<256, 32, 2, 8>(sms);
        run_rb<128, 128, 2, 4>(sms); run_rb<128, 128, 2, 8>(sms); run_rb<128, 32, 2, 4>(sms); run_rb<128, 64, 2, 4>(sms);
        return 0;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 256>("tf32", sms);
    run<0, 128>("tf32", sms);
    run<0, 64>("tf32", sms);
    run<0, 32>("tf32", sms);
    run<1, 256>("bf16", sms);
    run<1, 128>("bf16", sms);
    run<1, 64>("bf16", sms);
    run<0, 256, 4>("tf32", sms);
    run<0, 128, 6>("tf32", sms);
    run<0, 64, 8>("tf32", sms);
    run<1, 256, 4>("bf16", sms);
    run<1, 128, 6>("bf16", sms);
    run<0, 256>("tf32x1sm", 1);
    run<1, 256>("bf16x1sm", 1);
    return 0;
}
