// Probe: tcgen05.mma kind::tf32 with an MN-major A operand (no swizzle).
// One CTA, M=128, N=16, K=8.  Tries descriptor variants, prints max error.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ uint64_t mkdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// variant: 0 = A K-major (control), 1..4 = A MN-major with (lbo,sbo) choices
__global__ void probe(const float* A, const float* Bm, float* D, int variant, uint32_t lbo, uint32_t sbo) {
    __shared__ __align__(1024) float sA[128 * 8];
    __shared__ __align__(1024) float sB[16 * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    int tid = threadIdx.x;
    // A[m][k] row-major input
    for (int e = tid; e < 128 * 8; e += blockDim.x) {
        int m = e / 8, k = e % 8;
        float v = A[m * 8 + k];
        int off;
        if (variant == 0) off = (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;   // K-major
        else if (variant == 1) off = (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;              // MN-major compact
        else off = (m / 32) * 1024 + k * 128 + ((((m % 32) / 4) ^ (k % 8)) * 16) + (m % 4) * 4;   // MN SW128
        sA[off / 4] = v;
    }
    for (int e = tid; e < 16 * 8; e += blockDim.x) {
        int n = e / 8, k = e % 8;
        int off = (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
        sB[off / 4] = Bm[n * 8 + k];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = tslot;
    if (tid == 0) {
        uint32_t amn = variant == 0 ? 0u : 1u;
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amn << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        uint64_t ad = variant == 0 ? mkdesc(su32(sA), 128, 256) : mkdesc(su32(sA), lbo, sbo);
        if (variant == 2) ad |= (uint64_t)2 << 61;   // SWIZZLE_128B
        uint64_t bd = mkdesc(su32(sB), 128, 256);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    int w = tid / 32;
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 16; ++n) D[tid * 16 + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
    std::vector<float> A(128 * 8), Bm(16 * 8), ref(128 * 16);
    for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 7) % 11 - 5);
    for (int i = 0; i < 16 * 8; ++i) Bm[i] = (float)((i * 5) % 7 - 3);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            float s = 0;
            for (int k = 0; k < 8; ++k) s += A[m * 8 + k] * Bm[n * 8 + k];
            ref[m * 16 + n] = s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, Bm.size() * 4); cudaMalloc(&dD, ref.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bm.data(), Bm.size() * 4, cudaMemcpyHostToDevice);
    struct V { int variant; uint32_t lbo, sbo; const char* name; } vs[] = {
        {0, 0, 0, "K-major control"},
        {1, 128, 128, "MN lbo=128 sbo=128"},
        {1, 128, 4096, "MN lbo=128 sbo=4096"},
        {1, 4096, 128, "MN lbo=4096 sbo=128"},
        {1, 0, 128, "MN lbo=0 sbo=128"},
        {1, 128, 0, "MN lbo=128 sbo=0"},
        {2, 1024, 4096, "MN SW128 lbo=1024 sbo=4096"},
        {2, 4096, 1024, "MN SW128 lbo=4096 sbo=1024"},
        {2, 1024, 1024, "MN SW128 lbo=1024 sbo=1024"},
    };
    for (auto& v : vs) {
        cudaMemset(dD, 0, ref.size() * 4);
        probe<<<1, 128>>>(dA, dB, dD, v.variant, v.lbo, v.sbo);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(ref.size());
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (size_t i = 0; i < D.size(); ++i) { err = fmax(err, fabs(D[i] - ref[i])); mx = fmax(mx, fabs(D[i])); }
        printf("%-24s cuda=%s maxerr=%g max|D|=%g D[0..3]=%g %g %g %g ref=%g %g %g %g\n", v.name, cudaGetErrorString(e), err, mx,
               D[0], D[1], D[2], D[16], ref[0], ref[1], ref[2], ref[16]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
