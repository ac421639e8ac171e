// Probe (round 2): tcgen05.mma kind::tf32 with an MN-major A operand laid
// out as CUTLASS's "SW128_32B" atom (UMMA layout type 1, SWIZZLE_128B_BASE32B:
// 32-byte chunks XOR-swizzled within 128-byte rows, 4-row period), loaded by
// TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; and a TMA store
// (cp.async.bulk.tensor shared->global, SWIZZLE_128B) of the accumulator.
// One CTA, M = 128 (batch n), N = 64, K = 32 (4 MMAs of K = 8).
//   A global: Xs[l][n] (l = K index rows of 128 n, n contiguous = BSL layout)
//   B global: Kt[k][l] (K-major, SW128 as in production)
// Variant v selects (LBO, SBO) for the A descriptor.  Prints max |err|.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ uint64_t mkdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

constexpr int M = 128, N = 64, K = 32;

__global__ void probe(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                      const __grid_constant__ CUtensorMap ymap, float* D, uint32_t lbo, uint32_t sbo, int store_tma) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sA = su32(sm);                  // 4 boxes x [32 l][32 n] = 16 KB
    const uint32_t sB = sA + 16384;                // [64 k][32 l] SW128 = 8 KB
    const uint32_t sY = sB + 8192;                 // 2 x [32 rows][32 cols] SW128 per warp, 4 warps = 32 KB
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16384 + 8192)
                     : "memory");
        for (int g = 0; g < 4; ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(sA + g * 4096), "l"(&amap), "r"(g * 32), "r"(0), "r"(su32(&bar)) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(sB), "l"(&bmap), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W1;\n}\n" ::"r"(
                su32(&bar)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
        // idesc: D f32 (bit 4), A tf32 (7-9 = 2), B tf32 (10-12 = 2), A MN-major (bit 15), N>>3, M>>4
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(M >> 4) << 24);
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t ad = mkdesc(sA + s * 1024, lbo, sbo, 1);                 // SW128_32B (type 1)
            uint64_t bd = 0;                                                         // K-major SW128
            bd |= (uint64_t)(((sB + 32 * s) >> 4) & 0x3FFF);
            bd |= (uint64_t)1 << 16;
            bd |= (uint64_t)(1024 >> 4) << 32;
            bd |= (uint64_t)1 << 46;
            bd |= (uint64_t)2 << 61;
            const uint32_t acc = s > 0;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                     : "memory");
    }
    __syncwarp();
    {
        const uint32_t mb = su32(&mbar);
        asm volatile(
            "{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(mb)
            : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int warp = tid / 32, lane = tid % 32;
    const int row = warp * 32 + lane;
    for (int col0 = 0; col0 < N; col0 += 32) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%"
            "28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(tmem + ((uint32_t)(warp * 32) << 16) + col0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!store_tma) {
            for (int q = 0; q < 32; ++q) D[row * N + col0 + q] = __uint_as_float(r[q]);
        } else {
            // SW128 staging: row `lane` of the warp's [32 rows][32 floats] box, 16-byte chunk c at (c ^ (lane % 8))
            const uint32_t box = sY + (uint32_t)(warp * 2 + col0 / 32) * 4096;
            for (int c = 0; c < 8; ++c)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(box + lane * 128 + ((c ^ (lane % 8)) * 16)),
                             "r"(r[4 * c]), "r"(r[4 * c + 1]), "r"(r[4 * c + 2]), "r"(r[4 * c + 3]) : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&ymap),
                             "r"(col0), "r"(warp * 32), "r"(box) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (store_tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main() {
    std::vector<float> Xs(K * M), Kt(N * K), ref(M * N, 0.0);
    for (int l = 0; l < K; ++l)
        for (int n = 0; n < M; ++n) Xs[l * M + n] = (float)(((n * 7 + l * 3) % 11) - 5);
    for (int k = 0; k < N; ++k)
        for (int l = 0; l < K; ++l) Kt[k * K + l] = (float)(((k * 5 + l * 13) % 7) - 3);
    for (int n = 0; n < M; ++n)
        for (int k = 0; k < N; ++k) {
            double s = 0;
            for (int l = 0; l < K; ++l) s += (double)Xs[l * M + n] * Kt[k * K + l];
            ref[n * N + k] = (float)s;
        }
    float *dX, *dK, *dD;
    cudaMalloc(&dX, Xs.size() * 4);
    cudaMalloc(&dK, Kt.size() * 4);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dX, Xs.data(), Xs.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dK, Kt.data(), Kt.size() * 4, cudaMemcpyHostToDevice);
    auto fn = enc();
    CUtensorMap amap, bmap, ymap;
    cuuint32_t es[2] = {1, 1};
    {
        cuuint64_t dims[2] = {M, K}, str[1] = {M * 4};
        cuuint32_t box[2] = {32, 32};
        CUresult r = fn(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("amap encode %d\n", (int)r);
    }
    {
        cuuint64_t dims[2] = {K, N}, str[1] = {K * 4};
        cuuint32_t box[2] = {32, N};
        CUresult r = fn(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dK, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("bmap encode %d\n", (int)r);
    }
    {
        cuuint64_t dims[2] = {N, M}, str[1] = {N * 4};
        cuuint32_t box[2] = {32, 32};
        CUresult r = fn(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dD, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("ymap encode %d\n", (int)r);
    }
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    struct V {
        uint32_t lbo, sbo;
    } vs[] = {{4096, 512}, {512, 4096}, {4096, 1024}, {1024, 4096}};
    for (int store = 0; store < 2; ++store)
        for (auto v : vs) {
            cudaMemset(dD, 0, M * N * 4);
            probe<<<1, 128, 64 * 1024>>>(amap, bmap, ymap, dD, v.lbo, v.sbo, store);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> D(M * N);
            cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < M * N; ++i) mx = fmax(mx, fabs((double)D[i] - ref[i]));
            printf("store_tma=%d lbo=%u sbo=%u err=%s maxabs=%g D[0]=%g ref[0]=%g D[77*N+5]=%g ref=%g\n", store, v.lbo,
                   v.sbo, cudaGetErrorString(e), mx, D[0], ref[0], D[77 * N + 5], ref[77 * N + 5]);
            if (e != cudaSuccess) return 1;
        }
    return 0;
}
