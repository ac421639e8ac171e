// Probe (round 2): read throughput of TMA boxes with short inner runs -- the
// BSF d > 1 gather of the TF32 J-kernel -- against contiguous boxes and an
// LDGSTS (cp.async 16 B) gather by 128 threads.  No compute: a producer
// thread streams boxes into a P-slot ring, a consumer warp releases slots.
// X is B x N row-major (BSF), N = c*d with c = 128; every CTA walks its own
// tiles (round robin), every byte of X is read once.  Prints GB/s per shape.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(bar),
                 "r"(par) : "memory");
}

// mode 0: 3-D box {J, BL, 128} of X viewed [B][N/d][d] at (j0, l0, n0)
// mode 1: 2-D box {W, 128} of X viewed [B][N] at (col0, n0)
__global__ void __launch_bounds__(160) tma_probe(const __grid_constant__ CUtensorMap map, int mode, int ntiles, int nk,
                                                 int d, int J, int BL, int W, uint32_t box_bytes, int P) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[16], empty[16];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int p = 0; p < P; ++p) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[p])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su32(&empty[p])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int my = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int G = my * nk;
    if (tid == 0) {
        for (int g = 0; g < G; ++g) {
            const int p = g % P;
            if (g >= P) mbar_wait(su32(&empty[p]), ((g / P) - 1) & 1);
            const int t = blockIdx.x + (g / nk) * gridDim.x, kk = g % nk;
            // tile t -> (j-group fastest, n-block) ; a = 1
            const int njg = d / J;
            const int jg = t % njg, nb = t / njg;
            const uint32_t dst = su32(sm) + p * box_bytes;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[p])), "r"(box_bytes)
                         : "memory");
            if (mode == 0)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"(dst),
                    "l"(&map), "r"(jg * J), "r"(kk * (BL - 1)), "r"(nb * 128), "r"(su32(&full[p])) : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];" ::"r"(dst),
                    "l"(&map), "r"(jg * (W - 4) + kk * (W - 4) * njg), "r"(nb * 128), "r"(su32(&full[p])) : "memory");
        }
    } else if (tid >= 32 && tid < 64) {
        for (int g = 0; g < G; ++g) {
            const int p = g % P;
            mbar_wait(su32(&full[p]), (g / P) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[p])) : "memory");
        }
    }
    __syncthreads();
}

// LDGSTS gather: 128 threads, thread = row n; per stage each thread copies BL runs of J*4 bytes (16 B each)
__global__ void __launch_bounds__(128) ldgsts_probe(const float* X, int ntiles, int nk, int N, int d, int J, int BL,
                                                    int64_t B, int P) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    const int tid = threadIdx.x;
    const int my = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int G = my * nk;
    const int njg = d / J;
    const uint32_t stage = 128 * BL * J * 4;
    for (int g = 0; g < G; ++g) {
        const int p = g % P;
        const int t = blockIdx.x + (g / nk) * gridDim.x, kk = g % nk;
        const int jg = t % njg, nb = t / njg;
        const int64_t n = (int64_t)nb * 128 + tid;
        const float* src = X + n * N + (int64_t)(kk * BL) * d + jg * J;
        const uint32_t dst = su32(sm_raw) + p * stage + tid * BL * J * 4;
        for (int l = 0; l < BL; ++l)
            for (int q = 0; q < J / 4; ++q)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (l * J + 4 * q) * 4),
                             "l"(src + (int64_t)l * d + 4 * q) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (g >= P - 1) asm volatile("cp.async.wait_group %0;" ::"n"(2) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main() {
    const int64_t B = 25088;
    const int c = 128;
    auto fn = enc();
    cudaFuncSetAttribute(tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(ldgsts_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case {
        int d, J, mode, ctas;
    } cases[] = {{16, 4, 0, 1}, {16, 8, 0, 1}, {16, 16, 0, 1}, {64, 4, 0, 1}, {64, 8, 0, 1}, {64, 16, 0, 1},
                 {64, 32, 0, 1}, {4, 4, 1, 1}, {8, 8, 1, 1}, {16, 16, 1, 1}, {1, 1, 2, 1}, {16, 8, 3, 2}};
    for (auto cs : cases) {
        const int N = c * cs.d;
        float* X;
        cudaMalloc(&X, (size_t)B * N * 4);
        cudaMemset(X, 0, (size_t)B * N * 4);
        const int BL = cs.J >= 16 ? 9 : 17;              // 16 (8) l + 1 padding row (as the J-kernel)
        CUtensorMap map;
        cuuint32_t es[3] = {1, 1, 1};
        uint32_t box_bytes = 0;
        int nk = 0, ntiles = 0, W = 0;
        CUresult r = CUDA_SUCCESS;
        if (cs.mode == 0) {
            cuuint64_t dims[3] = {(cuuint64_t)cs.d, (cuuint64_t)c, (cuuint64_t)B};
            cuuint64_t str[2] = {(cuuint64_t)cs.d * 4, (cuuint64_t)N * 4};
            cuuint32_t box[3] = {(cuuint32_t)cs.J, (cuuint32_t)BL, 128};
            r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = cs.J * BL * 128 * 4;
            nk = c / (BL - 1);
            ntiles = (int)(B / 128) * (cs.d / cs.J);
        } else if (cs.mode == 1) {
            W = (cs.d <= 8 ? 16 : 8) * cs.d + 4;         // contiguous run: 16 (8) l x d j (+4 pad)
            cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)B};
            cuuint64_t str[1] = {(cuuint64_t)N * 4};
            cuuint32_t box[2] = {(cuuint32_t)W, 128};
            r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = W * 128 * 4;
            nk = c / (cs.d <= 8 ? 16 : 8);
            ntiles = (int)(B / 128);
        } else if (cs.mode == 2) {                       // BSF d = 1 SW128 box {32, 128}
            W = 36;
            cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)B};
            cuuint64_t str[1] = {(cuuint64_t)N * 4};
            cuuint32_t box[2] = {32, 128};
            r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            box_bytes = 32 * 128 * 4;
            nk = c / 32;
            ntiles = (int)(B / 128);
        }
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            continue;
        }
        int P = (int)(180 * 1024 / (box_bytes ? box_bytes : 65536));
        if (P > 6) P = 6;
        if (P < 2) P = 2;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            if (cs.mode == 3) {
                const int BLg = 16;
                const int nkg = c / BLg;
                const int ntg = (int)(B / 128) * (cs.d / cs.J);
                ldgsts_probe<<<sms * cs.ctas, 128, P * 128 * BLg * cs.J * 4>>>(X, ntg, nkg, N, cs.d, cs.J, BLg, B, P);
            } else {
                tma_probe<<<sms * cs.ctas, 160, P * box_bytes + 1024>>>(map, cs.mode, ntiles, nk, cs.d, cs.J, BL, W,
                                                                       box_bytes, P);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        const double bytes = (double)B * N * 4;
        printf("d=%d J=%d mode=%d P=%d box=%u B ctas/SM=%d  %s  %.1f us  %.0f GB/s (X %.0f MB)\n", cs.d, cs.J, cs.mode,
               P, box_bytes, cs.ctas, cudaGetErrorString(err), best * 1e3, bytes / best / 1e6, bytes / 1e6);
        cudaFree(X);
    }
    return 0;
}
