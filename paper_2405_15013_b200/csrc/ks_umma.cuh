// Shared device/host helpers for the tcgen05 KS kernels (ks_tf32.cu,
// ks_half_bsl.cu): PTX wrappers for mbarriers, TMA, tcgen05 MMA / TMEM loads,
// UMMA shared-memory descriptors, element traits, the coalescing BSF store and
// tensor-map encoding.  Everything has internal linkage (one copy per TU).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "ks_internal.h"

namespace {

constexpr int BM = 128;        // batch rows per tile = UMMA M

// ---- PTX wrappers ----------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
// TMA stores (shared -> global, bulk-group completion) and their waits
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(src) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(c2), "r"(src) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void sts32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ float lds32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// UMMA shared-memory descriptor for a K-major, 128-byte-swizzled operand:
// start address, LBO = 16 B (unused for swizzled K-major), SBO = 1024 B
// (stride between 8-row groups), version 1 (sm_100), layout type 2 (SW128).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// UMMA descriptor of an MN-major TF32 operand in the SW128_32B canonical layout
// (layout type 1; what TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes): 32-byte
// chunks XOR-swizzled in 128-byte rows; measured on B200 (scripts/probe_umma_mn.cu).
__device__ __forceinline__ uint64_t mn_sw128_32b_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)(lbo >> 4) << 16;             // LBO: next 32-n group
    d |= (uint64_t)(sbo >> 4) << 32;             // SBO: next group of 4 l rows
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;                      // SWIZZLE_128B_BASE32B
    return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, N, M = 128.
__host__ __device__ constexpr uint32_t make_idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

// Element type T: float (kind::tf32, the TF32 path) or __nv_bfloat16 / __half
// (kind::f16, the half-precision path, NEXT-3).  A 128-byte operand row holds
// BK = 128 / sizeof(T) elements; one MMA consumes 32 bytes of K (KSTEP elements).
template <typename T> struct ElemTraits;
template <> struct ElemTraits<float> {
    static constexpr uint32_t fmt = 2;  // TF32
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    __device__ static float to_f(float v) { return v; }
    __device__ static float from_f(float v) { return v; }
};
template <> struct ElemTraits<__nv_bfloat16> {
    static constexpr uint32_t fmt = 1;  // BF16
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct ElemTraits<__half> {
    static constexpr uint32_t fmt = 0;  // F16
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    __device__ static float to_f(__half v) { return __half2float(v); }
    __device__ static __half from_f(float v) { return __float2half_rn(v); }
};

// BSF epilogue store through a warp-private shared-memory scratch.  Lane l holds
// row n0w + l of the tile: v[j][k] is the output at element offset
// off0 + k*d + j of that row of Y (row pitch ldy).  Each row's KB x J values are
// packed into 16-byte units (row-major [k][j], pitch UR + 1 units: an odd
// number, so the per-row writes are bank-conflict-free) and read back so that
// consecutive lanes store consecutive units: one coalesced STG.128 per lane per
// pass instead of 32 rows' worth of sectors per store instruction.  A unit
// never straddles a run of J outputs unless the runs are contiguous (J == d).
template <typename T, int J, int KB>
struct WarpStore {
    static constexpr int EPU = 16 / (int)sizeof(T);           // elements per 16-byte unit
    static constexpr int UR = KB * J / EPU;                     // units per row
    static constexpr int PITCH = (UR + 1) * 16;
    static constexpr int BYTES = 32 * PITCH;                    // per warp
    static_assert((KB * J) % EPU == 0 && UR % 2 == 0, "whole units, odd pitch");
};

template <typename T, int J, int KB>
__device__ __forceinline__ void warp_store_rows(uint32_t scr, const float (&v)[J][KB], T* __restrict__ Y,
                                                int64_t n0w, int64_t B, int64_t ldy, int64_t off0, int d, int lane) {
    using W = WarpStore<T, J, KB>;
    constexpr int EPU = W::EPU, UR = W::UR;
#pragma unroll
    for (int q = 0; q < UR; ++q) {
        uint32_t w[4];
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int e = q * 4 + x;
                w[x] = __float_as_uint(v[e % J][e / J]);
            }
        } else {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int e0 = q * 8 + 2 * x, e1 = e0 + 1;
                const T lo = ElemTraits<T>::from_f(v[e0 % J][e0 / J]), hi = ElemTraits<T>::from_f(v[e1 % J][e1 / J]);
                w[x] = (uint32_t)reinterpret_cast<const uint16_t&>(lo) | ((uint32_t)reinterpret_cast<const uint16_t&>(hi) << 16);
            }
        }
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(scr + lane * W::PITCH + q * 16), "r"(w[0]),
                     "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < UR; ++t) {
        const int u = t * 32 + lane;
        const int r = u / UR, q = u % UR;
        uint32_t w[4];
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(scr + r * W::PITCH + q * 16) : "memory");
        const int e0 = q * EPU;
        const int64_t n = n0w + r;
        if (n < B)
            __stcs(reinterpret_cast<uint4*>(Y + n * ldy + off0 + (int64_t)(e0 / J) * d + (e0 % J)),
                   make_uint4(w[0], w[1], w[2], w[3]));
    }
    __syncwarp();
}

// Direct BSF store (no shared-memory staging): lane l holds row n0w + l, v[j][k]
// is the output at element offset off0 + k*d + j.  When the J outputs of one k
// are contiguous with the next k's (J == d) a lane stores 16-byte units of
// consecutive outputs; else each run of J outputs (J % 4 == 0) in 16-byte units.
// Each warp store instruction writes 32 rows x 16 bytes (half sectors that L2
// merges) but costs no shared-memory bandwidth -- the scarce resource of the
// TF32 kernels (tensor-core operand reads, TMA fills and transposes share it).
template <int J, int KB>
__device__ __forceinline__ void direct_store_rows(const float (&v)[J][KB], float* __restrict__ Y, int64_t n0w,
                                                  int64_t B, int64_t ldy, int64_t off0, int d, int lane) {
    const int64_t n = n0w + lane;
    if (n >= B) return;
    float* row = Y + n * ldy + off0;
    if (J == d) {
        static_assert((KB * J) % 4 == 0, "whole 16-byte units");
#pragma unroll
        for (int q = 0; q < KB * J / 4; ++q) {
            float w[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) w[x] = v[(q * 4 + x) % J][(q * 4 + x) / J];
            __stcs(reinterpret_cast<float4*>(row + q * 4), make_float4(w[0], w[1], w[2], w[3]));
        }
    } else {
#pragma unroll
        for (int k = 0; k < KB; ++k)
#pragma unroll
            for (int j4 = 0; j4 < J; j4 += 4)
                __stcs(reinterpret_cast<float4*>(row + (int64_t)k * d + j4),
                       make_float4(v[j4][k], v[j4 + 1][k], v[j4 + 2][k], v[j4 + 3][k]));
    }
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}

template <typename T>
__host__ __device__ constexpr uint32_t make_idesc_t(int n) {
    return (1u << 4) | (ElemTraits<T>::fmt << 7) | (ElemTraits<T>::fmt << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ uint64_t sw64_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;            // 8 rows x 64 B
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;                     // SWIZZLE_64B
    return d;
}

__device__ __forceinline__ uint64_t sw32_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(256 >> 4) << 32;            // 8 rows x 32 B
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)6 << 61;                     // SWIZZLE_32B
    return d;
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}

// ---- host: tensor maps, debug knobs -------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box, CUtensorMapSwizzle sw,
            CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims,
                    strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// KS_TF32_DEBUG (profiling experiments only): bit 0 skips the epilogue's global
// stores, bit 1 skips the transposers' shared-memory reads.  0 in production.
// KS_TF32_MAXGRID (tests): cap the persistent grid so small problems exercise
// several tiles per CTA.  0 / unset in production.
int max_grid() {
    static int v = [] {
        const char* e = getenv("KS_TF32_MAXGRID");
        return e ? atoi(e) : 0;
    }();
    return v;
}

int debug_flags() {
    static int v = [] {
        const char* e = getenv("KS_TF32_DEBUG");
        return e ? atoi(e) : 0;
    }();
    return v;
}

}  // namespace
