// TF32 tensor-core KS kernel (tcgen05.mma.kind::tf32, accumulators in TMEM)
// for the GEMM-like patterns where each (i, j) block is a genuine dense
// contraction (b, c >= 16; north star).  Not in the paper, whose kernel is
// CUDA-core only: on B200 the FP32 FFMA path is ALU-bound
// for b, c >= 48 (arithmetic intensity bc/(2(b+c)) > the FFMA ridge), so the
// tensor cores turn these factors HBM-bound again.
//
// One CTA owns the output tile Y[n0:n0+128, row_{i,j}[k0:k0+BN]]
// (output-stationary, Alg. 3; written exactly once).
//   UMMA view:  D[m][n] = sum_k A[m][k] B[n][k],  M = 128 batch rows,
//               N = BN outputs (k index of the KS block), K = l (c).
//   A = X[:, col_{i,j}]  -- BSL: MN-major (batch contiguous), BSF d=1: K-major
//   B = K[row_{i,j}, col_{i,j}] from k_tf32 (pre-rounded RNA, [q][k][l], K-major)
// Warp roles (160 threads):
//   warps 0-3  producers: cp.async 16-byte chunks of the X and K tiles straight
//              into the canonical no-swizzle UMMA smem layouts (core matrices
//              of 8 rows x 16 B), STAGES-deep ring, mbarrier full/empty;
//              then the epilogue: tcgen05.ld (32x32b) TMEM -> registers ->
//              coalesced global stores in the caller's layout.
//   warp 4     TMEM allocator + single-thread MMA issuer (tcgen05.mma,
//              tcgen05.commit -> empty[stage] / accumulator-ready barrier).
// X is fed as raw FP32 bits: the tensor core uses its TF32 part (truncation of
// the 13 low mantissa bits); K is rounded to nearest at pack time.  FP32
// accumulation.  Contract: normwise error <= 5e-3 (north star), DESIGN.md.
#include "ks_internal.h"

namespace {

constexpr int BM = 128;       // batch rows per CTA = UMMA M
constexpr int BKC = 32;       // l per pipeline stage (4 UMMA k-steps of 8)
constexpr int NPROD = 128;    // producer / epilogue threads
constexpr int NTHREADS = NPROD + 32;

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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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

// Shared-memory matrix descriptor, no swizzle (canonical "interleave" layout):
// start address, leading-dimension byte offset, stride-dimension byte offset,
// version 1 (sm_100), layout type 0.
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// Instruction descriptor: D f32, A/B tf32, A major (0 K, 1 MN), B K-major, N, M = 128.
__host__ __device__ constexpr uint32_t make_idesc(int a_mn_major, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn_major << 15) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
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

template <int BN>
struct Tf32Cfg {
    static constexpr int A_BYTES = BM * BKC * 4;          // 16 KB
    static constexpr int B_BYTES = BN * BKC * 4;          // BN * 128 B
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = (STAGE <= 32 * 1024) ? 3 : 2;
    static constexpr int BAR_BYTES = 128;
    static constexpr int SMEM = STAGES * STAGE + BAR_BYTES;
    static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static_assert(BN % 16 == 0 && BN <= 256, "UMMA N for M=128");
};

// Smem layouts (byte offsets inside a stage), no swizzle, 16-byte chunks:
//  K-major tile (rows r, K index l in [0,32)):   (r/8)*1024 + (l/4)*128 + (r%8)*16 + (l%4)*4
//      -> LBO (next 4-l chunk) = 128, SBO (next 8-row group) = 1024
//  MN-major A tile (rows m, l):                   (m/4)*512 + (l/8)*128 + (l%8)*16 + (m%4)*4
//      -> LBO (next 8-l group) = 128, SBO (next 4-row chunk) = 512
template <int LAYOUT, int BN>
__global__ void __launch_bounds__(NTHREADS, 1)
ks_tf32_kernel(const float* __restrict__ X, const float* __restrict__ Kt32, float* __restrict__ Y,
               int64_t B, int a, int b, int c, int d) {
    using C = Tf32Cfg<BN>;
    constexpr int S = C::STAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::STAGE);
    // bars[0..S): full, bars[S..2S): empty, bars[2S]: accumulator ready, bars[2S+1] (low 32 bits): tmem base
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accb = smem_u32(&bars[2 * S]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 1]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int nkc = b / BN;
    const int64_t nnb = (B + BM - 1) / BM;
    int64_t bid = blockIdx.x;
    const int kc = (int)(bid % nkc);
    bid /= nkc;
    const int64_t nb = bid % nnb;
    const int64_t q = bid / nnb;                 // q = i*d + j
    const int i = (int)(q / d), j = (int)(q % d);
    const int k0 = kc * BN;
    const int64_t n0 = nb * BM;
    const int64_t N = (int64_t)a * c * d, M = (int64_t)a * b * d;
    const int nk = (c + BKC - 1) / BKC;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, NPROD);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(accb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t smem0 = smem_u32(smem);

    if (warp < 4) {
        // ===================== producers =====================
        const float* xcol = nullptr;   // BSL: row s = i*c*d + l*d + j ; BSF: element (n, i*c*d + l)
        const float* kt = Kt32 + ((int64_t)q * b + k0) * c;   // [k][l] rows of this tile
        for (int t = 0; t < nk; ++t) {
            const int st = t % S;
            if (t >= S) mbar_wait(empty0 + 8 * st, ((t / S) - 1) & 1);
            const uint32_t sa = smem0 + st * C::STAGE;
            const uint32_t sb = sa + C::A_BYTES;
            const int l0 = t * BKC;
            // ---- A tile: 128 rows x 32 l = 1024 chunks of 16 B
#pragma unroll
            for (int r = 0; r < (BM * BKC / 4) / NPROD; ++r) {
                const int idx = tid + r * NPROD;
                if (LAYOUT == KS_LAYOUT_BSL) {
                    const int m4 = idx % (BM / 4), l = idx / (BM / 4);
                    const int64_t n = n0 + 4 * m4;
                    const bool ok = (l0 + l < c) && (n < B);
                    const float* src = X + ((int64_t)i * c * d + (int64_t)(ok ? l0 + l : 0) * d + j) * B + (ok ? n : 0);
                    cp_async16(sa + m4 * 512 + (l / 8) * 128 + (l % 8) * 16, src, ok ? 16u : 0u);
                } else {
                    const int l4 = idx % (BKC / 4), m = idx / (BKC / 4);
                    const int64_t n = n0 + m;
                    const bool ok = (l0 + 4 * l4 < c) && (n < B);
                    const float* src = X + (ok ? n : 0) * N + (int64_t)i * c + (ok ? l0 + 4 * l4 : 0);
                    cp_async16(sa + (m / 8) * 1024 + l4 * 128 + (m % 8) * 16, src, ok ? 16u : 0u);
                }
            }
            // ---- B tile: BN rows x 32 l
#pragma unroll
            for (int r = 0; r < (BN * BKC / 4 + NPROD - 1) / NPROD; ++r) {
                const int idx = tid + r * NPROD;
                if (idx < BN * BKC / 4) {
                    const int l4 = idx % (BKC / 4), kr = idx / (BKC / 4);
                    const bool ok = (l0 + 4 * l4 < c);
                    const float* src = kt + (int64_t)kr * c + (ok ? l0 + 4 * l4 : 0);
                    cp_async16(sb + (kr / 8) * 1024 + l4 * 128 + (kr % 8) * 16, src, ok ? 16u : 0u);
                }
            }
            cp_async_commit();
            if (t >= S - 1) {
                cp_async_wait<S - 1>();
                fence_proxy_async();
                mbar_arrive(full0 + 8 * ((t - (S - 1)) % S));
            }
        }
        cp_async_wait<0>();
        fence_proxy_async();
        for (int u = (nk > S - 1 ? nk - (S - 1) : 0); u < nk; ++u) mbar_arrive(full0 + 8 * (u % S));

        // ===================== epilogue =====================
        mbar_wait(accb, 0);
        tc_fence_after();
        const int row = warp * 32 + (tid & 31);          // TMEM lane = batch row in tile
        const int64_t n = n0 + row;
        const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int col = 0; col < BN; col += 16) {
            float v[16];
            tmem_ld16(tbase + col, v);
            if (n < B) {
                if (LAYOUT == KS_LAYOUT_BSL) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int64_t r = (int64_t)i * b * d + (int64_t)(k0 + col + e) * d + j;
                        __stcs(Y + r * B + n, v[e]);
                    }
                } else {
                    float* yp = Y + n * M + (int64_t)i * b + k0 + col;
#pragma unroll
                    for (int e = 0; e < 16; e += 4)
                        __stcs(reinterpret_cast<float4*>(yp + e), make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                }
            }
        }
    } else if (warp == 4) {
        // ===================== MMA issuer =====================
        if ((tid & 31) == 0) {
            constexpr uint32_t idesc = make_idesc(LAYOUT == KS_LAYOUT_BSL ? 1 : 0, BN);
            for (int t = 0; t < nk; ++t) {
                const int st = t % S;
                mbar_wait(full0 + 8 * st, (t / S) & 1);
                tc_fence_after();
                const uint32_t sa = smem0 + st * C::STAGE;
                const uint32_t sb = sa + C::A_BYTES;
                const int ksteps = min(BKC / 8, (c - t * BKC) / 8);
                for (int s = 0; s < ksteps; ++s) {
                    const uint64_t ad = (LAYOUT == KS_LAYOUT_BSL) ? make_desc(sa + s * 128, 128, 512)
                                                                  : make_desc(sa + s * 256, 128, 1024);
                    const uint64_t bd = make_desc(sb + s * 256, 128, 1024);
                    mma_tf32(tmem, ad, bd, idesc, (t > 0 || s > 0) ? 1u : 0u);
                }
                mma_commit(empty0 + 8 * st);
            }
            mma_commit(accb);
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    }
}

// ------------------------------------------------------------------ host ------
int pick_bn(int64_t b) {
    if (b <= 256 && b % 16 == 0) return (int)b;
    for (int bn : {256, 192, 128, 96, 64, 48, 32, 16})
        if (b % bn == 0) return bn;
    return 0;
}

template <int LAYOUT, int BN>
cudaError_t launch_bn(const ks_handle_s& h, const KsCall& call) {
    using C = Tf32Cfg<BN>;
    auto kern = ks_tf32_kernel<LAYOUT, BN>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t blocks = (h.b / BN) * ((call.B + BM - 1) / BM) * (h.a * h.d);
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    kern<<<(unsigned)blocks, NTHREADS, C::SMEM, call.stream>>>(call.X, h.k_tf32, call.Y, call.B, (int)h.a,
                                                                (int)h.b, (int)h.c, (int)h.d);
    ks::count_launch();
    return cudaGetLastError();
}

template <int LAYOUT>
cudaError_t launch_layout(const ks_handle_s& h, const KsCall& call) {
    switch (pick_bn(h.b)) {
        case 256: return launch_bn<LAYOUT, 256>(h, call);
        case 240: return launch_bn<LAYOUT, 240>(h, call);
        case 224: return launch_bn<LAYOUT, 224>(h, call);
        case 208: return launch_bn<LAYOUT, 208>(h, call);
        case 192: return launch_bn<LAYOUT, 192>(h, call);
        case 176: return launch_bn<LAYOUT, 176>(h, call);
        case 160: return launch_bn<LAYOUT, 160>(h, call);
        case 144: return launch_bn<LAYOUT, 144>(h, call);
        case 128: return launch_bn<LAYOUT, 128>(h, call);
        case 112: return launch_bn<LAYOUT, 112>(h, call);
        case 96: return launch_bn<LAYOUT, 96>(h, call);
        case 80: return launch_bn<LAYOUT, 80>(h, call);
        case 64: return launch_bn<LAYOUT, 64>(h, call);
        case 48: return launch_bn<LAYOUT, 48>(h, call);
        case 32: return launch_bn<LAYOUT, 32>(h, call);
        case 16: return launch_bn<LAYOUT, 16>(h, call);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

namespace ks {

bool tf32_supports(const ks_handle_s& h, const KsCall& call) {
    if (h.b < 16 || h.c < 16 || h.c % 8 != 0 || pick_bn(h.b) == 0) return false;
    if (h.a * h.d > (int64_t(1) << 30)) return false;
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y);
    if (al & 15) return false;
    if (call.layout == KS_LAYOUT_BSL) return call.B % 4 == 0;
    return h.d == 1;      // BSF with d > 1: FP32 kernels (TF32 gather not built yet)
}

cudaError_t tf32_launch(const ks_handle_s& h, const KsCall& call) {
    return call.layout == KS_LAYOUT_BSL ? launch_layout<KS_LAYOUT_BSL>(h, call)
                                        : launch_layout<KS_LAYOUT_BSF>(h, call);
}

}  // namespace ks
