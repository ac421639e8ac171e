// TF32 tensor-core KS kernel (tcgen05.mma.kind::tf32, accumulators in TMEM)
// for the GEMM-like patterns where each (i, j) block is a genuine dense
// contraction (b, c >= 16; north star).  Not in the paper, whose kernel is
// CUDA-core only: on B200 the FP32 FFMA path is ALU-bound
// for b, c >= 48 (arithmetic intensity bc/(2(b+c)) above the FFMA ridge), so
// the tensor cores turn these factors HBM-bound again.
//
// Work unit ("tile") = output block Y[n0:n0+128, row_{i,j}[k0:k0+BN]]
// (output-stationary, Alg. 3; each element written once).
//   UMMA view:  D[m][n] = sum_k A[m][k] B[n][k],  M = 128 batch rows,
//               N = BN outputs (k index of the KS block), K = l (c).
//   A = X[n0:n0+128, col_{i,j}], B = K[row_{i,j}, col_{i,j}] (k_tf32,
//   pre-rounded RNA at pack time, [q][k][l]); both K-major in shared memory
//   in the canonical no-swizzle layout (8-row x 16-byte core matrices).
//   (tcgen05 ignores the "MN-major" bit for kind::tf32 -- measured, see
//   scripts/probe_umma.cu -- so batch-contiguous BSL tiles are transposed on
//   the way in.)
// Persistent CTAs (grid <= 2 per SM), tiles round-robin; warp roles
// (288 threads):
//   warps 0-3  producers: X and K chunks (128 x 32 l, BN x 32 l) into a
//              STAGES-deep smem ring (mbarrier full/empty).  K and the
//              ld-contiguous BSF X tile go by cp.async 16 B; BSL X is read
//              as coalesced 4-byte columns and written transposed (STS.128).
//   warp 4     TMEM allocator + single-thread MMA issuer (double-buffered
//              accumulator: 2 x BN TMEM columns).
//   warps 5-8  epilogue: tcgen05.ld 32x32b -> registers -> coalesced global
//              stores in the caller's layout, overlapping the next tile's MMAs.
// X is fed as raw FP32 bits (the tensor core reads the TF32 part: truncation
// of the 13 low mantissa bits); FP32 accumulation.  Contract: normwise error
// <= 5e-3 (north star); DESIGN.md derives the per-element envelope.
#include "ks_internal.h"

namespace {

constexpr int BM = 128;       // batch rows per tile = UMMA M
constexpr int BKC = 32;       // l per pipeline stage (4 UMMA k-steps of 8)
constexpr int NPROD = 128;    // producer threads (warps 0-3)
constexpr int NEPI = 128;     // epilogue threads (warps 5-8)
constexpr int NTHREADS = NPROD + 32 + NEPI;

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
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// Shared-memory matrix descriptor, no swizzle: start, LBO, SBO, version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
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

template <int BN>
struct Tf32Cfg {
    static constexpr int A_BYTES = BM * BKC * 4;          // 16 KB
    static constexpr int B_BYTES = BN * BKC * 4;          // BN * 128 B
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = BN <= 64 ? 4 : BN <= 128 ? 3 : 2;
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM = STAGES * STAGE + BAR_BYTES;
    static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                   : 2 * BN <= 256 ? 256 : 512;
    static constexpr int CTAS_PER_SM = TMEM_COLS <= 256 ? 2 : 1;
    static_assert(BN % 16 == 0 && BN <= 256, "UMMA N for M=128");
};

struct TileCoord {
    int i, j, k0;
    int64_t n0;
    int64_t q;
};

__device__ __forceinline__ TileCoord decode(int64_t tile, int nkc, int64_t nnb, int d, int BN) {
    TileCoord t;
    const int kc = (int)(tile % nkc);
    tile /= nkc;
    t.n0 = (tile % nnb) * BM;
    t.q = tile / nnb;
    t.i = (int)(t.q / d);
    t.j = (int)(t.q % d);
    t.k0 = kc * BN;
    return t;
}

// K-major smem tile (rows r, K index l in [0,32)):  (r/8)*1024 + (l/4)*128 + (r%8)*16 + (l%4)*4
//   -> LBO (next 4-l chunk) = 128 B, SBO (next 8-row group) = 1024 B.
template <int LAYOUT, int BN>
__global__ void __launch_bounds__(NTHREADS, Tf32Cfg<BN>::CTAS_PER_SM)
ks_tf32_kernel(const float* __restrict__ X, const float* __restrict__ Kt32, float* __restrict__ Y,
               int64_t B, int a, int b, int c, int d, int64_t ntiles) {
    using C = Tf32Cfg<BN>;
    constexpr int S = C::STAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::STAGE);
    // [0,S) full  [S,2S) empty  [2S,2S+2) acc_full  [2S+2,2S+4) acc_empty  [2S+4] tmem slot
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accf0 = smem_u32(&bars[2 * S]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + 2]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 4]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int nkc = b / BN;
    const int64_t nnb = (B + BM - 1) / BM;
    const int64_t N = (int64_t)a * c * d, M = (int64_t)a * b * d;
    const int nk = (c + BKC - 1) / BKC;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, NPROD);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, NEPI);
        }
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
        // ============================ producers ============================
        // flat chunk index g over this CTA's tiles: tile = blockIdx.x + (g / nk) * gridDim.x
        const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
        const int64_t G = my_tiles * nk;
        float v[BKC];                                    // BSL: next chunk's column, prefetched
        auto load_bsl = [&](int64_t gg) {
            const TileCoord tc = decode(blockIdx.x + (gg / nk) * gridDim.x, nkc, nnb, d, BN);
            const int l0 = (int)(gg % nk) * BKC;
            const int64_t n = tc.n0 + tid;
            const bool nok = n < B;
            const float* xr = X + ((int64_t)tc.i * c * d + tc.j) * B + (nok ? n : 0);
            const int64_t ls = (int64_t)d * B;           // stride between consecutive l
#pragma unroll
            for (int l = 0; l < BKC; ++l) v[l] = (nok && l0 + l < c) ? __ldcs(xr + (int64_t)(l0 + l) * ls) : 0.f;
        };
        if (LAYOUT == KS_LAYOUT_BSL && G > 0) load_bsl(0);
        for (int64_t g = 0; g < G; ++g) {
            const TileCoord tc = decode(blockIdx.x + (g / nk) * gridDim.x, nkc, nnb, d, BN);
            const float* kt = Kt32 + (tc.q * b + tc.k0) * c;          // [k][l] rows of this tile
            const int t = (int)(g % nk);
            {
                const int st = (int)(g % S);
                if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                const uint32_t sa = smem0 + st * C::STAGE;
                const uint32_t sb = sa + C::A_BYTES;
                const int l0 = t * BKC;
                if (LAYOUT == KS_LAYOUT_BSL) {
                    // thread = batch row: its 32 l values (column loads, coalesced across the
                    // warp) go out as 8 K-major 16-B chunks; then prefetch the next chunk
#pragma unroll
                    for (int l4 = 0; l4 < BKC / 4; ++l4)
                        sts128(sa + (tid / 8) * 1024 + l4 * 128 + (tid % 8) * 16, v[4 * l4], v[4 * l4 + 1],
                               v[4 * l4 + 2], v[4 * l4 + 3]);
                    if (g + 1 < G) load_bsl(g + 1);
                } else {
                    // BSF, d = 1: row n, l contiguous: 16-B chunks straight into place
#pragma unroll
                    for (int r = 0; r < (BM * BKC / 4) / NPROD; ++r) {
                        const int idx = tid + r * NPROD;
                        const int l4 = idx % (BKC / 4), m = idx / (BKC / 4);
                        const int64_t n = tc.n0 + m;
                        const bool ok = (l0 + 4 * l4 < c) && (n < B);
                        const float* src = X + (ok ? n : 0) * N + (int64_t)tc.i * c + (ok ? l0 + 4 * l4 : 0);
                        cp_async16(sa + (m / 8) * 1024 + l4 * 128 + (m % 8) * 16, src, ok ? 16u : 0u);
                    }
                }
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
                // retire chunk g-(S-1): its cp.async have landed (wait_group) and this
                // thread's generic-proxy writes are made visible to the async proxy
                if (g >= S - 1) {
                    cp_async_wait<S - 1>();
                    fence_proxy_async();
                    mbar_arrive(full0 + 8 * (int)((g - (S - 1)) % S));
                }
            }
        }
        cp_async_wait<0>();
        fence_proxy_async();
        for (int64_t u = (G > S - 1 ? G - (S - 1) : 0); u < G; ++u) mbar_arrive(full0 + 8 * (int)(u % S));
    } else if (warp == 4) {
        // ============================ MMA issuer ============================
        if ((tid & 31) == 0) {
            constexpr uint32_t idesc = make_idesc(BN);
            int64_t g = 0;
            int64_t it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int ab = (int)(it & 1);
                if (it >= 2) mbar_wait(acce0 + 8 * ab, (uint32_t)(((it / 2) - 1) & 1));
                tc_fence_after();
                const uint32_t dtm = tmem + (uint32_t)(ab * BN);
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
                    tc_fence_after();
                    const uint32_t sa = smem0 + st * C::STAGE;
                    const uint32_t sb = sa + C::A_BYTES;
                    const int ksteps = min(BKC / 8, (c - t * BKC) / 8);
                    for (int s = 0; s < ksteps; ++s) {
                        mma_tf32(dtm, make_desc(sa + s * 256, 128, 1024), make_desc(sb + s * 256, 128, 1024),
                                 idesc, (t > 0 || s > 0) ? 1u : 0u);
                    }
                    mma_commit(empty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
            }
        }
        __syncwarp();
    } else {
        // ============================ epilogue ============================
        const int lq = warp & 3;                          // TMEM lane quarter this warp may access
        const int row = lq * 32 + (tid & 31);
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const TileCoord tc = decode(tile, nkc, nnb, d, BN);
            const int ab = (int)(it & 1);
            mbar_wait(accf0 + 8 * ab, (uint32_t)((it / 2) & 1));
            tc_fence_after();
            const int64_t n = tc.n0 + row;
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * BN);
#pragma unroll 1
            for (int col = 0; col < BN; col += 16) {
                float v[16];
                tmem_ld16(tbase + col, v);
                if (n < B) {
                    if (LAYOUT == KS_LAYOUT_BSL) {
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const int64_t r = (int64_t)tc.i * b * d + (int64_t)(tc.k0 + col + e) * d + tc.j;
                            __stcs(Y + r * B + n, v[e]);
                        }
                    } else {
                        float* yp = Y + n * M + (int64_t)tc.i * b + tc.k0 + col;
#pragma unroll
                        for (int e = 0; e < 16; e += 4)
                            __stcs(reinterpret_cast<float4*>(yp + e), make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acce0 + 8 * ab);
        }
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
    const int64_t ntiles = (h.b / BN) * ((call.B + BM - 1) / BM) * (h.a * h.d);
    const int64_t slots = (int64_t)ks::num_sms(h.device) * C::CTAS_PER_SM;
    const int64_t grid = ntiles < slots ? ntiles : slots;
    kern<<<(unsigned)grid, NTHREADS, C::SMEM, call.stream>>>(call.X, h.k_tf32, call.Y, call.B, (int)h.a,
                                                              (int)h.b, (int)h.c, (int)h.d, ntiles);
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
    if (call.layout == KS_LAYOUT_BSL) return (al & 3) == 0;
    return h.d == 1 && (al & 15) == 0;   // BSF d > 1: FP32 kernels (TF32 gather not built yet)
}

cudaError_t tf32_launch(const ks_handle_s& h, const KsCall& call) {
    return call.layout == KS_LAYOUT_BSL ? launch_layout<KS_LAYOUT_BSL>(h, call)
                                        : launch_layout<KS_LAYOUT_BSF>(h, call);
}

}  // namespace ks
