// Warp-specialised FP32 (CUDA-core FFMA) KS kernel for the layouts whose X
// operand needs no transposition on its way to shared memory: BSL (any d) and
// BSF with d = 1.  Same arithmetic as ks_ffma.cu / the generic kernel (one FP32
// FMA chain per output, l ascending: bit-identical results), different
// machinery:
//
//  * persistent CTAs (2 per SM), tiles = output blocks Y[n0:n0+128,
//    row_{i,j}[k0:k0+BN]] (output-stationary, Alg. 3, each
//    element written once);
//  * X and K^T chunks of 16 l arrive by TMA in an S-slot shared-memory ring
//    (mbarrier with transaction count per slot), running ahead across tile
//    boundaries -- the short reduction of a KS block (c = 48..128, 3-8 chunks)
//    made the register-staged kernel's per-tile prologue and global-load latency
//    visible (22-36% long-scoreboard stalls, ks_ffma.cu).  There is no producer
//    warp: the LAST of the 8 warps to finish reading a slot (shared-memory
//    counter, acq_rel) refills it, so a CTA is 8 warps and two CTAs fit the
//    per-SM-sub-partition register file at 128 registers per thread (a 9th
//    warp would cap them at 96);
//  * warp tile 64 x BN/4, thread micro-tile 8 x TN (TN = BN/16), operands from
//    shared memory, accumulators in registers, the epilogue stores straight from
//    registers while the other warps / the refills keep going.
//
// Operand layouts in shared memory (no permutation pass):
//   A, BSL:  [16 l][128 n] from the 3-D box {128 n, 1 j, 16 l} of X viewed as
//            [a c][d][B]; a thread reads float4 of 4 consecutive n per l.
//   A, BSF:  [128 n][16 l] from the 2-D box {16 l, 128 n}, SWIZZLE_64B; a thread
//            reads float4 of 4 consecutive l for rows ty + 8m (the swizzle puts
//            8 consecutive rows on 8 different bank groups).
//   B:       [16 l][BN k] from k_tile (K^T tiles).
#include "ks_umma.cuh"

namespace {

constexpr int WS_BK = 16;              // l per chunk
constexpr int WS_CWARPS = 8;           // warps per CTA, all compute
constexpr int WS_THREADS = 32 * WS_CWARPS;

// Warps split 2 x 4 (rows x outputs) for BN in {96, 128}: tile 128 rows, TN =
// BN/16; BN in {48, 64} uses 4 x 2 warps: tile 256 rows, TN = 6 / 8 (a 128-row
// tile would leave TN = 3 / 4: 3 shared loads per 32 FFMA instead of 4 per 64).
// KB = l per chunk: 16, or 32 for BN = 96 tiles when c % 32 == 0 (half the ring
// waits / refills per FFMA; the BSF A rows become 128 bytes, SWIZZLE_128B).
// WMX > 0 overrides the warps along the rows (WM x WN = 8): fewer rows per tile for
// problems whose default tiles do not fill the machine (a = d = 1: one b x b block,
// B / 128 tiles for 2 x 148 CTA slots).
template <int LAYOUT, int BN, int KB = WS_BK, int WMX = 0>
struct WsCfg {
    static constexpr int WM = WMX > 0 ? WMX : BN <= 64 ? 4 : 2;   // warps along the batch rows
    static constexpr int WN = 8 / WM;                      // warps along the outputs
    static constexpr int BMW = 64 * WM;                    // batch rows per tile
    static constexpr int TN = BN / (4 * WN);               // outputs per thread
    static constexpr int A_BYTES = KB * BMW * 4;
    static constexpr int B_BYTES = KB * BN * 4;
    static constexpr int SLOT = A_BYTES + B_BYTES;         // multiple of 1 KB (A stays 1 KB aligned)
    static constexpr int S = (108 * 1024) / SLOT > 8 ? 8 : (108 * 1024) / SLOT;
    static constexpr int BAR_OFF = S * SLOT;
    static constexpr int SMEM = BAR_OFF + 8 * 8 + 4 * 8 + 1024;     // full barriers, counters, align pad
    static_assert(BN == 48 || BN == 64 || BN == 96 || BN == 128, "BN");
    static_assert(BN % (4 * WN) == 0, "whole thread columns");
    // odd TN (the split-row tiles of BN = 48 / 96): FFMA2 lanes pair two rows of one
    // output instead of two outputs of one row (same fmaf chain per output)
    static constexpr bool RP = TN % 2 != 0;
    static_assert(SLOT % 1024 == 0, "slot alignment (SWIZZLE_64B A tiles)");
    static_assert(S * KB >= 64, "ring depth (l in flight)");
};

template <int LAYOUT, int BN, int KB = WS_BK, int WMX = 0>
__global__ void __launch_bounds__(WS_THREADS, 2)
ks_ffma_ws_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                  float* __restrict__ Y, const float* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d,
                  int64_t ntiles) {
    using C = WsCfg<LAYOUT, BN, KB, WMX>;
    constexpr int S = C::S;
    constexpr int TN = C::TN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t slot0 = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t cnt0 = smem_u32(&bars[8]);         // S u32 "warps done with slot" counters

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nkc = b / BN;
    constexpr int BMW = C::BMW;
    const int64_t nnb = (B + BMW - 1) / BMW;
    const int nk = c / KB;
    const int64_t M = (int64_t)a * b * d;

    // tile -> (k-chunk fastest, n-block, block q = i*d + j)
    auto decode = [&](int64_t tile, int& q, int& k0, int64_t& n0) {
        k0 = (int)(tile % nkc) * BN;
        tile /= nkc;
        n0 = (tile % nnb) * BMW;
        q = (int)(tile / nnb);
    };
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;             // chunks this CTA consumes
    auto issue = [&](int64_t gx) {               // one thread: TMA of chunk gx into slot gx % S
        int q, k0;
        int64_t n0;
        decode(blockIdx.x + (gx / nk) * gridDim.x, q, k0, n0);
        const int i = q / d, j = q % d;
        const int st = (int)(gx % S);
        const int l0 = (int)(gx % nk) * KB;
        const uint32_t sa = slot0 + st * C::SLOT;
        mbar_expect_tx(full0 + 8 * st, C::SLOT);
        if constexpr (LAYOUT == KS_LAYOUT_BSL)
            tma_3d(sa, &xmap, (int)n0, j, i * c + l0, full0 + 8 * st);
        else
            tma_2d(sa, &xmap, i * c + l0, (int)n0, full0 + 8 * st);
        tma_2d(sa + C::A_BYTES, &kmap, k0, q * c + l0, full0 + 8 * st);
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * s) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    __syncthreads();
    pdl_wait();                 // the prologue above overlaps the previous kernel's drain (PDL)
    pdl_launch_dependents();
    if (tid == 0)
        for (int64_t gx = 0; gx < S && gx < G; ++gx) issue(gx);

    const int wm = warp / C::WN, wn = warp % C::WN;   // WM x WN warps: 64 rows x BN/WN outputs each
    const int ty = lane >> 2, tx = lane & 3;
    const int colB = wn * (BN / C::WN) + tx * TN;
    int64_t g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int q, k0;
        int64_t n0;
        decode(tile, q, k0, n0);
        const int i = q / d, j = q % d;
        constexpr bool RP = C::RP;
        constexpr int A2M = RP ? 4 : 8, A2N = RP ? TN : TN / 2;
        uint64_t acc2[A2M][A2N];                  // (acc[m][2p], acc[m][2p+1]), or (acc[2q][e], acc[2q+1][e]) if RP
#pragma unroll
        for (int m = 0; m < A2M; ++m)
#pragma unroll
            for (int p = 0; p < A2N; ++p) acc2[m][p] = 0;

        for (int t = 0; t < nk; ++t, ++g) {
            const int st = (int)(g % S);
            mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
            const uint32_t sa = slot0 + st * C::SLOT;
            const uint32_t sb = sa + C::A_BYTES + colB * 4;
            if constexpr (LAYOUT == KS_LAYOUT_BSL) {
                // A[l][n]: rows wm*64 + ty*4 + {0..3} and +32
                const uint32_t pa = sa + (wm * 64 + ty * 4) * 4;
#pragma unroll
                for (int l = 0; l < KB; ++l) {
                    float av[8], bv[TN];
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(av[0]), "=f"(av[1]), "=f"(av[2]), "=f"(av[3]) : "r"(pa + l * BMW * 4));
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(av[4]), "=f"(av[5]), "=f"(av[6]), "=f"(av[7]) : "r"(pa + l * BMW * 4 + 128));
                    const uint32_t pb = sb + l * BN * 4;
                    if constexpr (TN % 4 == 0) {
#pragma unroll
                        for (int e = 0; e < TN; e += 4)
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(bv[e]), "=f"(bv[e + 1]), "=f"(bv[e + 2]), "=f"(bv[e + 3])
                                         : "r"(pb + e * 4));
                    } else if constexpr (RP) {        // odd TN: 4-byte aligned columns
#pragma unroll
                        for (int e = 0; e < TN; ++e) bv[e] = lds32(pb + e * 4);
                    } else {
#pragma unroll
                        for (int e = 0; e < TN; e += 2)
                            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(bv[e]), "=f"(bv[e + 1]) : "r"(pb + e * 4));
                    }
                    if constexpr (RP) {               // rows (2q, 2q+1): av[] is 4 consecutive rows per float4
#pragma unroll
                        for (int q = 0; q < 4; ++q)
#pragma unroll
                            for (int e = 0; e < TN; ++e)
                                acc2[q][e] = ffma2(f2pack(av[2 * q], av[2 * q + 1]), f2pack(bv[e], bv[e]), acc2[q][e]);
                    } else {
#pragma unroll
                        for (int m = 0; m < 8; ++m)
#pragma unroll
                            for (int p = 0; p < TN / 2; ++p)
                                acc2[m][p] = ffma2(f2pack(av[m], av[m]), f2pack(bv[2 * p], bv[2 * p + 1]), acc2[m][p]);
                    }
                }
            } else {
                // A[n][l] (64-byte rows, SWIZZLE_64B: 16-byte chunk u of row n at u ^ ((n >> 1) & 3)):
                // rows wm*64 + ty + 8m; one float4 = 4 consecutive l of a row
#pragma unroll
                for (int qd = 0; qd < KB / 4; ++qd) {
                    float4 av[8];
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        const int n = wm * 64 + ty + 8 * m;
                        const int sw = KB == 16 ? (n >> 1) & 3 : n & 7;        // SWIZZLE_64B / 128B
                        const uint32_t addr = sa + n * (KB * 4) + ((qd ^ sw) << 4);
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(av[m].x), "=f"(av[m].y), "=f"(av[m].z), "=f"(av[m].w) : "r"(addr));
                    }
#pragma unroll
                    for (int e4 = 0; e4 < 4; ++e4) {
                        const int l = qd * 4 + e4;
                        float bv[TN];
                        const uint32_t pb = sb + l * BN * 4;
                        if constexpr (TN % 4 == 0) {
#pragma unroll
                            for (int e = 0; e < TN; e += 4)
                                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                             : "=f"(bv[e]), "=f"(bv[e + 1]), "=f"(bv[e + 2]), "=f"(bv[e + 3])
                                             : "r"(pb + e * 4));
                        } else if constexpr (RP) {    // odd TN: 4-byte aligned columns
#pragma unroll
                            for (int e = 0; e < TN; ++e) bv[e] = lds32(pb + e * 4);
                        } else {
#pragma unroll
                            for (int e = 0; e < TN; e += 2)
                                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(bv[e]), "=f"(bv[e + 1]) : "r"(pb + e * 4));
                        }
                        auto comp = [&](int m) {
                            return e4 == 0 ? av[m].x : e4 == 1 ? av[m].y : e4 == 2 ? av[m].z : av[m].w;
                        };
                        if constexpr (RP) {           // rows (2q, 2q+1) = ty + 16q, ty + 16q + 8
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint64_t xp = f2pack(comp(2 * q), comp(2 * q + 1));
#pragma unroll
                                for (int e = 0; e < TN; ++e) acc2[q][e] = ffma2(xp, f2pack(bv[e], bv[e]), acc2[q][e]);
                            }
                        } else {
#pragma unroll
                            for (int m = 0; m < 8; ++m) {
                                const float x = comp(m);
#pragma unroll
                                for (int p = 0; p < TN / 2; ++p)
                                    acc2[m][p] = ffma2(f2pack(x, x), f2pack(bv[2 * p], bv[2 * p + 1]), acc2[m][p]);
                            }
                        }
                    }
                }
            }
            // generic reads of the slot done (fence: before the async-proxy refill);
            // the last warp to get here refills the slot with chunk g + S
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                uint32_t old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt0 + 4 * st)
                             : "memory");
                if (old == WS_CWARPS - 1) {
                    asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * st) : "memory");
                    if (g + S < G) issue(g + S);
                }
            }
        }

        // ---- epilogue: each owned Y element written exactly once ----------------
        float acc[8][TN];
        if constexpr (RP) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int e = 0; e < TN; ++e) {
                    acc[2 * q][e] = f2lo(acc2[q][e]);
                    acc[2 * q + 1][e] = f2hi(acc2[q][e]);
                }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int p = 0; p < TN / 2; ++p) {
                    acc[m][2 * p] = f2lo(acc2[m][p]);
                    acc[m][2 * p + 1] = f2hi(acc2[m][p]);
                }
        }
        if (bias) {                               // KSLinear bias (NEXT-2)
#pragma unroll
            for (int e = 0; e < TN; ++e) {
                const float bq = __ldg(bias + (int64_t)i * b * d + (int64_t)(k0 + colB + e) * d + j);
#pragma unroll
                for (int m = 0; m < 8; ++m) acc[m][e] += bq;
            }
        }
        if (act) {                                // epilogue activation (NEXT-2)
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int e = 0; e < TN; ++e) acc[m][e] = ks_act(acc[m][e], act);
        }
        if constexpr (LAYOUT == KS_LAYOUT_BSL) {
            const int64_t nr = n0 + wm * 64 + ty * 4;
#pragma unroll
            for (int e = 0; e < TN; ++e) {
                const int64_t r = (int64_t)i * b * d + (int64_t)(k0 + colB + e) * d + j;
                float* yr = Y + r * B + nr;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (nr + 32 * h < B)          // B % 4 == 0: a float4 of rows is all in or all out
                        __stcs(reinterpret_cast<float4*>(yr + 32 * h),
                               make_float4(acc[4 * h][e], acc[4 * h + 1][e], acc[4 * h + 2][e], acc[4 * h + 3][e]));
            }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int64_t n = n0 + wm * 64 + ty + 8 * m;
                if (n >= B) continue;
                float* yr = Y + n * M + (int64_t)i * b + k0 + colB;
                if constexpr (TN % 4 == 0) {
#pragma unroll
                    for (int e = 0; e < TN; e += 4)
                        __stcs(reinterpret_cast<float4*>(yr + e),
                               make_float4(acc[m][e], acc[m][e + 1], acc[m][e + 2], acc[m][e + 3]));
                } else if constexpr (RP) {
#pragma unroll
                    for (int e = 0; e < TN; ++e) __stcs(yr + e, acc[m][e]);
                } else {
#pragma unroll
                    for (int e = 0; e < TN; e += 2)
                        __stcs(reinterpret_cast<float2*>(yr + e), make_float2(acc[m][e], acc[m][e + 1]));
                }
            }
        }
    }
}

// ---- BSF, d % 4 == 0: four consecutive j per tile, all four in every thread --
// One TMA box {4 j, 17 l, 64 n} of X viewed as [B][a c][d] per chunk of 16 l
// brings the d-strided columns of 4 KS blocks as 16-byte vectors (the 17th l is
// padding: a staged row is 17 units of 16 bytes, so the 8 consecutive rows a
// warp reads fall on 8 different bank groups).  Instead of transposing the
// staged [n][l][j] chunk, every thread computes all 4 j for its rows: per l it
// reads one float4 (4 j) per row and one K^T vector per j -- 8 shared loads per
// 64 FFMA, no transposer, no extra shared-memory pass (a per-j variant that read
// A element-wise needed 10 loads per 64 FFMA and was slower than the
// register-staged kernel, profiles/r01_exp_ffma_wsj_negative.txt).
// Tile: 64 batch rows x BN outputs x 4 j; warps 2 (rows) x 4 (outputs); thread
// micro-tile 4 rows (ty + 8r) x 4 j x TK outputs, TK = BN / 16.
constexpr int WSG_BM = 64;

template <int TK>
struct WsgCfg {
    static constexpr int BN = 16 * TK;
    static constexpr int PITCH = (WS_BK + 1) * 16;        // staged row: 17 l x 4 j floats
    static constexpr int A_BYTES = WSG_BM * PITCH;         // 17 KB
    static constexpr int BJ_BYTES = WS_BK * BN * 4;        // per j
    static constexpr int SLOT0 = A_BYTES + 4 * BJ_BYTES;
    static constexpr int SLOT = (SLOT0 + 1023) / 1024 * 1024;
    static constexpr int S = (108 * 1024) / SLOT > 8 ? 8 : (108 * 1024) / SLOT;
    static constexpr int BAR_OFF = S * SLOT;
    static constexpr int SMEM = BAR_OFF + 8 * 8 + 4 * 8 + 1024;
    static_assert(TK == 2 || TK == 3 || TK == 4, "TK");
    static_assert(S >= 3, "ring depth");
};

template <int TK>
__global__ void __launch_bounds__(WS_THREADS, 2)
ks_ffma_wsg_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                   float* __restrict__ Y, const float* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d,
                   int64_t ntiles) {
    using C = WsgCfg<TK>;
    constexpr int S = C::S;
    constexpr int BN = C::BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t slot0 = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t cnt0 = smem_u32(&bars[8]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nkc = b / BN;
    const int njg = d / 4;
    const int64_t nnb = (B + WSG_BM - 1) / WSG_BM;
    const int nk = c / WS_BK;
    const int64_t M = (int64_t)a * b * d;

    // tile -> (k-chunk fastest, j-group, n-block, i): the k-chunks and j-groups of
    // one X tile run on neighbouring CTAs at the same time and share it in L2
    auto decode = [&](int64_t tile, int& i, int& j0, int& k0, int64_t& n0) {
        k0 = (int)(tile % nkc) * BN;
        tile /= nkc;
        j0 = (int)(tile % njg) * 4;
        tile /= njg;
        n0 = (tile % nnb) * WSG_BM;
        i = (int)(tile / nnb);
    };
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;
    auto issue = [&](int64_t gx) {
        int i, j0, k0;
        int64_t n0;
        decode(blockIdx.x + (gx / nk) * gridDim.x, i, j0, k0, n0);
        const int st = (int)(gx % S);
        const int l0 = (int)(gx % nk) * WS_BK;
        const uint32_t sa = slot0 + st * C::SLOT;
        mbar_expect_tx(full0 + 8 * st, C::A_BYTES + 4 * C::BJ_BYTES);
        if (d == 4)          // the 17 l x 4 j of a row are one contiguous run: one 272-byte box row
            tma_2d(sa, &xmap, (i * c + l0) * 4, (int)n0, full0 + 8 * st);
        else
            tma_3d(sa, &xmap, j0, i * c + l0, (int)n0, full0 + 8 * st);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
            tma_2d(sa + C::A_BYTES + jj * C::BJ_BYTES, &kmap, k0, (i * d + j0 + jj) * c + l0, full0 + 8 * st);
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * s) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_launch_dependents();
    if (tid == 0)
        for (int64_t gx = 0; gx < S && gx < G; ++gx) issue(gx);

    const int wm = warp >> 2, wn = warp & 3;
    const int ty = lane >> 2, tx = lane & 3;
    const int colB = wn * (4 * TK) + tx * TK;          // first of the thread's TK outputs
    int64_t g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int i, j0, k0;
        int64_t n0;
        decode(tile, i, j0, k0, n0);
        float acc[4][4][TK];                              // [row r][j][output e]
        constexpr int TK2 = TK % 2 == 0 ? TK / 2 : 1;     // FFMA2 pairs of outputs (TK even)
        uint64_t acc2[4][4][TK2];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
                for (int e = 0; e < TK; ++e) acc[r][jj][e] = 0.f;
#pragma unroll
                for (int p = 0; p < TK2; ++p) acc2[r][jj][p] = 0;
            }
        for (int t = 0; t < nk; ++t, ++g) {
            const int st = (int)(g % S);
            mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
            const uint32_t sa = slot0 + st * C::SLOT;
            const uint32_t pa = sa + (wm * 32 + ty) * C::PITCH;        // rows wm*32 + ty + 8r
            const uint32_t pb = sa + C::A_BYTES + colB * 4;
#pragma unroll
            for (int l = 0; l < WS_BK; ++l) {
                float4 av[4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(av[r].x), "=f"(av[r].y), "=f"(av[r].z), "=f"(av[r].w)
                                 : "r"(pa + r * 8 * C::PITCH + l * 16));
                float bv[4][TK];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const uint32_t q = pb + jj * C::BJ_BYTES + l * BN * 4;
                    if constexpr (TK == 4) {
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(bv[jj][0]), "=f"(bv[jj][1]), "=f"(bv[jj][2]), "=f"(bv[jj][3]) : "r"(q));
                    } else if constexpr (TK == 2) {
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(bv[jj][0]), "=f"(bv[jj][1]) : "r"(q));
                    } else {
#pragma unroll
                        for (int e = 0; e < TK; ++e) bv[jj][e] = lds32(q + e * 4);
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const float x[4] = {av[r].x, av[r].y, av[r].z, av[r].w};
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        if constexpr (TK % 2 == 0) {
#pragma unroll
                            for (int p = 0; p < TK2; ++p)
                                acc2[r][jj][p] = ffma2(f2pack(x[jj], x[jj]), f2pack(bv[jj][2 * p], bv[jj][2 * p + 1]),
                                                       acc2[r][jj][p]);
                        } else {
#pragma unroll
                            for (int e = 0; e < TK; ++e) acc[r][jj][e] = fmaf(x[jj], bv[jj][e], acc[r][jj][e]);
                        }
                    }
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                uint32_t old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt0 + 4 * st)
                             : "memory");
                if (old == WS_CWARPS - 1) {
                    asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * st) : "memory");
                    if (g + S < G) issue(g + S);
                }
            }
        }
        // epilogue: the 4 j of one (row, output k) are one 16-byte run of Y
        if constexpr (TK % 2 == 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int p = 0; p < TK2; ++p) {
                        acc[r][jj][2 * p] = f2lo(acc2[r][jj][p]);
                        acc[r][jj][2 * p + 1] = f2hi(acc2[r][jj][p]);
                    }
        }
        const int64_t rbase = (int64_t)i * b * d + (int64_t)(k0 + colB) * d + j0;
        if (bias) {
#pragma unroll
            for (int e = 0; e < TK; ++e) {
                const float4 bq = __ldg(reinterpret_cast<const float4*>(bias + rbase + (int64_t)e * d));
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    acc[r][0][e] += bq.x; acc[r][1][e] += bq.y; acc[r][2][e] += bq.z; acc[r][3][e] += bq.w;
                }
            }
        }
        if (act) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int e = 0; e < TK; ++e) acc[r][jj][e] = ks_act(acc[r][jj][e], act);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t n = n0 + wm * 32 + ty + 8 * r;
            if (n >= B) continue;
            float* yr = Y + n * M + rbase;
#pragma unroll
            for (int e = 0; e < TK; ++e)
                __stcs(reinterpret_cast<float4*>(yr + (int64_t)e * d),
                       make_float4(acc[r][0][e], acc[r][1][e], acc[r][2][e], acc[r][3][e]));
        }
    }
}

template <int TK>
cudaError_t launch_wsg(const ks_handle_s& h, const KsCall& call) {
    using C = WsgCfg<TK>;
    constexpr int BN = C::BN;
    CUtensorMap xmap, kmap;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.b, (cuuint64_t)(h.a * h.d * h.c)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.b * 4};
        const cuuint32_t kb[2] = {BN, WS_BK};
        if (!encode(&kmap, h.k_tile, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    if (h.d == 4) {        // d = 4: 2-D box {17 l x 4 j floats, rows} over the contiguous run (same smem image)
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {4 * (WS_BK + 1), WSG_BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[3] = {(cuuint64_t)h.d, (cuuint64_t)(h.a * h.c), (cuuint64_t)call.B};
        const cuuint64_t xs[2] = {(cuuint64_t)h.d * 4, (cuuint64_t)h.N * 4};
        const cuuint32_t xb[3] = {4, WS_BK + 1, WSG_BM};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    auto kern = ks_ffma_wsg_kernel<TK>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * (h.d / 4) * ((call.B + WSG_BM - 1) / WSG_BM) * h.a;
    int64_t slots = 2 * (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(WS_THREADS), C::SMEM, call.stream, xmap, kmap,
                                         call.Y, call.bias, call.act, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d, ntiles);
    ks::count_launch();
    return e;
}

// ---- BSF, d % 4 == 0, FFMA2: four j per tile, one j per LANE ---------------------
// Same staging as the four-j kernel (one TMA box {4 j, 17 l, 64 n} per chunk of 16 l,
// the K^T tiles of the 4 j), but the 4 lanes of a quad (tx = lane & 3) own j = tx:
// a thread's micro-tile is 8 rows (ty + 8m) x 8 outputs of ONE j, so per l it reads
// 8 scalars of A (rows x its j: the 32 lanes hit 32 distinct banks, row pitch 68
// words) and 2 float4 of its j's K^T row, then 32 FFMA2 -- twice
// the reuse of the four-j kernel, whose 4 rows x 4 j x TK micro-tile needed 8 float4
// loads per 64 FMA (2 bytes of shared memory per FMA: at most half the FFMA rate).
// Warps split the outputs: warp w owns k = 8w .. 8w+7 of the tile (BN = 8 NW).  The
// epilogue transposes each 4 x 4 (k, j) block across the quad with shuffles, so a
// lane writes the 4 j of one (row, k) as one float4 (d = 4: 64 contiguous bytes per
// quad).  The K^T tiles of the 4 j arrive interleaved by ONE 4-D TMA box
// {8 k, 4 j, BN/8 k-groups, 16 l} of k_tile: B[l][k-group][j][8 k], so the 4
// distinct addresses a warp reads per l (one per j) are 32 bytes apart and fall on
// 4 bank groups.  One FP32 FMA chain per output, l ascending: bit-identical.
constexpr int WSL_BM = 64;

template <int NW>
struct WslCfg {
    static constexpr int BN = 8 * NW;
    static constexpr int THREADS = 32 * NW;
    static constexpr int PITCH = (WS_BK + 1) * 16;         // staged row: 17 l x 4 j floats
    static constexpr int A_BYTES = WSL_BM * PITCH;          // 17 KB
    static constexpr int B_BYTES = 4 * WS_BK * BN * 4;      // [16 l][BN/8][4 j][8 k]
    static constexpr int SLOT0 = A_BYTES + B_BYTES;
    static constexpr int SLOT = (SLOT0 + 1023) / 1024 * 1024;
    static constexpr int S = (108 * 1024) / SLOT > 8 ? 8 : (108 * 1024) / SLOT;
    static constexpr int BAR_OFF = S * SLOT;
    static constexpr int SMEM = BAR_OFF + 8 * 8 + 4 * 8 + 1024;
    static_assert(NW == 6 || NW == 8, "BN in {48, 64}");
    static_assert(S >= 3, "ring depth");
};

template <int NW>
__global__ void __launch_bounds__(WslCfg<NW>::THREADS, 2)
ks_ffma_wsl_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                   float* __restrict__ Y, const float* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d,
                   int64_t ntiles) {
    using C = WslCfg<NW>;
    constexpr int S = C::S;
    constexpr int BN = C::BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t slot0 = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t cnt0 = smem_u32(&bars[8]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nkc = b / BN;
    const int njg = d / 4;
    const int64_t nnb = (B + WSL_BM - 1) / WSL_BM;
    const int nk = c / WS_BK;
    const int64_t M = (int64_t)a * b * d;

    auto decode = [&](int64_t tile, int& i, int& j0, int& k0, int64_t& n0) {
        k0 = (int)(tile % nkc) * BN;
        tile /= nkc;
        j0 = (int)(tile % njg) * 4;
        tile /= njg;
        n0 = (tile % nnb) * WSL_BM;
        i = (int)(tile / nnb);
    };
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;
    auto issue = [&](int64_t gx) {
        int i, j0, k0;
        int64_t n0;
        decode(blockIdx.x + (gx / nk) * gridDim.x, i, j0, k0, n0);
        const int st = (int)(gx % S);
        const int l0 = (int)(gx % nk) * WS_BK;
        const uint32_t sa = slot0 + st * C::SLOT;
        mbar_expect_tx(full0 + 8 * st, C::A_BYTES + C::B_BYTES);
        if (d == 4)          // the 17 l x 4 j of a row are one contiguous run: one 272-byte box row
            tma_2d(sa, &xmap, (i * c + l0) * 4, (int)n0, full0 + 8 * st);
        else
            tma_3d(sa, &xmap, j0, i * c + l0, (int)n0, full0 + 8 * st);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(sa + C::A_BYTES), "l"(&kmap), "r"(0), "r"(i * d + j0), "r"(k0 / 8), "r"(l0), "r"(full0 + 8 * st)
            : "memory");
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * s) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_launch_dependents();
    if (tid == 0)
        for (int64_t gx = 0; gx < S && gx < G; ++gx) issue(gx);

    const int ty = lane >> 2, tx = lane & 3;             // rows ty + 8m, j = j0 + tx
    const int colB = warp * 8;                           // outputs k0 + colB .. + 7
    int64_t g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int i, j0, k0;
        int64_t n0;
        decode(tile, i, j0, k0, n0);
        uint64_t acc2[8][4];                             // (acc[m][2p], acc[m][2p+1])
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int p = 0; p < 4; ++p) acc2[m][p] = 0;
        for (int t = 0; t < nk; ++t, ++g) {
            const int st = (int)(g % S);
            mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
            const uint32_t sa = slot0 + st * C::SLOT;
            const uint32_t pa = sa + ty * C::PITCH + tx * 4;                       // row ty, j = tx
            const uint32_t pb = sa + C::A_BYTES + (warp * 4 + tx) * 32;            // B[l][warp][tx][8]
#pragma unroll
            for (int l = 0; l < WS_BK; ++l) {
                float x[8], bv[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) x[m] = lds32(pa + m * 8 * C::PITCH + l * 16);
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(bv[0]), "=f"(bv[1]), "=f"(bv[2]), "=f"(bv[3]) : "r"(pb + l * BN * 16));
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(bv[4]), "=f"(bv[5]), "=f"(bv[6]), "=f"(bv[7]) : "r"(pb + l * BN * 16 + 16));
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        acc2[m][p] = ffma2(f2pack(x[m], x[m]), f2pack(bv[2 * p], bv[2 * p + 1]), acc2[m][p]);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                uint32_t old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt0 + 4 * st)
                             : "memory");
                if (old == NW - 1) {
                    asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * st) : "memory");
                    if (g + S < G) issue(g + S);
                }
            }
        }
        // epilogue: per row m and half h, the quad holds a 4 (k) x 4 (j) block, lane tx
        // with j = tx; after the exchange lane tx holds k = colB + 4h + tx, j = j0 .. j0+3
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int64_t n = n0 + ty + 8 * m;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float blk[4] = {f2lo(acc2[m][2 * h]), f2hi(acc2[m][2 * h]), f2lo(acc2[m][2 * h + 1]),
                                      f2hi(acc2[m][2 * h + 1])};
                float out[4];
#pragma unroll
                for (int sx = 0; sx < 4; ++sx) {           // exchange with the lane tx ^ sx
                    const int want = tx ^ sx;              // the partner's k offset = my j slot
                    const float send = want == 0 ? blk[0] : want == 1 ? blk[1] : want == 2 ? blk[2] : blk[3];
                    const float got = __shfl_xor_sync(0xffffffffu, send, sx);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        if (jj == (tx ^ sx)) out[jj] = got;
                }
                const int64_t r = (int64_t)i * b * d + (int64_t)(k0 + colB + 4 * h + tx) * d + j0;
                if (bias) {
                    const float4 bq = __ldg(reinterpret_cast<const float4*>(bias + r));
                    out[0] += bq.x; out[1] += bq.y; out[2] += bq.z; out[3] += bq.w;
                }
                if (act) {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) out[jj] = ks_act(out[jj], act);
                }
                if (n < B) __stcs(reinterpret_cast<float4*>(Y + n * M + r), make_float4(out[0], out[1], out[2], out[3]));
            }
        }
    }
}

template <int NW>
cudaError_t launch_wsl(const ks_handle_s& h, const KsCall& call) {
    using C = WslCfg<NW>;
    constexpr int BN = C::BN;
    CUtensorMap xmap, kmap;
    if (h.d == 4) {        // d = 4: 2-D box {17 l x 4 j floats, rows} over the contiguous run (same smem image)
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {4 * (WS_BK + 1), WSL_BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[3] = {(cuuint64_t)h.d, (cuuint64_t)(h.a * h.c), (cuuint64_t)call.B};
        const cuuint64_t xs[2] = {(cuuint64_t)h.d * 4, (cuuint64_t)h.N * 4};
        const cuuint32_t xb[3] = {4, WS_BK + 1, WSL_BM};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    {   // k_tile[(q c + l) b + k] as 4-D {8 k, a d q, b/8 k-groups, c l}: box {8, 4, BN/8, 16}
        const cuuint64_t kd[4] = {8, (cuuint64_t)(h.a * h.d), (cuuint64_t)(h.b / 8), (cuuint64_t)h.c};
        const cuuint64_t ks[3] = {(cuuint64_t)(h.c * h.b) * 4, 32, (cuuint64_t)h.b * 4};
        const cuuint32_t kb[4] = {8, 4, BN / 8, WS_BK};
        if (!encode(&kmap, h.k_tile, 4, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    auto kern = ks_ffma_wsl_kernel<NW>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * (h.d / 4) * ((call.B + WSL_BM - 1) / WSL_BM) * h.a;
    int64_t slots = 2 * (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(C::THREADS), C::SMEM, call.stream, xmap,
                                         kmap, call.Y, call.bias, call.act, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d,
                                         ntiles);
    ks::count_launch();
    return e;
}

// warps along the outputs for the lane-j kernel: BN = 64 (8 warps) or 48 (6); 0 = unsupported
int pick_nw_wsl(int64_t b) { return b % 64 == 0 ? 8 : b % 48 == 0 ? 6 : 0; }

// TK (outputs per thread per j) for the 4-j kernel: the widest of 4, 3, 2 with
// 16 TK dividing b; 0 = unsupported.
int pick_tk_wsg(int64_t b) {
    for (int tk : {4, 3, 2})
        if (b % (16 * tk) == 0) return tk;
    return 0;
}

// ---- BSF, d in {2, 3}: all d j per tile, every thread computes all of them ---
// The 16 l x d j values of a chunk are one contiguous run of an X row: 2-D box
// {16 d + 4 floats, RW n} (4 floats of padding: 4d + 1 16-byte units per staged
// row, an odd number, so 8 consecutive rows fall on 8 bank groups).  Per group
// of 4 l a row holds 4d floats = d float4s (element l' * d + j); a thread
// loads them for each of its R rows plus one K^T vector per (l', j), and does
// R x d x TK x 4 FFMA: 12 shared loads per 128 FFMA for d = 2 (R = 8) and 24
// per 192 for d = 3 (R = 4).  Tile RW = 16 R rows x BN outputs x d j; warps 2
// (rows) x 4 (outputs); thread rows ty + 8r (r < R).  The epilogue writes the
// d TK consecutive outputs of a row as float4s.
template <int D, int TK>
struct WscCfg {
    static constexpr int R = D == 2 ? 8 : 4;               // rows per thread
    static constexpr int RW = 16 * R;                      // rows per tile
    static constexpr int BN = 16 * TK;
    static constexpr int PITCH = (WS_BK * D + 4) * 4;
    static constexpr int A_BYTES = RW * PITCH;
    static constexpr int BJ_BYTES = WS_BK * BN * 4;
    static constexpr int SLOT0 = A_BYTES + D * BJ_BYTES;
    static constexpr int SLOT = (SLOT0 + 1023) / 1024 * 1024;
    static constexpr int S = (108 * 1024) / SLOT > 8 ? 8 : (108 * 1024) / SLOT;
    static constexpr int BAR_OFF = S * SLOT;
    static constexpr int SMEM = BAR_OFF + 8 * 8 + 4 * 8 + 1024;
    static_assert(D == 2 || D == 3, "D");
    static_assert(TK == 2 || TK == 3 || TK == 4, "TK");
    static_assert((D * TK) % 2 == 0, "float2 epilogue units");
    static_assert(S >= 3, "ring depth");
};

template <int D, int TK>
__global__ void __launch_bounds__(WS_THREADS, 2)
ks_ffma_wsc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                   float* __restrict__ Y, const float* __restrict__ bias, int act, int64_t B, int a, int b, int c,
                   int64_t ntiles) {
    using C = WscCfg<D, TK>;
    constexpr int S = C::S;
    constexpr int BN = C::BN;
    constexpr int R = C::R;
    constexpr int RW = C::RW;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t slot0 = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t cnt0 = smem_u32(&bars[8]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nkc = b / BN;
    const int64_t nnb = (B + RW - 1) / RW;
    const int nk = c / WS_BK;
    const int64_t M = (int64_t)a * b * D;

    auto decode = [&](int64_t tile, int& i, int& k0, int64_t& n0) {   // k-chunk fastest, n-block, i
        k0 = (int)(tile % nkc) * BN;
        tile /= nkc;
        n0 = (tile % nnb) * RW;
        i = (int)(tile / nnb);
    };
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;
    auto issue = [&](int64_t gx) {
        int i, k0;
        int64_t n0;
        decode(blockIdx.x + (gx / nk) * gridDim.x, i, k0, n0);
        const int st = (int)(gx % S);
        const int l0 = (int)(gx % nk) * WS_BK;
        const uint32_t sa = slot0 + st * C::SLOT;
        mbar_expect_tx(full0 + 8 * st, C::A_BYTES + D * C::BJ_BYTES);
        tma_2d(sa, &xmap, (i * c + l0) * D, (int)n0, full0 + 8 * st);
#pragma unroll
        for (int jj = 0; jj < D; ++jj)
            tma_2d(sa + C::A_BYTES + jj * C::BJ_BYTES, &kmap, k0, (i * D + jj) * c + l0, full0 + 8 * st);
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * s) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_launch_dependents();
    if (tid == 0)
        for (int64_t gx = 0; gx < S && gx < G; ++gx) issue(gx);

    const int wm = warp >> 2, wn = warp & 3;
    const int ty = lane >> 2, tx = lane & 3;
    const int colB = wn * (4 * TK) + tx * TK;
    int64_t g = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int i, k0;
        int64_t n0;
        decode(tile, i, k0, n0);
        float acc[R][D][TK];
        constexpr int TK2 = TK % 2 == 0 ? TK / 2 : 1;     // FFMA2 pairs of outputs (TK even)
        uint64_t acc2[R][D][TK2];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int jj = 0; jj < D; ++jj) {
#pragma unroll
                for (int e = 0; e < TK; ++e) acc[r][jj][e] = 0.f;
#pragma unroll
                for (int p = 0; p < TK2; ++p) acc2[r][jj][p] = 0;
            }
        for (int t = 0; t < nk; ++t, ++g) {
            const int st = (int)(g % S);
            mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
            const uint32_t sa = slot0 + st * C::SLOT;
            const uint32_t pa = sa + (wm * (8 * R) + ty) * C::PITCH;       // rows wm*8R + ty + 8r
            const uint32_t pb = sa + C::A_BYTES + colB * 4;
#pragma unroll
            for (int lq = 0; lq < WS_BK / 4; ++lq) {
                float bv[4][D][TK];                       // [l' of the quad][j][e]
#pragma unroll
                for (int h = 0; h < 4; ++h)
#pragma unroll
                    for (int jj = 0; jj < D; ++jj) {
                        const uint32_t q = pb + jj * C::BJ_BYTES + (4 * lq + h) * BN * 4;
                        if constexpr (TK == 4) {
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(bv[h][jj][0]), "=f"(bv[h][jj][1]), "=f"(bv[h][jj][2]), "=f"(bv[h][jj][3])
                                         : "r"(q));
                        } else if constexpr (TK == 2) {
                            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(bv[h][jj][0]), "=f"(bv[h][jj][1]) : "r"(q));
                        } else {
#pragma unroll
                            for (int e = 0; e < TK; ++e) bv[h][jj][e] = lds32(q + e * 4);
                        }
                    }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float x[4 * D];                       // x[l' * D + j]
#pragma unroll
                    for (int u = 0; u < D; ++u)
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(x[4 * u]), "=f"(x[4 * u + 1]), "=f"(x[4 * u + 2]), "=f"(x[4 * u + 3])
                                     : "r"(pa + r * 8 * C::PITCH + (lq * D + u) * 16));
#pragma unroll
                    for (int h = 0; h < 4; ++h)
#pragma unroll
                        for (int jj = 0; jj < D; ++jj) {
                            if constexpr (TK % 2 == 0) {
                                const float xv = x[h * D + jj];
#pragma unroll
                                for (int p = 0; p < TK2; ++p)
                                    acc2[r][jj][p] = ffma2(f2pack(xv, xv), f2pack(bv[h][jj][2 * p], bv[h][jj][2 * p + 1]),
                                                           acc2[r][jj][p]);
                            } else {
#pragma unroll
                                for (int e = 0; e < TK; ++e)
                                    acc[r][jj][e] = fmaf(x[h * D + jj], bv[h][jj][e], acc[r][jj][e]);
                            }
                        }
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                uint32_t old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt0 + 4 * st)
                             : "memory");
                if (old == WS_CWARPS - 1) {
                    asm volatile("st.shared.u32 [%0], 0;" ::"r"(cnt0 + 4 * st) : "memory");
                    if (g + S < G) issue(g + S);
                }
            }
        }
        // epilogue: outputs (k, j), k in [k0+colB, +TK), j < D, are D TK consecutive floats
        if constexpr (TK % 2 == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int jj = 0; jj < D; ++jj)
#pragma unroll
                    for (int p = 0; p < TK2; ++p) {
                        acc[r][jj][2 * p] = f2lo(acc2[r][jj][p]);
                        acc[r][jj][2 * p + 1] = f2hi(acc2[r][jj][p]);
                    }
        }
        const int64_t rbase = (int64_t)i * b * D + (int64_t)(k0 + colB) * D;
        if (bias) {
#pragma unroll
            for (int e = 0; e < TK; ++e)
#pragma unroll
                for (int jj = 0; jj < D; ++jj) {
                    const float bq = __ldg(bias + rbase + D * e + jj);
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r][jj][e] += bq;
                }
        }
        if (act) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int jj = 0; jj < D; ++jj)
#pragma unroll
                    for (int e = 0; e < TK; ++e) acc[r][jj][e] = ks_act(acc[r][jj][e], act);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t n = n0 + wm * (8 * R) + ty + 8 * r;
            if (n >= B) continue;
            float* yr = Y + n * M + rbase;
            float o[D * TK];
#pragma unroll
            for (int e = 0; e < TK; ++e)
#pragma unroll
                for (int jj = 0; jj < D; ++jj) o[D * e + jj] = acc[r][jj][e];
#pragma unroll
            for (int u = 0; u < D * TK; u += 2) __stcs(reinterpret_cast<float2*>(yr + u), make_float2(o[u], o[u + 1]));
        }
    }
}

template <int D, int TK>
cudaError_t launch_wsc(const ks_handle_s& h, const KsCall& call) {
    using C = WscCfg<D, TK>;
    constexpr int BN = C::BN;
    CUtensorMap xmap, kmap;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.b, (cuuint64_t)(h.a * h.d * h.c)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.b * 4};
        const cuuint32_t kb[2] = {BN, WS_BK};
        if (!encode(&kmap, h.k_tile, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {(cuuint32_t)(WS_BK * D + 4), (cuuint32_t)C::RW};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    auto kern = ks_ffma_wsc_kernel<D, TK>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * ((call.B + C::RW - 1) / C::RW) * h.a;
    int64_t slots = 2 * (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(WS_THREADS), C::SMEM, call.stream, xmap, kmap,
                                         call.Y, call.bias, call.act, call.B, (int)h.a, (int)h.b, (int)h.c, ntiles);
    ks::count_launch();
    return e;
}

// TK for the all-j kernel: as pick_tk_wsg, but d TK even (float2 epilogue units).
int pick_tk_wsc(int64_t b, int64_t d) {
    for (int tk : {4, 3, 2})
        if (b % (16 * tk) == 0 && (d * tk) % 2 == 0) return tk;
    return 0;
}

template <int D>
cudaError_t launch_wsc_tk(const ks_handle_s& h, const KsCall& call) {
    switch (pick_tk_wsc(h.b, D)) {
        case 4: return launch_wsc<D, 4>(h, call);
        case 3: if constexpr ((D * 3) % 2 == 0) return launch_wsc<D, 3>(h, call); break;
        case 2: return launch_wsc<D, 2>(h, call);
    }
    return cudaErrorInvalidValue;
}

template <int LAYOUT, int BN, int KB = WS_BK, int WMX = 0>
cudaError_t launch_ws(const ks_handle_s& h, const KsCall& call) {
    using C = WsCfg<LAYOUT, BN, KB, WMX>;
    CUtensorMap xmap, kmap;
    {
        // k_tile: [(i*d + j)*c + l][k], b floats per row
        const cuuint64_t kd[2] = {(cuuint64_t)h.b, (cuuint64_t)(h.a * h.d * h.c)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.b * 4};
        const cuuint32_t kb[2] = {BN, KB};
        if (!encode(&kmap, h.k_tile, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    if (LAYOUT == KS_LAYOUT_BSL) {
        const cuuint64_t xd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c)};
        const cuuint64_t xs[2] = {(cuuint64_t)call.B * 4, (cuuint64_t)(h.d * call.B) * 4};
        const cuuint32_t xb[3] = {(cuuint32_t)C::BMW, 1, KB};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {KB, (cuuint32_t)C::BMW};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, KB == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    auto kern = ks_ffma_ws_kernel<LAYOUT, BN, KB, WMX>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * ((call.B + C::BMW - 1) / C::BMW) * (h.a * h.d);
    int64_t slots = 2 * (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(WS_THREADS), C::SMEM, call.stream, xmap, kmap,
                                         call.Y, call.bias, call.act, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d, ntiles);
    ks::count_launch();
    return e;
}

int pick_bn_ws(int64_t b) {
    for (int bn : {128, 96, 64, 48})
        if (b % bn == 0) return bn;
    return 0;
}

// Underfilled launches (fewer default tiles than 2 CTAs x SMs, e.g. a = d = 1 with
// B = 25088: 196 tiles of 128 rows for 296 slots, the last 48 SMs running two
// tiles while 100 run one) take tiles of half the rows (BN = 128: 64 rows, thread
// micro-tile 8 x 4; BN = 96, BSL: 64 rows, 8 x 3 with row-pair FFMA2; BN = 64: 128
// rows): the busiest SM then holds 1.5 default tiles' work instead of 2
// (BN = 48 splits measured 0.85-1.13x: not used).  KS_FFMA_SPLITM=0 disables (experiments).
bool ws_split_rows(const ks_handle_s& h, const KsCall& call, int bn) {
    static const bool on = [] {
        const char* e = getenv("KS_FFMA_SPLITM");
        return !(e && atoi(e) == 0);
    }();
    if (!on || bn == 0) return false;
    const int64_t rows = bn > 64 ? 128 : 256;
    const int64_t tiles = (h.b / bn) * ((call.B + rows - 1) / rows) * (h.a * h.d);
    return tiles < 2 * (int64_t)ks::num_sms(h.device);   // (not the KS_TF32_MAXGRID test cap: the shape stays)
}

template <int LAYOUT, int KB>
cudaError_t launch_ws_kb(const ks_handle_s& h, const KsCall& call) {
    const int bn = pick_bn_ws(h.b);
    if (KB == WS_BK && ws_split_rows(h, call, bn)) {
        switch (bn) {
            case 128: return launch_ws<LAYOUT, 128, KB, 1>(h, call);
            case 96:         // TN = 3: row-pair FFMA2; BSL only (BSF's A rows need a pack per pair:
                             // (1,96,96,1) BSF 0.93x, BSL 1.16x, profiles/r03/oddtn_time.jsonl)
                if constexpr (LAYOUT == KS_LAYOUT_BSL) return launch_ws<LAYOUT, 96, KB, 1>(h, call);
                break;
            case 64: return launch_ws<LAYOUT, 64, KB, 2>(h, call);
        }
    }
    switch (bn) {
        case 128: return launch_ws<LAYOUT, 128, KB>(h, call);
        case 96: return launch_ws<LAYOUT, 96, KB>(h, call);
        case 64: return launch_ws<LAYOUT, 64, KB>(h, call);
        case 48: return launch_ws<LAYOUT, 48, KB>(h, call);
    }
    return cudaErrorInvalidValue;
}

template <int LAYOUT>
cudaError_t launch_ws_layout(const ks_handle_s& h, const KsCall& call) {
    // 32 l per staged chunk pays only for b = 96 tiles (9-12 %: BSL (2,96,96,16) 365 -> 327 us,
    // BSF (64,96,96,1) 839 -> 745 us); elsewhere it is 0-10 % slower
    // (profiles/r01_ffma_kb32_negative.txt).  KS_FFMA_KB32=0 disables.
    if ((call.knobs & KS_KNOB_KB32) && h.c % 32 == 0 && pick_bn_ws(h.b) == 96)
        return LAYOUT == KS_LAYOUT_BSL && ws_split_rows(h, call, 96) ? launch_ws<LAYOUT, 96, 32, 1>(h, call)
                                                                     : launch_ws<LAYOUT, 96, 32>(h, call);
    return launch_ws_kb<LAYOUT, WS_BK>(h, call);
}

}  // namespace

namespace ks {

// BSL (any d) or BSF with d = 1: b a multiple of 48 or 64.  BSF with d % 4 == 0
// (four-j kernel, 16-byte aligned bias) or d in {2, 3} (all-j contiguous kernel):
// b a multiple of 32 or 48 (d = 3: of 32).  c a multiple
// of 16; 16-byte aligned X / Y; 32-bit TMA coordinates.  KS_FFMA_WS=0 /
// KS_FFMA_WSG=0 disable (experiments).
bool ffma_ws_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (!(call.knobs & KS_KNOB_FFMA_WS) || h.dtype != KS_DTYPE_F32) return false;
    if (call.layout == KS_LAYOUT_BSF && h.d > 1) {            // four-j kernel (d % 4 == 0)
        if (!(call.knobs & KS_KNOB_FFMA_WSG) || h.c % WS_BK != 0) return false;
        if (h.d % 4 == 0 ? pick_tk_wsg(h.b) == 0 : (h.d > 3 || pick_tk_wsc(h.b, h.d) == 0)) return false;
        if (h.d % 4 == 0 && (reinterpret_cast<uintptr_t>(call.bias) & 15) != 0) return false;
    } else if (pick_bn_ws(h.b) == 0 || h.c % WS_BK != 0) {
        return false;
    }
    if (h.a * h.d * h.c >= (int64_t(1) << 31) || call.B >= (int64_t(1) << 31)) return false;
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y);
    if (al & 15) return false;
    if (call.layout == KS_LAYOUT_BSL && call.B % 4 != 0) return false;
    return true;
}

cudaError_t ffma_ws_launch(const ks_handle_s& h, const KsCall& call) {
    if (call.layout == KS_LAYOUT_BSL) return launch_ws_layout<KS_LAYOUT_BSL>(h, call);
    if (h.d == 2) return launch_wsc_tk<2>(h, call);        // all d j per thread
    if (h.d == 3) return launch_wsc_tk<3>(h, call);
    if (h.d > 1) {
        if ((call.knobs & KS_KNOB_FFMA_WSL) && pick_nw_wsl(h.b) != 0)
            return pick_nw_wsl(h.b) == 8 ? launch_wsl<8>(h, call) : launch_wsl<6>(h, call);
        switch (pick_tk_wsg(h.b)) {
            case 4: return launch_wsg<4>(h, call);
            case 3: return launch_wsg<3>(h, call);
            case 2: return launch_wsg<2>(h, call);
        }
        return cudaErrorInvalidValue;
    }
    return launch_ws_layout<KS_LAYOUT_BSF>(h, call);
}

}  // namespace ks
