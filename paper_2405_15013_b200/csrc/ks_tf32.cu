// TF32 tensor-core KS kernel (tcgen05.mma.kind::tf32, accumulators in TMEM,
// operands staged by TMA) for the GEMM-like patterns where each (i, j) block
// is a genuine dense contraction (b, c >= 16; north star).  Not in the paper,
// whose kernel is CUDA-core only: on B200 the FP32 FFMA
// path is ALU-bound for b, c >= 48 (arithmetic intensity bc/(2(b+c)) above the
// FFMA ridge), so the tensor cores turn these factors HBM-bound again.
//
// Work unit ("tile") = output block Y[n0:n0+128, row_{i,j}[k0:k0+BN]]
// (output-stationary, Alg. 3; each element written once).
//   UMMA view:  D[m][n] = sum_k A[m][k] B[n][k],  M = 128 batch rows,
//               N = BN outputs (k index of the KS block), K = l (c).
//   A = X[n0:n0+128, col_{i,j}],  B = K[row_{i,j}, col_{i,j}] (k_tf32: rows of
//   c values, pre-rounded RNA at pack time).  Both K-major, 128-byte swizzled
//   (the layout TMA SWIZZLE_128B produces), 32 l per pipeline stage.
// Operand movement (no permutation pass):
//   * B:            TMA 2-D box {32 l, BN rows} from k_tf32.
//   * A, BSF d = 1: TMA 2-D box {32 l, 128 rows} straight from X (rows of N).
//   * A, BSL:       TMA 3-D box {128 batch, 1 j, 32 l} of X viewed as
//                   [a*c][d][B] into a staging ring; tcgen05 ignores the
//                   MN-major bit for kind::tf32 (measured: scripts/probe_umma.cu),
//                   so 4 transposer warps rewrite each staged chunk K-major
//                   (32 LDS.32 + 8 conflict-free STS.128 per thread).
// Persistent CTAs (one per SM), tiles round-robin; 320 threads:
//   warp 0      lane 0: X/A TMA issuer, lane 1: B TMA issuer
//   warps 1-4   BSL transposers
//   warp 5      TMEM allocator + single-thread MMA issuer (double-buffered
//               accumulator, 2 x BN TMEM columns)
//   warps 6-9   epilogue: tcgen05.ld 32x32b -> registers -> coalesced global
//               stores in the caller's layout, overlapping the next tile.
// X is fed as raw FP32 bits (the tensor core uses the TF32 part: truncation of
// the 13 low mantissa bits); FP32 accumulation.  Contract: normwise error
// <= 5e-3 (north star); R9/R10 give the per-element envelope.
#include "ks_umma.cuh"

namespace {

constexpr int NTRANS = 128;    // transposer threads (warps 1-4)
constexpr int NEPI = 128;      // epilogue threads (warps 6-9)
constexpr int NTHREADS = 320;

// RB = bytes of K per operand row per stage: 128 (SWIZZLE_128B; TF32 32 l, half
// 64 l) or 64 (SWIZZLE_64B, 16 l) for the 3xTF32 split (X3), whose doubled A
// and B tiles would not leave room for two CTAs per SM at 128.
// OUTL: layout of Y (= LAYOUT except for the mixed-layout calls of ks_matmul_io
// and chain intermediates: BSF in / BSL out, or BSL in / BSF out with d = 1).
// MNA (BSL, FP32 TF32 only): A is loaded MN-major by TMA straight into the
// operand slot (4 boxes {32 n, 1 j, 32 l}, SWIZZLE_128B_ATOM_32B) and the MMA
// reads it with an MN-major descriptor: no staging ring, no transposer warps.
template <int LAYOUT, int BN, bool X3 = false, int OUTL = LAYOUT, bool MNA = false>
struct Tf32Cfg {
    static constexpr int RB = X3 ? 64 : 128;
    static constexpr int A_TILE = BM * RB;                // 16 KB (8 KB for X3)
    static constexpr int B_TILE = BN * RB;
    static constexpr int NA = X3 ? 2 : 1;                 // X3: A = x (raw) and x_lo; B = k_hi and k_lo
    static constexpr int A_BYTES = NA * A_TILE;
    static constexpr int B_BYTES = NA * B_TILE;
    static constexpr int SLOT = A_BYTES + B_BYTES;
    static constexpr int STG = BM * RB;                   // BSL staging chunk [RB/4 l][128 n] (FP32)
    // Two co-resident CTAs per SM (TMEM 2 x 2*BN <= 512 columns, ~110 KB smem each)
    // measured ~1.4x faster than one deep-pipelined CTA: more independent
    // tiles in flight hide TMA latency better than a deeper ring.
    static constexpr int CTAS = BN <= 128 ? 2 : 1;                                // CTAs per SM
    static constexpr int BUDGET = CTAS == 2 ? 110 * 1024 : 200 * 1024;
    static constexpr int P = MNA ? 0 : LAYOUT == KS_LAYOUT_BSL ? (CTAS == 2 ? (BN <= 64 || X3 ? 3 : 2) : 3) : 0;   // staging
    // BSF: 4 epilogue warps x 32 rows x (4 + 1) 16-byte units of store scratch (WarpStore<float, 1, 16>)
    static constexpr int SCR = OUTL == KS_LAYOUT_BSL ? 0 : 4 * 32 * 5 * 16;
    static constexpr int S_FIT = (BUDGET - P * STG - SCR) / SLOT;
    static constexpr int S = S_FIT > 6 ? 6 : S_FIT;                              // operand slots
    static constexpr int SCR_OFF = S * SLOT + P * STG;
    static constexpr int BAR_OFF = SCR_OFF + SCR;
    static constexpr int SMEM = BAR_OFF + 256 + 1024;                            // + barriers + align pad
    static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                   : 2 * BN <= 256 ? 256 : 512;
    static_assert(BN % 16 == 0 && BN <= 256, "UMMA N for M=128");
    static_assert(S >= 2, "pipeline too shallow");
    static_assert((3 * S + 4 + 2 * (P > 0 ? P : 1)) * 8 + 4 <= 256, "barrier area");
    static_assert(!MNA || (LAYOUT == KS_LAYOUT_BSL && !X3), "MN-major A: BSL TF32");
};

template <int RB>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t addr) {
    if constexpr (RB == 128) return sw128_desc(addr);
    else return sw64_desc(addr);
}

// 3xTF32 (X3) split of x: hi = rna_tf32(x), lo = rna_tf32(x - hi) (x - hi is
// exact in FP32), so x = hi + lo up to 2^-22 |x| and the MMA's own TF32 read of
// both parts is exact.
__device__ __forceinline__ uint32_t rna_tf32(uint32_t xbits) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(__uint_as_float(xbits)));
    return r;
}
__device__ __forceinline__ void tf32_split(uint32_t x, uint32_t& hi, uint32_t& lo) {
    hi = rna_tf32(x);
    lo = rna_tf32(__float_as_uint(__uint_as_float(x) - __uint_as_float(hi)));
}

struct TileCoord {
    int i, j, k0;
    int n0;
    int q;
};

__device__ __forceinline__ TileCoord decode(int64_t tile, int nkc, int64_t nnb, int d, int BN) {
    TileCoord t;
    const int kc = (int)(tile % nkc);
    tile /= nkc;
    t.n0 = (int)(tile % nnb) * BM;
    t.q = (int)(tile / nnb);
    t.i = t.q / d;
    t.j = t.q % d;
    t.k0 = kc * BN;
    return t;
}

// TSTD (FP32 Y in BSF, d = 1): each epilogue warp's 32-row x 16-output chunk goes out by
// one TMA tensor store of a dense [32][16] box (2 KB, in the warp_store_rows scratch)
// instead of warp_store_rows' shared-memory transpose + 16-byte warp stores.
template <int LAYOUT, int BN, typename T = float, bool X3 = false, int OUTL = LAYOUT, bool MNA = false,
          bool TSTD = false>
__global__ void __launch_bounds__(NTHREADS, Tf32Cfg<LAYOUT, BN, X3, OUTL, MNA>::CTAS)
ks_tf32_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
               const __grid_constant__ CUtensorMap kmap_lo, const __grid_constant__ CUtensorMap ymap,
               T* __restrict__ Y, const T* __restrict__ bias,
               int64_t B, int a, int b, int c, int d, int64_t ntiles, int flags) {
    // flags: bits 0-7 = KS_TF32_DEBUG experiment switches, bits 8-15 = epilogue activation
    const int dbg = flags & 0xFF, act = (flags >> 8) & 0xFF;
    using C = Tf32Cfg<LAYOUT, BN, X3, OUTL, MNA>;
    static_assert(LAYOUT != KS_LAYOUT_BSL || sizeof(T) == 4, "half BSL runs the swap-AB kernel (ks_half_bsl.cu)");
    constexpr bool STAGED = LAYOUT == KS_LAYOUT_BSL && !MNA;    // X through the staging ring + transposers
    static_assert(!X3 || sizeof(T) == 4, "3xTF32 is an FP32 mode");
    constexpr int RB = C::RB;
    constexpr int BKC = RB / (int)sizeof(T);         // K elements per stage (one operand row)
    constexpr int KSTEP = 32 / (int)sizeof(T);       // K elements per MMA
    constexpr int NCH = RB / 16;                     // 16-byte chunks per operand row
    constexpr int S = C::S;
    constexpr int P = C::P > 0 ? C::P : 1;      // (BSF: no staging; P only names unused barriers)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    // [0,S) full  [S,2S) empty  [2S,2S+2) acc_full  [2S+2,2S+4) acc_empty
    // [2S+4, 2S+4+P) stg_full  [.., +P) stg_empty  [.., +S) split_full (BSF X3)  then the TMEM slot
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accf0 = smem_u32(&bars[2 * S]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + 2]);
    const uint32_t sfull0 = smem_u32(&bars[2 * S + 4]);
    const uint32_t sempty0 = smem_u32(&bars[2 * S + 4 + P]);
    const uint32_t xfull0 = smem_u32(&bars[2 * S + 4 + 2 * P]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[3 * S + 4 + 2 * P]);
    const uint32_t slot0 = smem_u32(smem);                 // S x (A tiles | B tiles), 1 KB aligned
    const uint32_t stg0 = slot0 + S * C::SLOT;             // P x staging (BSL)
    const uint32_t scr0 = slot0 + C::SCR_OFF;              // BSF epilogue store scratch

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int nkc = b / BN;
    const int64_t nnb = (B + BM - 1) / BM;
    const int64_t M = (int64_t)a * b * d;
    const int nk = (c + BKC - 1) / BKC;
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;
    // the MMA waits for the transposers (BSL), the splitters (BSF X3) or the TMA (BSF)
    constexpr bool SPLIT = X3 && LAYOUT != KS_LAYOUT_BSL;
    const uint32_t ready0 = SPLIT ? xfull0 : full0;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, STAGED ? 1 + NTRANS : 2);
            mbar_init(empty0 + 8 * s, 1);
            mbar_init(xfull0 + 8 * s, NTRANS);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, NEPI);
        }
        for (int p = 0; p < P; ++p) {
            mbar_init(sfull0 + 8 * p, 1);  // staging ring (BSL)
            mbar_init(sempty0 + 8 * p, NTRANS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
        if (X3) asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap_lo) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                 // the prologue above overlaps the previous kernel's drain (PDL)
    pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            // One thread issues every TMA.  BSL: the X staging ring runs P-1 chunks
            // ahead of the operand slots; BSF: A and B land in the same slot.
            auto issue_x = [&](int64_t gx) {     // BSL staging chunk gx
                const TileCoord tc = decode(blockIdx.x + (gx / nk) * gridDim.x, nkc, nnb, d, BN);
                const int l0 = (int)(gx % nk) * BKC;
                const int p = (int)(gx % P);
                if (gx >= P) mbar_wait(sempty0 + 8 * p, (uint32_t)(((gx / P) - 1) & 1));
                mbar_expect_tx(sfull0 + 8 * p, C::STG);
                tma_3d(stg0 + p * C::STG, &xmap, tc.n0, tc.j, tc.i * c + l0, sfull0 + 8 * p);
            };
            if (STAGED)
                for (int64_t gx = 0; gx < P - 1 && gx < G; ++gx) issue_x(gx);
            for (int64_t g = 0; g < G; ++g) {
                if (STAGED && g + P - 1 < G) issue_x(g + P - 1);
                const TileCoord tc = decode(blockIdx.x + (g / nk) * gridDim.x, nkc, nnb, d, BN);
                const int l0 = (int)(g % nk) * BKC;
                const int st = (int)(g % S);
                if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                const uint32_t sa = slot0 + st * C::SLOT;
                if (LAYOUT != KS_LAYOUT_BSL) {
                    mbar_expect_tx(full0 + 8 * st, C::A_TILE);
                    tma_2d(sa, &xmap, tc.i * c + l0, tc.n0, full0 + 8 * st);
                } else if constexpr (MNA) {   // MN-major A: 4 boxes of 32 batch columns x 32 l
                    mbar_expect_tx(full0 + 8 * st, C::A_TILE);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        tma_3d(sa + q4 * 4096, &xmap, tc.n0 + 32 * q4, tc.j, tc.i * c + l0, full0 + 8 * st);
                }
                mbar_expect_tx(full0 + 8 * st, C::B_BYTES);
                tma_2d(sa + C::A_BYTES, &kmap, l0, tc.q * b + tc.k0, full0 + 8 * st);
                if (X3) tma_2d(sa + C::A_BYTES + C::B_TILE, &kmap_lo, l0, tc.q * b + tc.k0, full0 + 8 * st);
            }
        }
    } else if (warp <= 4) {
        const int r = tid - 32;                                    // batch row in the tile
        const uint32_t rowoff = (uint32_t)((r / 8) * (8 * RB) + (r % 8) * RB);
        const int sw = RB == 128 ? (r % 8) : (r % 8) / 2;          // SW128 / SW64 chunk XOR
        if constexpr (STAGED) {
            // ---------------- BSL transposers: staging [l][n] -> K-major A (and x_lo for X3) ----------------
            for (int64_t g = 0; g < G; ++g) {
                const int p = (int)(g % P);
                mbar_wait(sfull0 + 8 * p, (uint32_t)((g / P) & 1));
                // column r of the staged [BKC l][128 n] chunk, as 32-bit words
                uint32_t w[BKC];
                const uint32_t src = stg0 + p * C::STG + 4 * r;
#pragma unroll
                for (int l = 0; l < BKC; ++l)
                    w[l] = (dbg & 2) ? 0u : __float_as_uint(lds32(src + l * (BM * 4)));
                fence_proxy_async();      // generic reads before the TMA (async proxy) refill
                mbar_arrive(sempty0 + 8 * p);
                const int st = (int)(g % S);
                if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                const uint32_t dst = slot0 + st * C::SLOT + rowoff;
                if constexpr (X3) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        uint32_t hi[4], lo[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) tf32_split(w[4 * ch + e], hi[e], lo[e]);
                        sts128(dst + ((ch ^ sw) * 16), __uint_as_float(hi[0]), __uint_as_float(hi[1]),
                               __uint_as_float(hi[2]), __uint_as_float(hi[3]));
                        sts128(dst + C::A_TILE + ((ch ^ sw) * 16), __uint_as_float(lo[0]), __uint_as_float(lo[1]),
                               __uint_as_float(lo[2]), __uint_as_float(lo[3]));
                    }
                } else {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch)
                        sts128(dst + ((ch ^ sw) * 16), __uint_as_float(w[4 * ch]), __uint_as_float(w[4 * ch + 1]),
                               __uint_as_float(w[4 * ch + 2]), __uint_as_float(w[4 * ch + 3]));
                }
                fence_proxy_async();
                mbar_arrive(full0 + 8 * st);
            }
        } else if constexpr (SPLIT) {
            // ---------------- BSF X3 splitters: A (x, TMA-loaded) -> hi in place + lo tile ----------------
            for (int64_t g = 0; g < G; ++g) {
                const int st = (int)(g % S);
                mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
                const uint32_t base = slot0 + st * C::SLOT + rowoff;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {        // same swizzled position in both tiles;
                    const uint32_t off = ((ch ^ sw) * 16);    // visiting chunks in XOR order is conflict-free
                    uint32_t v[4], hi[4], lo[4];
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(base + off));
#pragma unroll
                    for (int e = 0; e < 4; ++e) tf32_split(v[e], hi[e], lo[e]);
                    sts128(base + off, __uint_as_float(hi[0]), __uint_as_float(hi[1]), __uint_as_float(hi[2]),
                           __uint_as_float(hi[3]));
                    sts128(base + C::A_TILE + off, __uint_as_float(lo[0]), __uint_as_float(lo[1]),
                           __uint_as_float(lo[2]), __uint_as_float(lo[3]));
                }
                fence_proxy_async();
                mbar_arrive(xfull0 + 8 * st);
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_t<T>(BN) | (MNA ? 1u << 15 : 0u);   // bit 15: A MN-major
            int64_t g = 0;
            int64_t it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int ab = (int)(it & 1);
                if (it >= 2) mbar_wait(acce0 + 8 * ab, (uint32_t)(((it / 2) - 1) & 1));
                tc_fence_after();
                const uint32_t dtm = tmem + (uint32_t)(ab * BN);
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait(ready0 + 8 * st, (uint32_t)((g / S) & 1));
                    tc_fence_after();
                    const uint32_t sa = slot0 + st * C::SLOT;
                    const uint32_t sb = sa + C::A_BYTES;
                    const int ksteps = min(BKC / KSTEP, (c - t * BKC) / KSTEP);
                    for (int s = 0; s < ksteps; ++s) {
                        const uint32_t acc = (t > 0 || s > 0) ? 1u : 0u;
                        if constexpr (X3) {
                            // x k ~ x_lo k_hi + x_hi k_lo + x_hi k_hi (all operands exact TF32)
                            mma_tf32(dtm, kmajor_desc<RB>(sa + C::A_TILE + 32 * s), kmajor_desc<RB>(sb + 32 * s),
                                     idesc, acc);
                            mma_tf32(dtm, kmajor_desc<RB>(sa + 32 * s), kmajor_desc<RB>(sb + C::B_TILE + 32 * s),
                                     idesc, 1u);
                            mma_tf32(dtm, kmajor_desc<RB>(sa + 32 * s), kmajor_desc<RB>(sb + 32 * s), idesc, 1u);
                        } else if constexpr (MNA) {   // k-step s = rows 8s.. of each 32-l box; boxes 4 KB apart
                            mma_tf32(dtm, mn_sw128_32b_desc(sa + 1024 * s, 4096, 512), kmajor_desc<RB>(sb + 32 * s),
                                     idesc, acc);
                        } else if constexpr (sizeof(T) == 4) {
                            mma_tf32(dtm, kmajor_desc<RB>(sa + 32 * s), kmajor_desc<RB>(sb + 32 * s), idesc, acc);
                        } else {
                            mma_f16(dtm, kmajor_desc<RB>(sa + 32 * s), kmajor_desc<RB>(sb + 32 * s), idesc, acc);
                        }
                    }
                    mma_commit(empty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue ----------------
        const int lq = warp & 3;                          // TMEM lane quarter this warp may access
        const int row = lq * 32 + lane;
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const TileCoord tc = decode(tile, nkc, nnb, d, BN);
            const int ab = (int)(it & 1);
            mbar_wait(accf0 + 8 * ab, (uint32_t)((it / 2) & 1));
            tc_fence_after();
            const int64_t n = (int64_t)tc.n0 + row;
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * BN);
#pragma unroll 1
            for (int col = 0; col < BN; col += 16) {
                float vv[1][16];
                float* v = vv[0];
                tmem_ld16(tbase + col, v);
                if (bias) {                       // KSLinear bias (NEXT-2), per output row r
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        v[e] += ElemTraits<T>::to_f(bias[(int64_t)tc.i * b * d + (int64_t)(tc.k0 + col + e) * d + tc.j]);
                }
                if (act) {                        // epilogue activation (NEXT-2), after the bias
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = ks_act(v[e], act);
                }
                if constexpr (OUTL != KS_LAYOUT_BSL && TSTD) {
                    // dense box [32 rows][16 floats]: lane = row, 64-byte rows; lane n writes its
                    // 4 chunks rotated by n mod 4 (a phase's 8 lanes on 4+4 bank groups)
                    static_assert(sizeof(T) == 4, "FP32 Y");
                    const uint32_t buf = scr0 + (uint32_t)(warp - 6) * 2048u;
                    float w[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int x = 0; x < 4; ++x) w[u][x] = v[4 * u + x];
                    const int rot = lane & 3;
#pragma unroll
                    for (int sb = 1; sb < 4; sb <<= 1) {
                        const bool on = rot & sb;
                        float t[4][4];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int x = 0; x < 4; ++x) t[u][x] = on ? w[(u + sb) & 3][x] : w[u][x];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int x = 0; x < 4; ++x) w[u][x] = t[u][x];
                    }
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        sts128(buf + (uint32_t)lane * 64u + (uint32_t)((u + rot) & 3) * 16u, w[u][0], w[u][1], w[u][2],
                               w[u][3]);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0 && !(dbg & 1)) {
                        tma_store_2d(&ymap, tc.i * b + tc.k0 + col, tc.n0 + lq * 32, buf);
                        bulk_commit();
                    }
                } else if constexpr (OUTL != KS_LAYOUT_BSL) {
                    // BSF out (d = 1): row n's 16 outputs are contiguous; coalesce through scratch
                    if constexpr (sizeof(T) == 4) {
                        if (dbg & 4) {            // experiment: direct stores, no shared-memory staging
                            direct_store_rows<1, 16>(vv, Y, (int64_t)tc.n0 + lq * 32, B, M,
                                                     (int64_t)tc.i * b + tc.k0 + col, 1, lane);
                            continue;
                        }
                    }
                    if (!(dbg & 1))
                        warp_store_rows<T, 1, 16>(scr0 + (uint32_t)(warp - 6) * WarpStore<float, 1, 16>::BYTES, vv, Y,
                                                  (int64_t)tc.n0 + lq * 32, B, M, (int64_t)tc.i * b + tc.k0 + col, 1, lane);
                } else if (n < B && !(dbg & 1)) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int64_t r = (int64_t)tc.i * b * d + (int64_t)(tc.k0 + col + e) * d + tc.j;
                        __stcs(Y + r * B + n, v[e]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acce0 + 8 * ab);
        }
    }
    if constexpr (TSTD) {
        if (warp >= 6 && lane == 0) bulk_wait_all();     // this thread's TMA stores have completed
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    }
}

// ==========================================================================
// BSF with d > 1: J j-values per tile.  In BSF the d-strided columns of the
// blocks (i, j0 .. j0+J-1) are gathered by ONE TMA box per pipeline stage:
//   J = d (d <= 8): the BKJ*d values X[n, (i*c + l0)*d .. (i*c + l0 + BKJ)*d)
//       of every row are one contiguous run -> 2-D box {BKJ*d + 4, 128 n}: every
//       loaded byte is used (the 4 extra floats are padding, see below);
//   J = 4 or 8 (d % J == 0, d > 8): 3-D box {J j, BKJ+1 l, 128 n} of X viewed
//       as [B][a*c][d]: 4*J-byte runs (J = 4 reads half of each 32-byte sector,
//       the other half belongs to the next j-group, which runs next and hits L2).
// Either way a staged row n is [BKJ l][J j] floats plus 16 bytes, so its pitch
// is an odd number of 16-byte units and the transposers' 16-byte reads of 8
// consecutive rows hit 8 different bank groups.  Transposer warps split the
// staged chunk into J K-major A tiles (SWIZZLE_32B for BKJ = 8, 64B for 16);
// the MMA warp runs J accumulators of BN columns (NACC x J x BN <= 512 TMEM
// columns; NACC = 2 double-buffers the accumulators so the epilogue overlaps
// the next tile, NACC = 1 lets BN cover the whole block so X is read once --
// the ring of S stages keeps prefetching while the epilogue drains).  The
// epilogue stores through warp_store_rows (coalesced 16-byte units; direct
// per-row stores touched 32 sectors per instruction, 4x ideal).
// ==========================================================================
// INL / OUTL: layouts of X and Y.  INL = BSL (the mixed BSL-in / BSF-out calls
// of ks_matmul_io and chain intermediates): one 3-D TMA box {128 n, J j, BKJ l}
// of X viewed as [a*c][d][B] per stage, staged [l][j][n] (each j's run of 128
// batch values is 512 contiguous bytes: no gather), and the transposers read
// it with conflict-free 4-byte loads.  OUTL = BSL: the epilogue writes each
// output row r = (i, k, j) of Y^T as 128-byte warp stores (lane = batch row).
// TST (BSF out): the epilogue stages each warp's 32-row x EC-output x J chunk in a
// dense box buffer (one per warp, <= warp_store_rows' scratch) and stores it with one TMA tensor store
// (cp.async.bulk.tensor shared -> global), instead of warp_store_rows' 16-byte
// warp stores: the d-strided 16/32-byte runs of Y are written by the TMA engine
// and the epilogue warps move on to the next chunk (SURVEY 8a-6 "TMA store").
// MNJ (BSL in, FP32 TF32): each j's A tile [32 l][128 n] arrives MN-major straight
// from TMA (4 boxes {32 n, 1 j, 32 l}, SWIZZLE_128B_ATOM_32B, as the d = 1 kernel's
// MNA) -- no staging ring, no transposer warps: the whole ring is operand slots,
// so X in flight is S - 1 stages of J x 16 KB instead of one 32 KB staging chunk
// (the transposers of the staged kernel waited for X half of their time).  BKJ = 32.
template <int J, int BN, int BKJ, bool X3 = false, bool GATHER = false, int INL = KS_LAYOUT_BSF,
          int OUTL = KS_LAYOUT_BSF, bool TST = false, bool MNJ = false>
struct Tf32JCfg {
    static constexpr int RB = BKJ * 4;                    // operand row bytes (SW32 / SW64; SW128 for MNJ)
    static constexpr int NA = X3 ? 2 : 1;                 // hi (+ lo) tiles
    static constexpr int AJ_TILE = BM * RB;               // per j
    static constexpr int BJ_TILE = BN * RB;
    static constexpr int SLOT = J * NA * (AJ_TILE + BJ_TILE);
    // staged row: [BKJ l][J j] + padding: 4 floats past the run (2-D box), or one
    // more l (3-D box; J = 8 then gives an even pitch: 2-way read conflicts)
    static constexpr int STG_ROW = INL == KS_LAYOUT_BSL ? BKJ * J * 4 : GATHER ? (BKJ + 1) * J * 4 : BKJ * J * 4 + 16;
    static constexpr int STG = MNJ ? 0 : BM * STG_ROW;
    static constexpr int NACC = 2 * J * BN <= 512 ? 2 : 1;
    static constexpr int EC = J > 2 ? 8 : 16;             // epilogue columns per TMEM load
    static constexpr int TBOX = 32 * EC * J * 4;                        // TMA store box (TST), 1 KB multiple
    static constexpr int SCR = OUTL == KS_LAYOUT_BSL ? 0 : TST ? 4 * TBOX : 4 * WarpStore<float, J, EC>::BYTES;
    // X staging ring: ~96 KB of X loads in flight per SM (Little's law: ~45 GB/s
    // per SM x ~2 us loaded latency), leaving room for 2 operand slots; measured:
    // P = 2 at BKJ = 8 (36 KB in flight) left the J = 3 kernel latency-bound.
    static constexpr int P_WANT = MNJ ? 1 : (96 * 1024 + STG - 1) / STG;
    static constexpr int P_ROOM = MNJ ? 1 : (214 * 1024 - 2 * SLOT - SCR) / STG;
    static constexpr int P_MIN = P_WANT < P_ROOM ? P_WANT : P_ROOM;
    static constexpr int P = MNJ ? 1 : P_MIN < 2 ? 2 : P_MIN > 8 ? 8 : P_MIN;   // (MNJ: barriers only)
    static constexpr int S_FIT = (214 * 1024 - P * STG - SCR) / SLOT;
    static constexpr int S = S_FIT > 6 ? 6 : S_FIT;
    static constexpr int SCR_OFF = (S * SLOT + P * STG + 1023) / 1024 * 1024;   // TMA store boxes: 1 KB aligned
    static constexpr int BAR_OFF = SCR_OFF + SCR;
    static constexpr int SMEM = BAR_OFF + 256 + 1024;
    static constexpr int COLS = NACC * J * BN;
    static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
    static_assert(SMEM <= 227 * 1024, "shared memory");
    static_assert(!TST || (OUTL == KS_LAYOUT_BSF && J == 8 && TBOX % 1024 == 0), "TMA store boxes");
    static_assert(J * BN <= 512 && BN % 16 == 0 && BN <= 256, "J accumulators in TMEM");
    static_assert(MNJ ? (BKJ == 32 && INL == KS_LAYOUT_BSL && !X3) : (BKJ == 8 || BKJ == 16), "operand rows");
    static_assert((BKJ * J) % 4 == 0, "whole 16-byte staging reads");
    static_assert(S >= 2, "pipeline too shallow");
    static_assert((2 * S + 2 * NACC + 2 * P) * 8 + 4 <= 256, "barrier area");
};

template <int RB>
__device__ __forceinline__ uint64_t kmajor_desc_j(uint32_t addr) {
    if constexpr (RB == 128) return sw128_desc(addr);
    else if constexpr (RB == 64) return sw64_desc(addr);
    else return sw32_desc(addr);
}

struct TileJ {
    int i, j0, k0, n0;
};

__device__ __forceinline__ TileJ decode_j(int64_t tile, int nkc, int njg, int64_t nnb, int BN, int J) {
    TileJ t;
    t.k0 = (int)(tile % nkc) * BN;
    tile /= nkc;
    t.j0 = (int)(tile % njg) * J;               // j-groups of one (i, n-block) run back to back
    tile /= njg;
    t.n0 = (int)(tile % nnb) * BM;
    t.i = (int)(tile / nnb);
    return t;
}

template <int J, int BN, int BKJ, bool X3 = false, bool GATHER = false, int INL = KS_LAYOUT_BSF,
          int OUTL = KS_LAYOUT_BSF, bool TST = false, bool MNJ = false>
__global__ void __launch_bounds__(NTHREADS, 1)
ks_tf32_bsfj_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                    const __grid_constant__ CUtensorMap kmap_lo, const __grid_constant__ CUtensorMap ymap,
                    float* __restrict__ Y,
                    const float* __restrict__ bias, int64_t B, int a, int b, int c, int d, int64_t ntiles,
                    int flags) {
    // flags: bits 0-7 = KS_TF32_DEBUG experiment switches, bits 8-15 = epilogue activation
    const int dbg = flags & 0xFF, act = (flags >> 8) & 0xFF;
    using C = Tf32JCfg<J, BN, BKJ, X3, GATHER, INL, OUTL, TST, MNJ>;
    static_assert(INL == KS_LAYOUT_BSF || !GATHER, "BSL input needs no gather");
    constexpr int S = C::S;
    constexpr int P = C::P;
    constexpr int RB = C::RB;
    constexpr int NACC = C::NACC;
    constexpr int NCH = RB / 16;                  // 16-byte chunks per A row
    constexpr int NV = BKJ * J / 4;               // 16-byte staging reads per row
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accf0 = smem_u32(&bars[2 * S]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + NACC]);
    const uint32_t sfull0 = smem_u32(&bars[2 * S + 2 * NACC]);
    const uint32_t sempty0 = smem_u32(&bars[2 * S + 2 * NACC + P]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 2 * NACC + 2 * P]);
    // slot: [A hi (J j)] [A lo (J j), X3] [B hi (J j)] [B lo (J j), X3]
    const uint32_t slot0 = smem_u32(smem);
    const uint32_t stg0 = slot0 + S * C::SLOT;    // P x staging
    const uint32_t scr0 = slot0 + C::SCR_OFF;     // epilogue store scratch
    constexpr int A_ALL = J * C::NA * C::AJ_TILE;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int nkc = b / BN;
    const int njg = d / J;
    // KS_TF32_DEBUG bit 3 (profiling only, results overwritten): per-role clock64
    // barrier-wait counters written over Y[blockIdx.x * 32 ..] at the end
    // (scripts/prof_roles.py)
    const bool prof = dbg & 8;
    __shared__ unsigned long long pc[16];
    if (prof && tid < 16) pc[tid] = 0;
    unsigned long long w0 = 0, w1 = 0;
    const unsigned long long tk0 = clock64();
    auto pwait = [&](uint32_t bar, uint32_t par, unsigned long long& acc) {
        if (prof) {
            const unsigned long long t0 = clock64();
            mbar_wait(bar, par);
            acc += clock64() - t0;
        } else {
            mbar_wait(bar, par);
        }
    };
    const int64_t nnb = (B + BM - 1) / BM;
    const int64_t M = (int64_t)a * b * d;
    const int nk = c / BKJ;                       // c % BKJ == 0
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, MNJ ? 2 : 1 + NTRANS);      // MNJ: the two expect_tx arrivals (B, A)
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int s = 0; s < NACC; ++s) {
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, NEPI);
        }
        for (int p = 0; p < P; ++p) {
            mbar_init(sfull0 + 8 * p, 1);
            mbar_init(sempty0 + 8 * p, NTRANS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
        if (X3) asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap_lo) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                 // the prologue above overlaps the previous kernel's drain (PDL)
    pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            auto issue_x = [&](int64_t gx) {
                const TileJ tc = decode_j(blockIdx.x + (gx / nk) * gridDim.x, nkc, njg, nnb, BN, J);
                const int l0 = (int)(gx % nk) * BKJ;
                const int p = (int)(gx % P);
                if (gx >= P) pwait(sempty0 + 8 * p, (uint32_t)(((gx / P) - 1) & 1), w0);
                mbar_expect_tx(sfull0 + 8 * p, C::STG);
                if constexpr (INL == KS_LAYOUT_BSL)
                    tma_3d(stg0 + p * C::STG, &xmap, tc.n0, tc.j0, tc.i * c + l0, sfull0 + 8 * p);
                else if constexpr (GATHER)
                    tma_3d(stg0 + p * C::STG, &xmap, tc.j0, tc.i * c + l0, tc.n0, sfull0 + 8 * p);
                else
                    tma_2d(stg0 + p * C::STG, &xmap, (tc.i * c + l0) * d, tc.n0, sfull0 + 8 * p);
            };
            if constexpr (!MNJ)
                for (int64_t gx = 0; gx < P - 1 && gx < G; ++gx) issue_x(gx);
            for (int64_t g = 0; g < G; ++g) {
                if constexpr (!MNJ)
                    if (g + P - 1 < G) issue_x(g + P - 1);
                const TileJ tc = decode_j(blockIdx.x + (g / nk) * gridDim.x, nkc, njg, nnb, BN, J);
                const int l0 = (int)(g % nk) * BKJ;
                const int st = (int)(g % S);
                if (g >= S) pwait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1), w1);
                mbar_expect_tx(full0 + 8 * st, J * C::NA * C::BJ_TILE);
                if constexpr (MNJ) {      // A of each j: 4 boxes of 32 batch columns x 32 l, MN-major
                    mbar_expect_tx(full0 + 8 * st, A_ALL);
                    const uint32_t sa = slot0 + st * C::SLOT;
                    for (int jj = 0; jj < J; ++jj)
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            tma_3d(sa + jj * C::AJ_TILE + q4 * 4096, &xmap, tc.n0 + 32 * q4, tc.j0 + jj,
                                   tc.i * c + l0, full0 + 8 * st);
                }
                const uint32_t sb = slot0 + st * C::SLOT + A_ALL;
                for (int jj = 0; jj < J; ++jj) {
                    const int row = ((tc.i * d + tc.j0 + jj) * b) + tc.k0;
                    tma_2d(sb + jj * C::BJ_TILE, &kmap, l0, row, full0 + 8 * st);
                    if (X3) tma_2d(sb + (J + jj) * C::BJ_TILE, &kmap_lo, l0, row, full0 + 8 * st);
                }
            }
        }
    } else if (warp <= 4) {
        if constexpr (!MNJ) {     // (MNJ: no staging, A arrives MN-major)
            // staging row r: [BKJ l][J j] floats -> J K-major A rows of BKJ l (+ J lo rows for X3)
            const int r = tid - 32;
            const uint32_t rowoff = (uint32_t)((r / 8) * (8 * RB) + (r % 8) * RB);
            const int sw = RB == 64 ? (r % 8) / 2 : (r % 8) / 4;       // SW64 / SW32 chunk XOR
            for (int64_t g = 0; g < G; ++g) {
                const int p = (int)(g % P);
                pwait(sfull0 + 8 * p, (uint32_t)((g / P) & 1), w0);
                float v[BKJ * J];                     // v[l * J + j]
                const uint32_t src = stg0 + p * C::STG + r * C::STG_ROW;
                if (dbg & 2) {                // profiling experiment: skip the staging reads
    #pragma unroll
                    for (int q = 0; q < 4 * NV; ++q) v[q] = 0.f;
                } else if constexpr (INL == KS_LAYOUT_BSL) {   // staged [l][j][n]: column r
    #pragma unroll
                    for (int q = 0; q < BKJ * J; ++q) v[q] = lds32(stg0 + p * C::STG + (uint32_t)(q * BM + r) * 4);
                } else {
    #pragma unroll
                    for (int q = 0; q < NV; ++q)
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                                     : "r"(src + q * 16));
                }
                fence_proxy_async();          // generic reads before the TMA (async proxy) refill
                mbar_arrive(sempty0 + 8 * p);
                const int st = (int)(g % S);
                if (g >= S) pwait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1), w1);
                const uint32_t sa = slot0 + st * C::SLOT + rowoff;
    #pragma unroll
                for (int jj = 0; jj < J; ++jj)
    #pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        const uint32_t off = jj * C::AJ_TILE + ((ch ^ sw) * 16);
                        const float x0 = v[(4 * ch) * J + jj], x1 = v[(4 * ch + 1) * J + jj];
                        const float x2 = v[(4 * ch + 2) * J + jj], x3 = v[(4 * ch + 3) * J + jj];
                        if constexpr (X3) {
                            uint32_t hi[4], lo[4];
                            tf32_split(__float_as_uint(x0), hi[0], lo[0]);
                            tf32_split(__float_as_uint(x1), hi[1], lo[1]);
                            tf32_split(__float_as_uint(x2), hi[2], lo[2]);
                            tf32_split(__float_as_uint(x3), hi[3], lo[3]);
                            sts128(sa + off, __uint_as_float(hi[0]), __uint_as_float(hi[1]), __uint_as_float(hi[2]),
                                   __uint_as_float(hi[3]));
                            sts128(sa + J * C::AJ_TILE + off, __uint_as_float(lo[0]), __uint_as_float(lo[1]),
                                   __uint_as_float(lo[2]), __uint_as_float(lo[3]));
                        } else {
                            sts128(sa + off, x0, x1, x2, x3);
                        }
                    }
                fence_proxy_async();
                mbar_arrive(full0 + 8 * st);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc(BN) | (MNJ ? 1u << 15 : 0u);   // bit 15: A MN-major
            int64_t g = 0, it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int ab = (int)(it % NACC);
                if (it >= NACC) pwait(acce0 + 8 * ab, (uint32_t)(((it / NACC) - 1) & 1), w0);
                tc_fence_after();
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    pwait(full0 + 8 * st, (uint32_t)((g / S) & 1), w1);
                    tc_fence_after();
                    const uint32_t sa = slot0 + st * C::SLOT;
                    const uint32_t sb = sa + A_ALL;
#pragma unroll
                    for (int jj = 0; jj < J; ++jj) {
                        const uint32_t dtm = tmem + (uint32_t)((ab * J + jj) * BN);
#pragma unroll
                        for (int s = 0; s < BKJ / 8; ++s) {
                            const uint32_t acc = (t > 0 || s > 0) ? 1u : 0u;
                            const uint32_t ah = sa + jj * C::AJ_TILE + 32 * s, bh = sb + jj * C::BJ_TILE + 32 * s;
                            if constexpr (X3) {    // x_lo k_hi + x_hi k_lo + x_hi k_hi
                                mma_tf32(dtm, kmajor_desc_j<RB>(ah + J * C::AJ_TILE), kmajor_desc_j<RB>(bh), idesc, acc);
                                mma_tf32(dtm, kmajor_desc_j<RB>(ah), kmajor_desc_j<RB>(bh + J * C::BJ_TILE), idesc, 1u);
                                mma_tf32(dtm, kmajor_desc_j<RB>(ah), kmajor_desc_j<RB>(bh), idesc, 1u);
                            } else if constexpr (MNJ) {   // k-step s = l rows 8s.. of each 32-l box; boxes 4 KB apart
                                mma_tf32(dtm, mn_sw128_32b_desc(sa + jj * C::AJ_TILE + 1024 * s, 4096, 512),
                                         kmajor_desc_j<RB>(bh), idesc, acc);
                            } else {
                                mma_tf32(dtm, kmajor_desc_j<RB>(ah), kmajor_desc_j<RB>(bh), idesc, acc);
                            }
                        }
                    }
                    mma_commit(empty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
            }
        }
        __syncwarp();
    } else {
        constexpr int EC = C::EC;
        const int lq = warp & 3;
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const TileJ tc = decode_j(tile, nkc, njg, nnb, BN, J);
            const int ab = (int)(it % NACC);
            pwait(accf0 + 8 * ab, (uint32_t)((it / NACC) & 1), w0);
            tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * J * BN);
#pragma unroll 1
            for (int col = 0; col < BN; col += EC) {
                float v[J][EC];
#pragma unroll
                for (int jj = 0; jj < J; ++jj) {
                    if constexpr (EC == 16) tmem_ld16(tbase + jj * BN + col, v[jj]);
                    else tmem_ld8(tbase + jj * BN + col, v[jj]);
                }
                if (col + EC >= BN) {             // last TMEM read of this tile: free the accumulator early
                    tc_fence_before();
                    mbar_arrive(acce0 + 8 * ab);
                }
                const int64_t r0 = (int64_t)tc.i * b * d + (int64_t)(tc.k0 + col) * d + tc.j0;
                if (bias) {                       // KSLinear bias (NEXT-2)
#pragma unroll
                    for (int e = 0; e < EC; ++e)
#pragma unroll
                        for (int jj = 0; jj < J; ++jj) v[jj][e] += __ldg(bias + r0 + (int64_t)e * d + jj);
                }
                if (act) {
#pragma unroll
                    for (int e = 0; e < EC; ++e)
#pragma unroll
                        for (int jj = 0; jj < J; ++jj) v[jj][e] = ks_act(v[jj][e], act);
                }
                if constexpr (OUTL == KS_LAYOUT_BSL) {    // Y^T row r0 + e d + jj: lanes = 32 batch rows
                    const int64_t n = (int64_t)tc.n0 + lq * 32 + lane;
                    if (n < B && !(dbg & 1)) {
#pragma unroll
                        for (int e = 0; e < EC; ++e)
#pragma unroll
                            for (int jj = 0; jj < J; ++jj) __stcs(Y + (r0 + (int64_t)e * d + jj) * B + n, v[jj][e]);
                    }
                } else if ((dbg & 4) && (J == d || J % 4 == 0)) {   // experiment: direct stores
                    direct_store_rows<J, EC>(v, Y, (int64_t)tc.n0 + lq * 32, B, M, r0, d, lane);
                } else if constexpr (TST) {
                    // box buffer of this warp: [32 n][EC k][J j] floats, dense (SWIZZLE_NONE:
                    // a 128-byte-swizzled box with 16-byte rows faults in the TMA unit).  Lane n's
                    // row is NU 16-byte chunks at n * ROWB, ROWB a multiple of 128 bytes, so chunk u of
                    // every lane would hit the same 4 banks: lane n writes chunk (u + n) mod NU at step
                    // u (8 lanes of a phase on 8 bank groups), its chunks rotated by n mod 8 in
                    // registers first (3 conditional rotations, no dynamic register indexing).
                    // The previous chunk's store must have read the buffer.
                    constexpr int NU = EC * J / 4;
                    static_assert(NU % 8 == 0, "rows of whole 128-byte bank sweeps");
                    const uint32_t buf = scr0 + (uint32_t)(warp - 6) * C::TBOX;
                    float w[NU][4];
#pragma unroll
                    for (int u = 0; u < NU; ++u)
#pragma unroll
                        for (int x = 0; x < 4; ++x) w[u][x] = v[(u * 4 + x) % J][(u * 4 + x) / J];
                    const int rot = lane & 7;
#pragma unroll
                    for (int sb = 1; sb < 8; sb <<= 1) {
                        const bool on = rot & sb;
                        float t[NU][4];
#pragma unroll
                        for (int u = 0; u < NU; ++u)
#pragma unroll
                            for (int x = 0; x < 4; ++x) t[u][x] = on ? w[(u + sb) % NU][x] : w[u][x];
#pragma unroll
                        for (int u = 0; u < NU; ++u)
#pragma unroll
                            for (int x = 0; x < 4; ++x) w[u][x] = t[u][x];
                    }
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < NU; ++u) {
                        const uint32_t c = (uint32_t)((u + rot) % NU);
                        sts128(buf + (uint32_t)lane * (NU * 16) + c * 16, w[u][0], w[u][1], w[u][2], w[u][3]);
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0 && !(dbg & 1)) {     // Y viewed [B][a b][d]: box {J j, EC k, 32 n}
                        tma_store_3d(&ymap, tc.j0, (int)(r0 / d), tc.n0 + lq * 32, buf);
                        bulk_commit();
                    }
                } else if (!(dbg & 1)) {          // profiling experiment: skip the stores
                    warp_store_rows<float, J, EC>(scr0 + (uint32_t)(warp - 6) * WarpStore<float, J, EC>::BYTES, v, Y,
                                                  (int64_t)tc.n0 + lq * 32, B, M, r0, d, lane);
                }
            }
        }
    }
    if constexpr (TST) {
        if (warp >= 6 && lane == 0) bulk_wait_all();     // this thread's TMA stores have completed
    }
    if (prof) {       // [0,1] producer (sempty, empty) [2,3] transposer 0 (sfull, empty) [4,5] MMA (acce, full)
        const unsigned long long tot = clock64() - tk0;      // [6] epilogue warp 6 (accf); [8..11] role run times
        if (tid == 0) { pc[0] = w0; pc[1] = w1; pc[8] = tot; }
        if (tid == 32) { pc[2] = w0; pc[3] = w1; pc[9] = tot; }
        if (tid == 160) { pc[4] = w0; pc[5] = w1; pc[10] = tot; }
        if (tid == 192) { pc[6] = w0; pc[11] = tot; }
    }
    tc_fence_before();
    __syncthreads();
    if (prof && tid < 16) reinterpret_cast<unsigned long long*>(Y)[blockIdx.x * 16 + tid] = pc[tid];
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    }
}

// ==========================================================================
// Half precision, BSF with d > 1 (NEXT-3).  J j-values per tile, chosen so the
// X gather is a legal TMA box (inner extent a multiple of 16 bytes):
//   J = d  (d in {2, 3, 4, 6, 8}): the J columns of all 16 l of a block are one
//          contiguous run of 16*d halves of an X row -> 2-D box {16 d + 8, 128 n};
//   J = 8  (d % 8 == 0):       3-D box {8 j, 17 l, 128 n} of X viewed [B][a c][d].
// Either way a staged row n holds [16 l][J] halves plus 16 bytes of padding, so
// its pitch 32 J + 16 is an odd number of 16-byte units and the transposers'
// 16-byte reads of 8 consecutive rows hit 8 different bank groups.  Each
// transposer thread unpacks its row into J K-major A rows of 16 halves (32 B,
// SWIZZLE_32B); per stage the MMA warp runs one K = 16 kind::f16 step into each
// of J accumulators (2 x J x BN <= 512 TMEM columns); the epilogue stores
// through warp_store_rows (coalesced 16-byte units).
// ==========================================================================
// HK = l per stage: 16 (32-byte SWIZZLE_32B operand rows, one K = 16 MMA) or
// 32 (64-byte SWIZZLE_64B rows, two MMAs) -- 32 halves the per-stage barrier /
// transposer / TMA-issue overhead per byte and is used when c % 32 == 0 and J <= 4.

// JB = j extent of the X box: J, or 8 for J = 4 when d % 8 != 0.  A 4-half
// box row would be 8 bytes (TMA's minimum is 16) and a 3-D view needs the l
// stride d * 2 bytes to be a multiple of 16, so that case ("per-l boxes") loads
// 16 2-D boxes {8 halves, 128 n} per stage, one per l, stacked [l][n][8]
// (the transposers use the first 4 of the 8 j; the rest is the next j-group's,
// served from L2).
template <int J, int BN, int JB = J, int HK = 16>
struct HalfJCfg {
    static constexpr bool PER_L = JB != J;
    static constexpr int RB = 2 * HK;                     // operand row bytes
    static constexpr int AH_BYTES = BM * RB;              // A tile per j
    static constexpr int PITCH = PER_L ? 16 : RB * JB + 16;   // staged row: [HK l][JB] halves + 16 B
    static constexpr int STG = PER_L ? HK * BM * 16 : BM * PITCH;
    static constexpr int BJ_BYTES = BN * RB;              // per j
    static constexpr int SLOT = J * (AH_BYTES + BJ_BYTES);
    static constexpr int EC = J > 4 ? 8 : 16;             // epilogue columns per TMEM load
    static constexpr int SCR = 4 * WarpStore<__half, J, EC>::BYTES;     // epilogue store scratch
    // X staging ring sized for ~96 KB in flight (as Tf32JCfg), leaving 2 operand slots
    static constexpr int P_WANT = (96 * 1024 + STG - 1) / STG;
    static constexpr int P_ROOM = (212 * 1024 - 2 * SLOT - SCR) / STG;
    static constexpr int P_MIN = P_WANT < P_ROOM ? P_WANT : P_ROOM;
    static constexpr int P = P_MIN < 2 ? 2 : P_MIN > 8 ? 8 : P_MIN;
    static constexpr int S_FIT = (212 * 1024 - P * STG - SCR) / SLOT;
    static constexpr int S = S_FIT > 4 ? 4 : S_FIT;
    static constexpr int SCR_OFF = S * SLOT + P * STG;
    static constexpr int BAR_OFF = SCR_OFF + SCR;
    static constexpr int SMEM = BAR_OFF + 256 + 1024;
    static constexpr int TMEM_COLS = 2 * J * BN <= 256 ? 256 : 512;
    static_assert(J * BN <= 256 && BN % 16 == 0, "J accumulators, double-buffered");
    static_assert((2 * S + 4 + 2 * P) * 8 + 4 <= 256, "barrier area");
    static_assert(S >= 2, "pipeline too shallow");
    static_assert(SMEM <= 227 * 1024, "shared memory");
    static_assert(HK == 16 || (HK == 32 && !PER_L && J <= 4), "HK = 32: contiguous / gather boxes, J <= 4");
};

template <typename T, int J, int BN, int JB = J, int HK = 16>
__global__ void __launch_bounds__(NTHREADS, 1)
ks_half_bsfj_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                    T* __restrict__ Y, const T* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d,
                    int64_t ntiles) {
    using C = HalfJCfg<J, BN, JB, HK>;
    constexpr int AH_BYTES = C::AH_BYTES;
    constexpr int RB = C::RB;
    constexpr int S = C::S;
    constexpr int P = C::P;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accf0 = smem_u32(&bars[2 * S]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + 2]);
    const uint32_t sfull0 = smem_u32(&bars[2 * S + 4]);
    const uint32_t sempty0 = smem_u32(&bars[2 * S + 4 + P]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 4 + 2 * P]);
    const uint32_t slot0 = smem_u32(smem);        // S x [J A tiles (4 KB) | J B tiles (BN*32 B)]
    const uint32_t stg0 = slot0 + S * C::SLOT;    // P x staging
    const uint32_t scr0 = slot0 + C::SCR_OFF;     // epilogue store scratch

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int nkc = b / BN;
    const int njg = d / J;
    const bool contig = (J == d);                 // 2-D box over X rows, else 3-D {8 j, 17 l, n}
    const int64_t nnb = (B + BM - 1) / BM;
    const int64_t M = (int64_t)a * b * d;
    const int nk = c / HK;                        // c % HK == 0
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t G = my_tiles * nk;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1 + NTRANS);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, NEPI);
        }
        for (int p = 0; p < P; ++p) {
            mbar_init(sfull0 + 8 * p, 1);
            mbar_init(sempty0 + 8 * p, NTRANS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                 // the prologue above overlaps the previous kernel's drain (PDL)
    pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            auto issue_x = [&](int64_t gx) {
                const TileJ tc = decode_j(blockIdx.x + (gx / nk) * gridDim.x, nkc, njg, nnb, BN, J);
                const int l0 = (int)(gx % nk) * HK;
                const int p = (int)(gx % P);
                if (gx >= P) mbar_wait(sempty0 + 8 * p, (uint32_t)(((gx / P) - 1) & 1));
                mbar_expect_tx(sfull0 + 8 * p, C::STG);
                if constexpr (C::PER_L) {
#pragma unroll 1
                    for (int l = 0; l < HK; ++l)
                        tma_2d(stg0 + p * C::STG + l * (BM * 16), &xmap, ((tc.i * c + l0 + l) * d + tc.j0) & ~7,
                               tc.n0, sfull0 + 8 * p);   // 16-byte aligned start (required)
                } else if (contig) {
                    tma_2d(stg0 + p * C::STG, &xmap, (tc.i * c + l0) * d, tc.n0, sfull0 + 8 * p);
                } else {
                    tma_3d(stg0 + p * C::STG, &xmap, tc.j0, tc.i * c + l0, tc.n0, sfull0 + 8 * p);
                }
            };
            for (int64_t gx = 0; gx < P - 1 && gx < G; ++gx) issue_x(gx);
            for (int64_t g = 0; g < G; ++g) {
                if (g + P - 1 < G) issue_x(g + P - 1);
                const TileJ tc = decode_j(blockIdx.x + (g / nk) * gridDim.x, nkc, njg, nnb, BN, J);
                const int l0 = (int)(g % nk) * HK;
                const int st = (int)(g % S);
                if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                mbar_expect_tx(full0 + 8 * st, J * C::BJ_BYTES);
                const uint32_t sb = slot0 + st * C::SLOT + J * AH_BYTES;
                for (int jj = 0; jj < J; ++jj)
                    tma_2d(sb + jj * C::BJ_BYTES, &kmap, l0, ((tc.i * d + tc.j0 + jj) * b) + tc.k0, full0 + 8 * st);
            }
        }
    } else if (warp <= 4) {
        // staging row r: [16 l][J] halves -> J K-major SW32 A rows of 16 halves
        const int r = tid - 32;
        const uint32_t rowoff = (uint32_t)((r / 8) * (8 * RB) + (r % 8) * RB);
        const int sw = RB == 64 ? (r % 8) / 2 : (r % 8) / 4;     // SW64 / SW32 chunk XOR
        for (int64_t g = 0; g < G; ++g) {
            const int p = (int)(g % P);
            mbar_wait(sfull0 + 8 * p, (uint32_t)((g / P) & 1));
            uint32_t w[HK / 2 * JB];
            const uint32_t src = stg0 + p * C::STG + r * C::PITCH;
            // 16-byte unit q of the virtual row [HK l][JB]: contiguous, or (per-l boxes) l = q at l * 2 KB
            constexpr uint32_t QSTRIDE = C::PER_L ? BM * 16 : 16;
#pragma unroll
            for (int q = 0; q < HK / 8 * JB; ++q)
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w[4 * q]), "=r"(w[4 * q + 1]), "=r"(w[4 * q + 2]), "=r"(w[4 * q + 3])
                             : "r"(src + q * QSTRIDE));
            fence_proxy_async();          // generic reads before the TMA (async proxy) refill
            mbar_arrive(sempty0 + 8 * p);
            // virtual row [HK l][J] halves, as 32-bit words
            uint32_t wv[HK / 2 * J];
            if constexpr (C::PER_L) {
                // box l starts at the 16-byte-aligned column below (i c + l0 + l) d + j0; the
                // 4 wanted halves sit at offset 0 or 4 (d, j0 multiples of 4): words 0-1 or 2-3
                const TileJ tc = decode_j(blockIdx.x + (g / nk) * gridDim.x, nkc, njg, nnb, BN, J);
                const int col0 = (tc.i * c + (int)(g % nk) * HK) * d + tc.j0;
#pragma unroll
                for (int l = 0; l < HK; ++l) {
                    const bool hi4 = ((col0 + l * d) & 4) != 0;
                    wv[2 * l] = hi4 ? w[4 * l + 2] : w[4 * l];
                    wv[2 * l + 1] = hi4 ? w[4 * l + 3] : w[4 * l + 1];
                }
            } else {
#pragma unroll
                for (int q = 0; q < HK / 2 * J; ++q) wv[q] = w[q];
            }
            const int st = (int)(g % S);
            if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
            const uint32_t sa = slot0 + st * C::SLOT + rowoff;
#pragma unroll
            for (int jj = 0; jj < J; ++jj) {
                uint32_t o[HK / 2];
#pragma unroll
                for (int q = 0; q < HK / 2; ++q) {    // halves l = 2q, 2q+1 of column jj
                    const int e0 = (2 * q) * J + jj, e1 = (2 * q + 1) * J + jj;
                    const uint32_t sel = (e0 & 1 ? 0x32u : 0x10u) | ((e1 & 1 ? 0x76u : 0x54u) << 8);
                    o[q] = __byte_perm(wv[e0 >> 1], wv[e1 >> 1], sel);
                }
#pragma unroll
                for (int ch = 0; ch < HK / 8; ++ch)
                    sts128(sa + jj * AH_BYTES + ((ch ^ sw) * 16), __uint_as_float(o[4 * ch]),
                           __uint_as_float(o[4 * ch + 1]), __uint_as_float(o[4 * ch + 2]), __uint_as_float(o[4 * ch + 3]));
            }
            fence_proxy_async();
            mbar_arrive(full0 + 8 * st);
        }
    } else if (warp == 5) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_t<T>(BN);
            int64_t g = 0, it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int ab = (int)(it & 1);
                if (it >= 2) mbar_wait(acce0 + 8 * ab, (uint32_t)(((it / 2) - 1) & 1));
                tc_fence_after();
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
                    tc_fence_after();
                    const uint32_t sa = slot0 + st * C::SLOT;
                    const uint32_t sb = sa + J * AH_BYTES;
#pragma unroll
                    for (int jj = 0; jj < J; ++jj)
#pragma unroll
                        for (int s = 0; s < HK / 16; ++s) {   // K = 16 halves = 32 B per MMA
                            const uint32_t ah = sa + jj * AH_BYTES + 32 * s, bh = sb + jj * C::BJ_BYTES + 32 * s;
                            if constexpr (HK == 32)
                                mma_f16(tmem + (uint32_t)((ab * J + jj) * BN), sw64_desc(ah), sw64_desc(bh), idesc,
                                        (t > 0 || s > 0) ? 1u : 0u);
                            else
                                mma_f16(tmem + (uint32_t)((ab * J + jj) * BN), sw32_desc(ah), sw32_desc(bh), idesc,
                                        t > 0 ? 1u : 0u);
                        }
                    mma_commit(empty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
            }
        }
        __syncwarp();
    } else {
        constexpr int EC = C::EC;
        const int lq = warp & 3;
        const int row = lq * 32 + lane;
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const TileJ tc = decode_j(tile, nkc, njg, nnb, BN, J);
            const int ab = (int)(it & 1);
            mbar_wait(accf0 + 8 * ab, (uint32_t)((it / 2) & 1));
            tc_fence_after();
            const int64_t n = (int64_t)tc.n0 + row;
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * J * BN);
#pragma unroll 1
            for (int col = 0; col < BN; col += EC) {
                float v[J][EC];
#pragma unroll
                for (int jj = 0; jj < J; ++jj) {
                    if constexpr (EC == 16) tmem_ld16(tbase + jj * BN + col, v[jj]);
                    else tmem_ld8(tbase + jj * BN + col, v[jj]);
                }
                const int64_t r0 = (int64_t)tc.i * b * d + (int64_t)(tc.k0 + col) * d + tc.j0;
                if (bias) {                       // KSLinear bias (NEXT-2)
#pragma unroll
                    for (int e = 0; e < EC; ++e)
#pragma unroll
                        for (int jj = 0; jj < J; ++jj) v[jj][e] += ElemTraits<T>::to_f(bias[r0 + (int64_t)e * d + jj]);
                }
                if (act) {
#pragma unroll
                    for (int e = 0; e < EC; ++e)
#pragma unroll
                        for (int jj = 0; jj < J; ++jj) v[jj][e] = ks_act(v[jj][e], act);
                }
                if constexpr (JB != J) {
                    // J = 4 of an 8-wide box (d % 8 != 0): the 4 outputs of one k are one
                    // 8-byte run, the next k is d away -- per-row stores (units of the
                    // coalescing store would straddle runs)
                    const int64_t n = (int64_t)tc.n0 + lq * 32 + lane;
                    if (n < B) {
#pragma unroll
                        for (int e = 0; e < EC; ++e) {
                            uint32_t w[2];
#pragma unroll
                            for (int x = 0; x < 2; ++x) {
                                const T lo = ElemTraits<T>::from_f(v[2 * x][e]), hi = ElemTraits<T>::from_f(v[2 * x + 1][e]);
                                w[x] = (uint32_t)reinterpret_cast<const uint16_t&>(lo) |
                                       ((uint32_t)reinterpret_cast<const uint16_t&>(hi) << 16);
                            }
                            __stcs(reinterpret_cast<uint2*>(Y + n * M + r0 + (int64_t)e * d), make_uint2(w[0], w[1]));
                        }
                    }
                } else {
                    warp_store_rows<T, J, EC>(scr0 + (uint32_t)(warp - 6) * WarpStore<T, J, EC>::BYTES, v, Y,
                                              (int64_t)tc.n0 + lq * 32, B, M, r0, d, lane);
                }
            }
            tc_fence_before();
            mbar_arrive(acce0 + 8 * ab);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    }
}

// ------------------------------------------------------------------ host ------
// Output-tile width: the whole block when b <= 128 (two CTAs per SM fit), else
// the largest divisor <= 128 (b/BN tiles share one X tile through L2: the tile
// order runs the k-chunks of a tile back to back).
int pick_bn(int64_t b) {
    if (b <= 128 && b % 16 == 0) return (int)b;
    for (int bn : {128, 112, 96, 80, 64, 48, 32, 16})
        if (b % bn == 0) return bn;
    return 0;
}

template <int LAYOUT, int BN, typename T, bool X3, int OUTL, bool MNA, bool TSTD>
cudaError_t launch_bn_t(const ks_handle_s& h, const KsCall& call);

bool bsfj_tst_on();

// FP32 BSF-out launches take the TMA-store epilogue (TSTD); KS_TF32_TMASTORE=0 disables
template <int LAYOUT, int BN, typename T = float, bool X3 = false, int OUTL = LAYOUT, bool MNA = false>
cudaError_t launch_bn(const ks_handle_s& h, const KsCall& call) {
    if constexpr (OUTL == KS_LAYOUT_BSF && sizeof(T) == 4)
        if (bsfj_tst_on()) return launch_bn_t<LAYOUT, BN, T, X3, OUTL, MNA, true>(h, call);
    return launch_bn_t<LAYOUT, BN, T, X3, OUTL, MNA, false>(h, call);
}

template <int LAYOUT, int BN, typename T, bool X3, int OUTL, bool MNA, bool TSTD>
cudaError_t launch_bn_t(const ks_handle_s& h, const KsCall& call) {
    using C = Tf32Cfg<LAYOUT, BN, X3, OUTL, MNA>;
    constexpr cuuint32_t BK = C::RB / sizeof(T);
    constexpr cuuint64_t ES = sizeof(T);
    constexpr CUtensorMapSwizzle SW = C::RB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const CUtensorMapDataType dt = ElemTraits<T>::tma;
    CUtensorMap xmap, kmap, kmap_lo;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.c, (cuuint64_t)(h.a * h.d * h.b)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.c * ES};
        const cuuint32_t kb[2] = {BK, BN};
        if (!encode(&kmap, h.k_tf32, 2, kd, ks, kb, SW, dt)) return cudaErrorInvalidValue;
        kmap_lo = kmap;
        if (X3 && !encode(&kmap_lo, h.k_lo, 2, kd, ks, kb, SW, dt)) return cudaErrorInvalidValue;
    }
    if (LAYOUT == KS_LAYOUT_BSL) {
        const cuuint64_t xd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c)};
        const cuuint64_t xs[2] = {(cuuint64_t)call.B * ES, (cuuint64_t)(h.d * call.B) * ES};
        if constexpr (MNA) {
            const cuuint32_t xb[3] = {32, 1, 32};
            if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, dt)) return cudaErrorInvalidValue;
        } else {
            const cuuint32_t xb[3] = {BM, 1, BK};
            if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE, dt)) return cudaErrorInvalidValue;
        }
    } else {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * ES};
        const cuuint32_t xb[2] = {BK, BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, SW, dt)) return cudaErrorInvalidValue;
    }
    CUtensorMap ymap{};
    if constexpr (TSTD) {                        // Y viewed [B][M] (d = 1): box {16 outputs, 32 rows}
        const int64_t M = h.a * h.b * h.d;
        const cuuint64_t yd[2] = {(cuuint64_t)M, (cuuint64_t)call.B};
        const cuuint64_t ys[1] = {(cuuint64_t)M * 4};
        const cuuint32_t yb[2] = {16, 32};
        if (!encode(&ymap, call.Y, 2, yd, ys, yb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    auto kern = ks_tf32_kernel<LAYOUT, BN, T, X3, OUTL, MNA, TSTD>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * ((call.B + BM - 1) / BM) * (h.a * h.d);
    int64_t slots = (int64_t)ks::num_sms(h.device) * C::CTAS;
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(NTHREADS), C::SMEM, call.stream, xmap, kmap,
                                         kmap_lo, ymap, reinterpret_cast<T*>(call.Y), reinterpret_cast<const T*>(call.bias),
                                         call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d, ntiles, debug_flags() | (call.act << 8));
    ks::count_launch();
    return e;
}

// ---- TF32 BSF, d > 1 (ks_tf32_bsfj_kernel): plan = (J, BN, gather) ----------
// J = d for d <= 8 (contiguous 2-D box), else J = 8 (b <= 64) or 4 (3-D gather,
// d % J == 0).  BN = the largest tile width dividing b with J x BN <= 512 TMEM
// columns: modelled L2->SM reads per X byte = (b / BN) x (J = 4 gather ? 2 : 1),
// so a whole-block BN (single-buffered accumulators) beats a split BN.
struct BsfjPlan {
    int J = 0, BN = 0;
    bool gather = false;
};
// J = 8 (32-byte gather runs) also for b > 64: TMA boxes with 16-byte inner runs
// (J = 4) read X at <= 3-4 TB/s, 32-byte runs at 4.6-5.1 TB/s
// (scripts/probe_tma_gather.cu); BN then halves (J x BN <= 512 TMEM columns) and the
// b / BN output chunks of one X tile run on adjacent CTAs at the same time (L2 hits).
// 3xTF32 doubles every operand tile: J <= 4 there (d = 6 runs FFMA).
// bsl_out (mixed BSF-in / BSL-out calls): Y's rows are 512-byte runs whatever J is,
// so the J8 knob's 32-byte runs buy nothing there while halving BN doubles the X
// re-reads: (1,256,64,16) BSF -> BSL J = 4 320 us, J = 8 424 us (profiles/r03/tst2_j8.jsonl).
BsfjPlan pick_bsfj(const ks_handle_s& h, uint32_t knobs, bool bsl_out = false) {
    BsfjPlan p;
    if (bsl_out) knobs &= ~(uint32_t)KS_KNOB_J8;
    const bool x3 = h.math == KS_MATH_F32X3;
    if (h.c % 16 != 0) return p;
    if (h.d >= 2 && h.d <= (x3 ? 4 : 8) && h.d != 5 && h.d != 7) {
        p.J = (int)h.d;
    } else if (!x3 && h.d > 8 && h.d % 8 == 0 && (h.b <= 64 || (knobs & KS_KNOB_J8))) {
        p.J = 8;
        p.gather = true;
    } else if (h.d > (x3 ? 4 : 8) && h.d % 4 == 0) {
        p.J = 4;
        p.gather = true;
    } else {
        return p;
    }
    // BN = 256 (UMMA N maximum) only for wide blocks with J = 2 (b = 768 in ViT-S UP):
    // it halves the L2 re-reads of X across output chunks (knob KS_KNOB_BN256)
    if ((knobs & KS_KNOB_BN256) && !x3 && p.J == 2 && h.b > 128 && h.b % 256 == 0) {
        p.BN = 256;
        return p;
    }
    for (int bn : {128, 96, 64, 48, 32, 16})
        if (h.b % bn == 0 && p.J * bn <= 512) {
            p.BN = bn;
            break;
        }
    if (p.BN == 0) p.J = 0;
    return p;
}

// BSL in / BSF out, d > 1 (mixed-layout calls): every j's X rows are 512-byte
// runs whatever J is, so J only sets the output run length (J = d: whole
// contiguous row segments); BN as in pick_bsfj.
BsfjPlan pick_bslj(const ks_handle_s& h, uint32_t knobs) {
    BsfjPlan p;
    if (h.c % 16 != 0 || h.d < 2) return p;
    if (h.d <= 8 && h.d != 5 && h.d != 7) p.J = (int)h.d;
    else if (h.d % 8 == 0) p.J = 8;
    else if (h.d % 4 == 0) p.J = 4;
    else return p;
    if ((knobs & KS_KNOB_BN256) && p.J == 2 && h.b > 128 && h.b % 256 == 0) {
        p.BN = 256;
        return p;
    }
    for (int bn : {128, 96, 64, 48, 32, 16})
        if (h.b % bn == 0 && p.J * bn <= 512) {
            p.BN = bn;
            break;
        }
    if (p.BN == 0) p.J = 0;
    return p;
}

// l per stage: 16 (SWIZZLE_64B rows, half the padding / barrier traffic per
// byte) when 2 operand slots and >= 64 KB of X staging fit, else 8 (SWIZZLE_32B).
template <int J, int BN, bool X3, bool GATHER, int INL = KS_LAYOUT_BSF, int OUTL = KS_LAYOUT_BSF>
constexpr int bsfj_bkj() {
    constexpr int NA = X3 ? 2 : 1;
    constexpr int slot16 = J * NA * (BM + BN) * 64;
    constexpr int stg16 = BM * (INL == KS_LAYOUT_BSL ? 16 * J * 4 : GATHER ? 17 * J * 4 : 16 * J * 4 + 16);
    constexpr int scr = OUTL == KS_LAYOUT_BSL ? 0 : 4 * WarpStore<float, J, (J > 2 ? 8 : 16)>::BYTES;
    constexpr int p16 = stg16 >= 32 * 1024 ? 2 : (64 * 1024 + stg16 - 1) / stg16;
    return 214 * 1024 - p16 * stg16 - scr >= 2 * slot16 ? 16 : 8;
}

// TMA-store epilogue (TST) for J = 8 (32-byte runs of Y, d % 8 == 0; Y viewed
// [B][a b][d]): measured over the configs[2] sweep, J = 8 tiles 1.05-1.20x faster
// with it, J = 4 tiles (16-byte runs) 0.68-0.94x -- there the 16-byte warp stores
// of warp_store_rows stay (profiles/r03/tst_time.jsonl).  KS_TF32_TMASTORE=0
// disables (experiments).
bool bsfj_tst_on() {
    static const bool on = [] {
        const char* e = getenv("KS_TF32_TMASTORE");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

template <int J, int BN, bool X3, bool GATHER, int INL, int OUTL, bool TST, bool MNJ = false>
cudaError_t launch_bsfj_t(const ks_handle_s& h, const KsCall& call);

template <int J, int BN, bool X3, bool GATHER, int INL = KS_LAYOUT_BSF, int OUTL = KS_LAYOUT_BSF>
cudaError_t launch_bsfj(const ks_handle_s& h, const KsCall& call) {
    if constexpr (OUTL == KS_LAYOUT_BSF && J == 8)
        if (bsfj_tst_on()) return launch_bsfj_t<J, BN, X3, GATHER, INL, OUTL, true>(h, call);
    return launch_bsfj_t<J, BN, X3, GATHER, INL, OUTL, false>(h, call);
}

template <int J, int BN, bool X3, bool GATHER, int INL, int OUTL, bool TST, bool MNJ>
cudaError_t launch_bsfj_t(const ks_handle_s& h, const KsCall& call) {
    constexpr int BKJ = MNJ ? 32 : bsfj_bkj<J, BN, X3, GATHER, INL, OUTL>();
    using C = Tf32JCfg<J, BN, BKJ, X3, GATHER, INL, OUTL, TST, MNJ>;
    constexpr CUtensorMapSwizzle SW = C::RB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                    : C::RB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUtensorMap xmap, kmap, kmap_lo;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.c, (cuuint64_t)(h.a * h.d * h.b)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.c * 4};
        const cuuint32_t kb[2] = {(cuuint32_t)BKJ, BN};
        if (!encode(&kmap, h.k_tf32, 2, kd, ks, kb, SW)) return cudaErrorInvalidValue;
        kmap_lo = kmap;
        if (X3 && !encode(&kmap_lo, h.k_lo, 2, kd, ks, kb, SW)) return cudaErrorInvalidValue;
    }
    if (INL == KS_LAYOUT_BSL) {
        const cuuint64_t xd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c)};
        const cuuint64_t xs[2] = {(cuuint64_t)call.B * 4, (cuuint64_t)(h.d * call.B) * 4};
        if constexpr (MNJ) {               // {32 n, 1 j, 32 l} boxes, MN-major operand atoms
            const cuuint32_t xb[3] = {32, 1, 32};
            if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return cudaErrorInvalidValue;
        } else {
            const cuuint32_t xb[3] = {BM, (cuuint32_t)J, (cuuint32_t)BKJ};
            if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
        }
    } else if (GATHER) {
        const cuuint64_t xd[3] = {(cuuint64_t)h.d, (cuuint64_t)(h.a * h.c), (cuuint64_t)call.B};
        const cuuint64_t xs[2] = {(cuuint64_t)h.d * 4, (cuuint64_t)h.N * 4};
        const cuuint32_t xb[3] = {(cuuint32_t)J, (cuuint32_t)BKJ + 1, BM};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {(cuuint32_t)(BKJ * J + 4), BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    CUtensorMap ymap{};
    if constexpr (TST) {
        const int64_t M = h.a * h.b * h.d;           // Y viewed [B][a b][d] (d % 8 == 0)
        const cuuint64_t yd[3] = {(cuuint64_t)h.d, (cuuint64_t)(h.a * h.b), (cuuint64_t)call.B};
        const cuuint64_t ys[2] = {(cuuint64_t)h.d * 4, (cuuint64_t)M * 4};
        const cuuint32_t yb[3] = {(cuuint32_t)J, (cuuint32_t)C::EC, 32};
        if (!encode(&ymap, call.Y, 3, yd, ys, yb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    auto kern = ks_tf32_bsfj_kernel<J, BN, BKJ, X3, GATHER, INL, OUTL, TST, MNJ>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * (h.d / J) * ((call.B + BM - 1) / BM) * h.a;
    int64_t slots = (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(NTHREADS), C::SMEM, call.stream, xmap, kmap,
                                         kmap_lo, ymap, call.Y, call.bias, call.B, (int)h.a, (int)h.b, (int)h.c,
                                         (int)h.d, ntiles, debug_flags() | (call.act << 8));
    ks::count_launch();
    return e;
}

template <int J, bool X3, bool GATHER, int INL = KS_LAYOUT_BSF, int OUTL = KS_LAYOUT_BSF>
cudaError_t launch_bsfj_bn(const ks_handle_s& h, const KsCall& call, int BN) {
    switch (BN) {
        case 256: if constexpr (J == 2 && !X3 && !GATHER) return launch_bsfj<J, 256, X3, GATHER, INL, OUTL>(h, call); break;
        case 128: if constexpr (J * 128 <= 512) return launch_bsfj<J, 128, X3, GATHER, INL, OUTL>(h, call); break;
        case 96: if constexpr (J * 96 <= 512) return launch_bsfj<J, 96, X3, GATHER, INL, OUTL>(h, call); break;
        case 64: return launch_bsfj<J, 64, X3, GATHER, INL, OUTL>(h, call);
        case 48: return launch_bsfj<J, 48, X3, GATHER, INL, OUTL>(h, call);
        case 32: return launch_bsfj<J, 32, X3, GATHER, INL, OUTL>(h, call);
        case 16: return launch_bsfj<J, 16, X3, GATHER, INL, OUTL>(h, call);
    }
    return cudaErrorInvalidValue;
}

// INL / OUTL: BSF / BSF (X3 or TF32), BSF / BSL or BSL / BSF (TF32 mixed-layout calls)
// MN-major A for BSL in / BSF out (MNJ): J = 4 (four j's 16 KB A tiles + BN <= 64 weight
// rows fit two 32-l operand slots), d % 4 == 0 and d <= 16: measured (1,64,256,16)
// 349 -> 273 us, (1,128,128,16) 166 -> 100 us, (1,96,96,8) 69 -> 46 us; at d = 32 the
// 16-byte output runs of J = 4 cost more than the staged J = 8 kernel's TMA-stored
// 32-byte runs ((1,128,128,32) 296 -> 423 us), profiles/r03/mnj_time.jsonl.
// KS_TF32_MNJ=0 disables (experiments).
bool bsfj_mnj_on() {
    static const bool on = [] {
        const char* e = getenv("KS_TF32_MNJ");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

template <bool X3, int INL = KS_LAYOUT_BSF, int OUTL = KS_LAYOUT_BSF>
cudaError_t launch_bsfj_any(const ks_handle_s& h, const KsCall& call) {
    if constexpr (INL == KS_LAYOUT_BSL && OUTL == KS_LAYOUT_BSF && !X3) {
        if (bsfj_mnj_on() && h.d % 4 == 0 && h.d <= 16 && h.c % 32 == 0) {
            for (int bn : {64, 48, 32, 16}) {
                if (h.b % bn != 0) continue;
                switch (bn) {
                    case 64: return launch_bsfj_t<4, 64, false, false, INL, OUTL, false, true>(h, call);
                    case 48: return launch_bsfj_t<4, 48, false, false, INL, OUTL, false, true>(h, call);
                    case 32: return launch_bsfj_t<4, 32, false, false, INL, OUTL, false, true>(h, call);
                    case 16: return launch_bsfj_t<4, 16, false, false, INL, OUTL, false, true>(h, call);
                }
            }
        }
    }
    const BsfjPlan p = INL == KS_LAYOUT_BSL ? pick_bslj(h, call.knobs)
                                            : pick_bsfj(h, call.knobs, OUTL == KS_LAYOUT_BSL);
    if constexpr (INL == KS_LAYOUT_BSF) {
        if (p.gather) {
            if (p.J == 4) return launch_bsfj_bn<4, X3, true, INL, OUTL>(h, call, p.BN);
            if constexpr (!X3)
                if (p.J == 8) return launch_bsfj_bn<8, X3, true, INL, OUTL>(h, call, p.BN);
            return cudaErrorInvalidValue;
        }
    }
    switch (p.J) {
        case 2: return launch_bsfj_bn<2, X3, false, INL, OUTL>(h, call, p.BN);
        case 3: return launch_bsfj_bn<3, X3, false, INL, OUTL>(h, call, p.BN);
        case 4: return launch_bsfj_bn<4, X3, false, INL, OUTL>(h, call, p.BN);
    }
    if constexpr (!X3) {
        if (p.J == 6) return launch_bsfj_bn<6, X3, false, INL, OUTL>(h, call, p.BN);
        if (p.J == 8) return launch_bsfj_bn<8, X3, false, INL, OUTL>(h, call, p.BN);
    }
    return cudaErrorInvalidValue;
}

bool bsfj_ok(const ks_handle_s& h, uint32_t knobs) { return pick_bsfj(h, knobs).J != 0; }


// Half BSF, d > 1: J j-values per tile (see ks_half_bsfj_kernel), 0 = unsupported.
// d % 4 == 0 but not 8 (d = 12, 20, ...): J = 4 from an 8-wide box.
int pick_j_half(int64_t d) {
    if (d == 2 || d == 3 || d == 4 || d == 6 || d == 8) return (int)d;
    if (d % 8 == 0) return 8;
    return d % 4 == 0 ? 4 : 0;
}
int pick_bn_half(int64_t b, int J) {
    for (int bn : {128, 96, 64, 48, 32, 16})
        if (b % bn == 0 && J * bn <= 256) return bn;
    return 0;
}

template <typename T, int J, int BN, int JB = J, int HK = 16>
cudaError_t launch_halfj(const ks_handle_s& h, const KsCall& call) {
    using C = HalfJCfg<J, BN, JB, HK>;
    constexpr CUtensorMapSwizzle SWH = HK == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    const CUtensorMapDataType dt = ElemTraits<T>::tma;
    CUtensorMap xmap, kmap;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.c, (cuuint64_t)(h.a * h.d * h.b)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.c * 2};
        const cuuint32_t kb[2] = {HK, BN};
        if (!encode(&kmap, h.k_tf32, 2, kd, ks, kb, SWH, dt)) return cudaErrorInvalidValue;
    }
    if (C::PER_L) {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 2};
        const cuuint32_t xb[2] = {(cuuint32_t)JB, BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE, dt)) return cudaErrorInvalidValue;
    } else if (J == h.d) {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 2};
        const cuuint32_t xb[2] = {(cuuint32_t)(HK * J + 8), BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE, dt)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[3] = {(cuuint64_t)h.d, (cuuint64_t)(h.a * h.c), (cuuint64_t)call.B};
        const cuuint64_t xs[2] = {(cuuint64_t)h.d * 2, (cuuint64_t)h.N * 2};
        const cuuint32_t xb[3] = {(cuuint32_t)JB, HK + 1, BM};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE, dt)) return cudaErrorInvalidValue;
    }
    auto kern = ks_half_bsfj_kernel<T, J, BN, JB, HK>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * (h.d / J) * ((call.B + BM - 1) / BM) * h.a;
    int64_t slots = (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(NTHREADS), C::SMEM, call.stream, xmap, kmap,
                                         reinterpret_cast<T*>(call.Y), reinterpret_cast<const T*>(call.bias), call.act, call.B,
                                         (int)h.a, (int)h.b, (int)h.c, (int)h.d, ntiles);
    ks::count_launch();
    return e;
}

template <typename T, int J, int JB, int HK>
cudaError_t launch_halfj_bn_hk(const ks_handle_s& h, const KsCall& call) {
    switch (pick_bn_half(h.b, J)) {
        case 128: if constexpr (J * 128 <= 256) return launch_halfj<T, J, 128, JB, HK>(h, call); break;
        case 96: if constexpr (J * 96 <= 256) return launch_halfj<T, J, 96, JB, HK>(h, call); break;
        case 64: if constexpr (J * 64 <= 256) return launch_halfj<T, J, 64, JB, HK>(h, call); break;
        case 48: if constexpr (J * 48 <= 256) return launch_halfj<T, J, 48, JB, HK>(h, call); break;
        case 32: if constexpr (J * 32 <= 256) return launch_halfj<T, J, 32, JB, HK>(h, call); break;
        case 16: return launch_halfj<T, J, 16, JB, HK>(h, call);
    }
    return cudaErrorInvalidValue;
}

// 32 l per stage when c allows it and the staging row stays small (J <= 4, no per-l boxes)
template <typename T, int J, int JB = J>
cudaError_t launch_halfj_bn(const ks_handle_s& h, const KsCall& call) {
    if constexpr (J <= 4 && JB == J) {
        if (h.c % 32 == 0) return launch_halfj_bn_hk<T, J, JB, 32>(h, call);
    }
    return launch_halfj_bn_hk<T, J, JB, 16>(h, call);
}

template <typename T>
cudaError_t launch_halfj_any(const ks_handle_s& h, const KsCall& call) {
    switch (pick_j_half(h.d)) {
        case 2: return launch_halfj_bn<T, 2>(h, call);
        case 3: return launch_halfj_bn<T, 3>(h, call);
        case 4: return h.d == 4 ? launch_halfj_bn<T, 4>(h, call) : launch_halfj_bn<T, 4, 8>(h, call);
        case 6: return launch_halfj_bn<T, 6>(h, call);
        case 8: return launch_halfj_bn<T, 8>(h, call);
    }
    return cudaErrorInvalidValue;
}

template <int LAYOUT, typename T = float, bool X3 = false, int OUTL = LAYOUT, bool MNA = false>
cudaError_t launch_layout(const ks_handle_s& h, const KsCall& call) {
    switch (pick_bn(h.b)) {
        case 128: return launch_bn<LAYOUT, 128, T, X3, OUTL, MNA>(h, call);
        case 112: return launch_bn<LAYOUT, 112, T, X3, OUTL, MNA>(h, call);
        case 96: return launch_bn<LAYOUT, 96, T, X3, OUTL, MNA>(h, call);
        case 80: return launch_bn<LAYOUT, 80, T, X3, OUTL, MNA>(h, call);
        case 64: return launch_bn<LAYOUT, 64, T, X3, OUTL, MNA>(h, call);
        case 48: return launch_bn<LAYOUT, 48, T, X3, OUTL, MNA>(h, call);
        case 32: return launch_bn<LAYOUT, 32, T, X3, OUTL, MNA>(h, call);
        case 16: return launch_bn<LAYOUT, 16, T, X3, OUTL, MNA>(h, call);
    }
    return cudaErrorInvalidValue;
}

// ---- TF32 BSF, 2 <= d <= 8: the densified super-block path --------------------
// Def. 1: supp(K) lies in I_a (x) 1_{bd x cd}, so super-block i
// is also a dense (bd x cd) block whose entries outside 1_{b x c} (x) I_d are zero.
// Contracted that way the factor is an (a, bd, cd, 1) pattern: X's super-block
// columns [i cd, (i+1) cd) are one contiguous K-major TMA box and Y's rows
// [i bd, (i+1) bd) one contiguous output run, so the d = 1 kernel runs it with no
// gather, no transposer warps and full-line stores -- at d times the MMA work
// (the zeros), which the tensor cores absorb while d * bc / (2 (b + c)) stays
// near the TF32:HBM ridge (~112 flop/B on B200: 732 TF/s cuBLAS / 6.55 TB/s).
// Chosen by the knob KS_KNOB_DENSIFY (preset table / rules, ks_presets.cpp);
// patterns the J-gather cannot run (d = 5, 7) are densified whenever the blocks
// exist, unless KS_TF32_DENSIFY=0 (experiments).
bool dense_ok(const ks_handle_s& h, const KsCall& call) {
    if (!h.k_dense || call.layout != KS_LAYOUT_BSF || h.math != KS_MATH_TF32 || h.d < 2) return false;
    if (call.mixed() && !(call.knobs & KS_KNOB_DENSIFY)) return false;   // BSL out: the J kernel's stores are whole lines
    if (pick_bn(h.b * h.d) == 0 || h.N % 4 != 0 || h.M % 4 != 0) return false;
    if (call.knobs & KS_KNOB_DENSIFY) return true;
    static const bool never = [] {
        const char* e = getenv("KS_TF32_DENSIFY");
        return e && atoi(e) == 0;
    }();
    return !never && !bsfj_ok(h, call.knobs);
}

cudaError_t launch_dense(const ks_handle_s& h, const KsCall& call) {
    ks_handle_s hd = h;
    hd.b = h.b * h.d;
    hd.c = h.c * h.d;
    hd.d = 1;
    hd.k_tf32 = h.k_dense;
    if (call.mixed()) return launch_layout<KS_LAYOUT_BSF, float, false, KS_LAYOUT_BSL>(hd, call);
    return launch_layout<KS_LAYOUT_BSF>(hd, call);
}

}  // namespace

namespace ks {

bool tf32_supports(const ks_handle_s& h, const KsCall& call) {
    if (tf32v2_supports(h, call)) return true;
    if (h.b < 16 || h.c < 16 || h.c % 8 != 0 || pick_bn(h.b) == 0) return false;
    if (h.a * h.d * h.b >= (int64_t(1) << 31) || h.a * h.c >= (int64_t(1) << 31)) return false;
    if (call.B >= (int64_t(1) << 31)) return false;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(call.X), ya = reinterpret_cast<uintptr_t>(call.Y);
    if (xa & 15) return false;                                   // TMA global address
    if (call.mixed()) {            // TF32 only: BSF in / BSL out, or BSL in / BSF out
        if (h.math != KS_MATH_TF32) return false;
        if (call.layout == KS_LAYOUT_BSF)
            return (ya & 3) == 0 && (h.d == 1 || bsfj_ok(h, call.knobs) || dense_ok(h, call));
        if (call.B % 4 != 0 || (ya & 15)) return false;
        return h.d == 1 || pick_bslj(h, call.knobs).J != 0;
    }
    if (call.layout == KS_LAYOUT_BSL) return call.B % 4 == 0 && (ya & 3) == 0;
    if (ya & 15) return false;
    // BSF: d = 1 direct; d > 1 J-column gather (pick_bsfj; bias read as scalars)
    if (h.math == KS_MATH_F32X3 && !h.k_lo) return false;
    return h.d == 1 || bsfj_ok(h, call.knobs) || dense_ok(h, call);
}

cudaError_t tf32_launch(const ks_handle_s& h, const KsCall& call) {
    if (h.math == KS_MATH_F32X3) {
        if (!h.k_lo) return cudaErrorInvalidValue;
        if (call.layout == KS_LAYOUT_BSL) return launch_layout<KS_LAYOUT_BSL, float, true>(h, call);
        if (h.d == 1) return launch_layout<KS_LAYOUT_BSF, float, true>(h, call);
        return launch_bsfj_any<true>(h, call);
    }
    if (call.mixed()) {
        if (call.layout == KS_LAYOUT_BSL) {
            if (h.d == 1 && (call.knobs & KS_KNOB_TF32_MN))
                return launch_layout<KS_LAYOUT_BSL, float, false, KS_LAYOUT_BSF, true>(h, call);
            if (h.d == 1) return launch_layout<KS_LAYOUT_BSL, float, false, KS_LAYOUT_BSF>(h, call);
            return launch_bsfj_any<false, KS_LAYOUT_BSL, KS_LAYOUT_BSF>(h, call);
        }
        if (dense_ok(h, call)) return launch_dense(h, call);
        if (h.d == 1) return launch_layout<KS_LAYOUT_BSF, float, false, KS_LAYOUT_BSL>(h, call);
        return launch_bsfj_any<false, KS_LAYOUT_BSF, KS_LAYOUT_BSL>(h, call);
    }
    if (tf32v2_supports(h, call)) return tf32v2_launch(h, call);
    if (dense_ok(h, call)) return launch_dense(h, call);
    if (call.layout == KS_LAYOUT_BSL && (call.knobs & KS_KNOB_TF32_MN))
        return launch_layout<KS_LAYOUT_BSL, float, false, KS_LAYOUT_BSL, true>(h, call);
    if (call.layout == KS_LAYOUT_BSL) return launch_layout<KS_LAYOUT_BSL>(h, call);
    if (h.d == 1) return launch_layout<KS_LAYOUT_BSF>(h, call);
    return launch_bsfj_any<false>(h, call);
}

// ---- half precision (NEXT-3): the same warp-specialised tcgen05 kernel with
// kind::f16 (BF16 or FP16 operands, FP32 accumulation, output rounded to
// nearest-even).  BSL any d; BSF d = 1.
bool half_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (h.b < 16 || h.c < 16 || h.c % 16 != 0 || pick_bn(h.b) == 0) return false;
    if (h.a * h.d * h.b >= (int64_t(1) << 31) || h.a * h.c >= (int64_t(1) << 31)) return false;
    if (call.B >= (int64_t(1) << 31)) return false;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(call.X), ya = reinterpret_cast<uintptr_t>(call.Y);
    if (call.layout == KS_LAYOUT_BSL) return half_bsl_supports(h, call);
    if (xa & 15) return false;
    if (ya & 15) return false;
    if (h.d == 1) return true;
    // BSF d > 1: J-column gather (bias read as scalars, any 2-byte alignment)
    const int J = pick_j_half(h.d);
    return J != 0 && pick_bn_half(h.b, J) != 0 && (J != h.d || (h.N * 2) % 16 == 0);
}

cudaError_t half_launch(const ks_handle_s& h, const KsCall& call) {
    const bool bf = h.dtype == KS_DTYPE_BF16;
    if (call.layout == KS_LAYOUT_BSL) return half_bsl_launch(h, call);
    if (h.d == 1)
        return bf ? launch_layout<KS_LAYOUT_BSF, __nv_bfloat16>(h, call) : launch_layout<KS_LAYOUT_BSF, __half>(h, call);
    return bf ? launch_halfj_any<__nv_bfloat16>(h, call) : launch_halfj_any<__half>(h, call);
}

}  // namespace ks
