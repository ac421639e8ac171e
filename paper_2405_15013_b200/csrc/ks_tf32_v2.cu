// TF32 tensor-core KS kernel, round 2 ("v2"): BSL (any d) and BSF with d = 1.
//
// Same contraction as ks_tf32.cu (output-stationary tile
// Y[n0:n0+128, row_{i,j}[k0:k0+BN]], Alg. 3, each element
// written once; UMMA D[m][n] = sum_k A[m][k] B[n][k], M = 128 batch rows,
// N = BN outputs, K = l), re-planned around three measured bottlenecks of the
// round-1 kernel (VERDICT r1 "What's weak" #3):
//   * no transposer warps: in BSL, X[col_ij][n0:n0+128] is MN-major (n
//     contiguous), and kind::tf32 accepts an MN-major A operand in the
//     "SW128_32B" canonical layout (UMMA layout type 1, SWIZZLE_128B_BASE32B:
//     32-byte chunks XOR-swizzled in 128-byte rows with a 4-row period) that
//     TMA writes directly (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).  Measured on
//     B200 by scripts/probe_umma_mn.cu (exact): LBO = 4096 B between 32-n
//     groups, SBO = 512 B between 4-l groups.  BSF d = 1 loads A K-major (SW128);
//   * resident weights: each persistent CTA owns a contiguous range of tiles
//     ordered (i, j) -> n-block -> k-chunk, so the packed K^T tile (BN x c,
//     K-major SW128, <= 112 KB) is loaded once per (i, j, k-chunk) segment and
//     reused by every n-block of the range (round 1 re-read it from L2 for
//     every tile: as many L2->SM bytes as X itself); one K buffer, or two
//     (double-buffered across segments) when they fit beside a 6-deep X ring;
//   * TMA-store epilogue: each epilogue warp stages its 32 rows x CW outputs in
//     shared memory (swizzled: conflict-free 16-byte writes) and one lane
//     issues cp.async.bulk.tensor shared->global, double-buffered with
//     bulk_group waits -- full-line writes that leave the warps' critical path
//     (round 1's per-thread stores amplified L1->L2 write bytes 1.9-2.4x).
// One CTA (256 threads) per SM:
//   warp 0 lane 0: X TMA producer (S-deep ring of 16 KB stages, 32 l each)
//   warp 1 lane 0: weight TMA producer (one segment ahead when NKB = 2)
//   warp 2:        TMEM allocator + single-thread MMA issuer (accumulators
//                  double-buffered: 2 x BN TMEM columns)
//   warp 3:        idle
//   warps 4-7:     epilogue (TMEM lane quarter = warp % 4)
// X is fed as raw FP32 bits (the tensor core reads the TF32 part: truncation,
// DESIGN.md R10); K is pre-rounded RNA at pack time; FP32 accumulation.
#include "ks_umma.cuh"

namespace {

constexpr int V2_THREADS = 256;
constexpr int V2_BM = 128;
constexpr int V2_STAGE = V2_BM * 128;            // 16 KB: 128 rows x 32 l x 4 B
constexpr int V2_SMEM_MAX = 227 * 1024;
constexpr int V2_KT_MAX = 112 * 1024;            // largest resident weight tile


struct V2Tile {
    int i, j, k0, n0;
    int64_t q;        // weight segment id: (i*d + j)*nkc + kc
};

// tile t -> (k-chunk fastest, then n-block, then (i, j)): consecutive tiles of
// a CTA share the weight segment when nkc == 1, and the X tile (L2) otherwise
__device__ __forceinline__ V2Tile v2_decode(int64_t t, int nkc, int64_t nnb, int d, int BN) {
    V2Tile r;
    const int kc = (int)(t % nkc);
    const int64_t rest = t / nkc;
    r.n0 = (int)(rest % nnb) * V2_BM;
    const int64_t ij = rest / nnb;
    r.i = (int)(ij / d);
    r.j = (int)(ij % d);
    r.k0 = kc * BN;
    r.q = ij * nkc + kc;
    return r;
}

template <int LAYOUT, int BN>
__global__ void __launch_bounds__(V2_THREADS, 1)
ks_tf32v2_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap ymap, const float* __restrict__ bias, int64_t B, int a, int b,
                 int c, int d, int64_t ntiles, int S, int NKB, uint32_t KT, int order_act, float* __restrict__ Yd) {
    const int order = order_act & 0xFF, act = (order_act >> 8) & 0xFF;   // bits 8-15: epilogue activation
    constexpr int CW = BN % 32 == 0 ? 32 : 16;          // output columns per store box
    constexpr uint32_t EBOX = 32 * CW * 4;               // one warp's staged box
    constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    constexpr bool BSL = LAYOUT == KS_LAYOUT_BSL;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t ring0 = smem_u32(smem);
    const uint32_t kbuf0 = ring0 + (uint32_t)S * V2_STAGE;
    const uint32_t epi0 = kbuf0 + (uint32_t)NKB * KT;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * V2_STAGE + (size_t)NKB * KT + 8 * EBOX);
    const uint32_t afull0 = smem_u32(&bars[0]);
    const uint32_t aempty0 = smem_u32(&bars[S]);
    const uint32_t kfull0 = smem_u32(&bars[2 * S]);
    const uint32_t kempty0 = smem_u32(&bars[2 * S + 2]);
    const uint32_t accf0 = smem_u32(&bars[2 * S + 4]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + 6]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 8]);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int nkc = b / BN;
    const int64_t nnb = (B + V2_BM - 1) / V2_BM;
    const int nk = (c + 31) / 32;
    // this CTA's tiles: a balanced contiguous range (order 0), or round-robin
    // t = blockIdx.x + k * gridDim.x (order 1: concurrent CTAs on adjacent tiles)
    const int ord = order & 1;
    const int64_t cnt = ord ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x
                              : (int64_t)(blockIdx.x + 1) * ntiles / gridDim.x - (int64_t)blockIdx.x * ntiles / gridDim.x;
    const int64_t tb = ord ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * ntiles / gridDim.x;
    const int64_t ts = ord ? (int64_t)gridDim.x : 1;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(afull0 + 8 * s, 1);
            mbar_init(aempty0 + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(kfull0 + 8 * s, 1);
            mbar_init(kempty0 + 8 * s, 1);
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&ymap) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
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
            // ---------------- X producer ----------------
            int64_t g = 0;
            for (int64_t k = 0; k < cnt; ++k) {
                const V2Tile tc = v2_decode(tb + k * ts, nkc, nnb, d, BN);
                for (int kk = 0; kk < nk; ++kk, ++g) {
                    const int st = (int)(g % S);
                    if (g >= S) mbar_wait(aempty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                    const uint32_t dst = ring0 + (uint32_t)st * V2_STAGE;
                    mbar_expect_tx(afull0 + 8 * st, V2_STAGE);
                    if constexpr (BSL) {
                        if (order & 4) {             // canonical atoms: [l-group][n-group][4 l][32 n], one 5-D box
                            asm volatile(
                                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                                ::"r"(dst), "l"(&xmap), "r"(0), "r"(0), "r"(tc.n0 / 32), "r"(tc.j),
                                  "r"((tc.i * c + 32 * kk) / 4), "r"(afull0 + 8 * st) : "memory");
                        } else {
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4)
                                tma_3d(dst + q4 * 4096, &xmap, tc.n0 + 32 * q4, tc.j, tc.i * c + 32 * kk,
                                       afull0 + 8 * st);
                        }
                    } else {
                        tma_2d(dst, &xmap, tc.i * c + 32 * kk, tc.n0, afull0 + 8 * st);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- weight producer: one load per segment ----------------
            int64_t u = 0, prev = -1;
            for (int64_t k = 0; k < cnt; ++k) {
                const V2Tile tc = v2_decode(tb + k * ts, nkc, nnb, d, BN);
                if (tc.q == prev) continue;
                prev = tc.q;
                const int kb = (int)(u % NKB);
                if (u >= NKB) mbar_wait(kempty0 + 8 * kb, (uint32_t)(((u / NKB) - 1) & 1));
                const uint32_t dst = kbuf0 + (uint32_t)kb * KT;
                mbar_expect_tx(kfull0 + 8 * kb, (uint32_t)nk * BN * 128);
                const int row0 = (int)((tc.i * (int64_t)d + tc.j) * b) + tc.k0;
                for (int kk = 0; kk < nk; ++kk) tma_2d(dst + kk * (BN * 128), &kmap, 32 * kk, row0, kfull0 + 8 * kb);
                ++u;
            }
        }
    } else if (warp == 2) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            uint32_t idesc = make_idesc(BN);
            if (BSL) idesc |= 1u << 15;                  // A MN-major
            int64_t g = 0, it = 0, u = -1, prev = -1;
            int kb = 0;
            for (int64_t k = 0; k < cnt; ++k, ++it) {
                const V2Tile tc = v2_decode(tb + k * ts, nkc, nnb, d, BN);
                if (tc.q != prev) {
                    prev = tc.q;
                    ++u;
                    kb = (int)(u % NKB);
                    mbar_wait(kfull0 + 8 * kb, (uint32_t)((u / NKB) & 1));
                }
                const int ab = (int)(it & 1);
                if (it >= 2) mbar_wait(acce0 + 8 * ab, (uint32_t)(((it / 2) - 1) & 1));
                tc_fence_after();
                const uint32_t dtm = tmem + (uint32_t)(ab * BN);
                const uint32_t kbase = kbuf0 + (uint32_t)kb * KT;
                for (int kk = 0; kk < nk; ++kk, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait(afull0 + 8 * st, (uint32_t)((g / S) & 1));
                    tc_fence_after();
                    const uint32_t sa = ring0 + (uint32_t)st * V2_STAGE;
                    const uint32_t sb = kbase + (uint32_t)kk * (BN * 128);
                    const int ksteps = min(4, (c - 32 * kk) / 8);
                    for (int s = 0; s < ksteps; ++s) {
                        const uint64_t ad = !BSL ? sw128_desc(sa + 32 * s)
                                            : (order & 4) ? mn_sw128_32b_desc(sa + 4096 * s, 512, 2048)
                                                          : mn_sw128_32b_desc(sa + 1024 * s, 4096, 512);
                        mma_tf32(dtm, ad, sw128_desc(sb + 32 * s), idesc, (kk > 0 || s > 0) ? 1u : 0u);
                    }
                    mma_commit(aempty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
                // last tile of this weight segment: release the buffer once these MMAs complete
                if (k + 1 == cnt || v2_decode(tb + (k + 1) * ts, nkc, nnb, d, BN).q != tc.q) mma_commit(kempty0 + 8 * kb);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> swizzled smem box -> TMA store ----------------
        const int wq = warp & 3;                         // TMEM lane quarter
        const uint32_t ebuf0 = epi0 + (uint32_t)wq * 2 * EBOX;
        const int64_t M = (int64_t)a * b * d;
        int64_t it = 0, ec = 0;
        for (int64_t k = 0; k < cnt; ++k, ++it) {
            const V2Tile tc = v2_decode(tb + k * ts, nkc, nnb, d, BN);
            const int ab = (int)(it & 1);
            mbar_wait(accf0 + 8 * ab, (uint32_t)((it / 2) & 1));
            tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ab * BN);
#pragma unroll 1
            for (int col = 0; col < BN; col += CW, ++ec) {
                float v[CW];
                tmem_ld16(tbase + col, v);
                if constexpr (CW == 32) tmem_ld16(tbase + col + 16, v + 16);
                if (col + CW >= BN) {                    // last TMEM read of the tile: free the accumulator
                    tc_fence_before();
                    mbar_arrive(acce0 + 8 * ab);
                }
                if (bias) {                              // KSLinear bias (NEXT-2), per output row r
#pragma unroll
                    for (int e = 0; e < CW; ++e) {
                        const int64_t kg = (int64_t)tc.i * b + tc.k0 + col + e;
                        v[e] += __ldg(bias + (BSL ? kg * d + tc.j : kg));
                    }
                }
                if (act) {                               // epilogue activation (NEXT-2)
#pragma unroll
                    for (int e = 0; e < CW; ++e) v[e] = ks_act(v[e], act);
                }
                if (BSL && (order & 2)) {                // experiment: direct coalesced stores (no TMA store)
                    const int64_t n = (int64_t)tc.n0 + wq * 32 + lane;
                    if (n < B) {
#pragma unroll
                        for (int e = 0; e < CW; ++e)
                            __stcs(Yd + (((int64_t)tc.i * b + tc.k0 + col + e) * d + tc.j) * B + n, v[e]);
                    }
                    continue;
                }
                const uint32_t buf = ebuf0 + (uint32_t)(ec & 1) * EBOX;
                if (lane == 0) bulk_wait_read1();        // the store issued from this buffer 2 boxes ago has read it
                __syncwarp();
                if constexpr (BSL) {
                    // box [CW k][32 n]: row k is 32 consecutive batch columns (lane = n)
#pragma unroll
                    for (int e = 0; e < CW; ++e) sts32(buf + e * 128 + lane * 4, v[e]);
                } else {
                    // box [32 n][CW k], SW128 (CW = 32) / SW64 (CW = 16): 16-byte chunk ch of row
                    // `lane` at (ch ^ x), x = lane % 8 (SW128) or (lane % 8) / 2 (SW64)
                    const int x = CW == 32 ? (lane & 7) : ((lane & 7) >> 1);
#pragma unroll
                    for (int ch = 0; ch < CW / 4; ++ch)
                        sts128(buf + lane * (CW * 4) + ((ch ^ x) * 16), v[4 * ch], v[4 * ch + 1], v[4 * ch + 2],
                               v[4 * ch + 3]);
                }
                fence_proxy_async();                     // generic writes -> async-proxy (TMA) reads
                __syncwarp();
                if (lane == 0) {
                    if constexpr (BSL)
                        tma_store_3d(&ymap, tc.n0 + 32 * wq, tc.j, tc.i * b + tc.k0 + col, buf);
                    else
                        tma_store_2d(&ymap, tc.i * b + tc.k0 + col, tc.n0 + 32 * wq, buf);
                    bulk_commit();
                }
            }
        }
        (void)M;
        if (lane == 0) bulk_wait_all();                  // Y complete before the grid retires (PDL consumers)
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}

// ------------------------------------------------------------------ host ------
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

struct V2Plan {
    int BN = 0, S = 0, NKB = 0;
    uint32_t KT = 0;
    int smem = 0;
};

int v2_epi_bytes(int BN) { return 8 * 32 * (BN % 32 == 0 ? 32 : 16) * 4; }

V2Plan v2_plan(const ks_handle_s& h, int64_t B, int sms, uint32_t knobs) {
    V2Plan p;
    const int64_t nk = (h.c + 31) / 32;
    for (int bn = 256; bn >= 16; bn -= 16)
        if (h.b % bn == 0 && nk * bn * 128 <= V2_KT_MAX) {
            p.BN = bn;
            break;
        }
    if (p.BN == 0) return p;
    // fill the machine: when the tile count is under 1.5 waves, halve the tile width
    const int64_t nnb = (B + V2_BM - 1) / V2_BM;
    static const int fill = env_int("KS_V2_FILL", 1);
    while (fill && p.BN % 32 == 0 && p.BN >= 64 && (h.b / p.BN) * nnb * h.a * h.d * 2 < (int64_t)sms * 3) p.BN /= 2;
    p.KT = (uint32_t)(nk * p.BN * 128);
    const int fixed = v2_epi_bytes(p.BN) + 256 + 1024;
    const int room2 = V2_SMEM_MAX - fixed - 2 * (int)p.KT;
    p.NKB = room2 >= ((knobs & KS_KNOB_V2_NKB2) ? 2 : 6) * V2_STAGE ? 2 : 1;
    const int room = V2_SMEM_MAX - fixed - p.NKB * (int)p.KT;
    p.S = room / V2_STAGE;
    static const int smax = env_int("KS_V2_SMAX", 8);
    if (p.S > smax) p.S = smax;
    if (p.S < 2) {
        p.BN = 0;
        return p;
    }
    p.smem = fixed + p.NKB * (int)p.KT + p.S * V2_STAGE;
    return p;
}

bool encode5(CUtensorMap* m, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
             const cuuint32_t* box) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bit 0: round-robin tiles (else contiguous ranges); bit 1: BSL direct stores (else
// TMA store); bit 2: BSL canonical SW128_32B atoms by one 5-D box (else 4 boxes).
// Default: contiguous ranges, TMA store, canonical atoms (1.35x faster than 4 boxes
// on (1,128,128,64) BSL, profiles/r02/exp_tf32_v2_j8.txt); KS_V2_ORDER overrides.
int v2_order(int64_t B) {
    static const int v = env_int("KS_V2_ORDER", -1);
    if (v >= 0) return v;
    return B % 32 == 0 ? 4 : 0;
}

template <int LAYOUT, int BN>
cudaError_t v2_launch_bn(const ks_handle_s& h, const KsCall& call, const V2Plan& p) {
    constexpr int CW = BN % 32 == 0 ? 32 : 16;
    CUtensorMap xmap, kmap, ymap;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.c, (cuuint64_t)(h.a * h.d * h.b)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.c * 4};
        const cuuint32_t kb[2] = {32, (cuuint32_t)BN};
        if (!encode(&kmap, h.k_tf32, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    }
    if (LAYOUT == KS_LAYOUT_BSL) {
        const cuuint64_t xd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c)};
        const cuuint64_t xs[2] = {(cuuint64_t)call.B * 4, (cuuint64_t)(h.d * call.B) * 4};
        const cuuint32_t xb[3] = {32, 1, 32};
        if (v2_order(call.B) & 4) {
            // 5-D view {32 n, 4 l, B/32 n-groups, d, a c / 4 l-groups}: one box per stage lands the
            // canonical SW128_32B atoms [l-group][n-group][4 l][32 n] (needs B % 32 == 0)
            const cuuint64_t xd5[5] = {32, 4, (cuuint64_t)call.B / 32, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c / 4)};
            const cuuint64_t xs5[4] = {(cuuint64_t)(h.d * call.B) * 4, 128, (cuuint64_t)call.B * 4,
                                       (cuuint64_t)(4 * h.d * call.B) * 4};
            const cuuint32_t xb5[5] = {32, 4, 4, 1, 8};
            if (!encode5(&xmap, call.X, xd5, xs5, xb5)) return cudaErrorInvalidValue;
        } else if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
            return cudaErrorInvalidValue;
        const cuuint64_t yd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.b)};
        const cuuint32_t yb[3] = {32, 1, (cuuint32_t)CW};
        if (!encode(&ymap, call.Y, 3, yd, xs, yb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t xd[2] = {(cuuint64_t)h.N, (cuuint64_t)call.B};
        const cuuint64_t xs[1] = {(cuuint64_t)h.N * 4};
        const cuuint32_t xb[2] = {32, V2_BM};
        if (!encode(&xmap, call.X, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
        const cuuint64_t yd[2] = {(cuuint64_t)h.M, (cuuint64_t)call.B};
        const cuuint64_t ys[1] = {(cuuint64_t)h.M * 4};
        const cuuint32_t yb[2] = {(cuuint32_t)CW, 32};
        if (!encode(&ymap, call.Y, 2, yd, ys, yb, CW == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
            return cudaErrorInvalidValue;
    }
    auto kern = ks_tf32v2_kernel<LAYOUT, BN>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, V2_SMEM_MAX);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * ((call.B + V2_BM - 1) / V2_BM) * (h.a * h.d);
    int64_t slots = (int64_t)ks::num_sms(h.device);
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e =
        ks::launch_pdl(kern, dim3((unsigned)grid), dim3(V2_THREADS), (size_t)p.smem, call.stream, xmap, kmap, ymap,
                       call.bias, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d, ntiles, p.S, p.NKB, p.KT,
                       v2_order(call.B) | (call.act << 8), call.Y);
    ks::count_launch();
    return e;
}

template <int LAYOUT>
cudaError_t v2_launch_layout(const ks_handle_s& h, const KsCall& call, const V2Plan& p) {
    switch (p.BN) {
#define KS_V2_CASE(n) \
    case n: return v2_launch_bn<LAYOUT, n>(h, call, p);
        KS_V2_CASE(16) KS_V2_CASE(32) KS_V2_CASE(48) KS_V2_CASE(64) KS_V2_CASE(80) KS_V2_CASE(96) KS_V2_CASE(112)
        KS_V2_CASE(128) KS_V2_CASE(144) KS_V2_CASE(160) KS_V2_CASE(176) KS_V2_CASE(192) KS_V2_CASE(208)
        KS_V2_CASE(224) KS_V2_CASE(240) KS_V2_CASE(256)
#undef KS_V2_CASE
    }
    return cudaErrorInvalidValue;
}


}  // namespace

namespace ks {

// TF32 (not 3xTF32), FP32 handle, BSL any d or BSF d = 1, 16-byte aligned
// X/Y with 16-byte row pitches (TMA), and a plan that fits shared memory.
bool tf32v2_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (!(call.knobs & KS_KNOB_TF32_V2) || h.dtype != KS_DTYPE_F32 || h.math != KS_MATH_TF32) return false;
    if (h.b < 16 || h.c < 16 || h.c % 8 != 0 || h.b % 16 != 0) return false;
    if (h.a * h.d * h.b >= (int64_t(1) << 31) || h.a * h.c >= (int64_t(1) << 31) || call.B >= (int64_t(1) << 31))
        return false;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(call.X), ya = reinterpret_cast<uintptr_t>(call.Y);
    if ((xa & 15) || (ya & 15)) return false;
    if (call.layout == KS_LAYOUT_BSL) {
        if (call.B % 4 != 0) return false;
    } else {
        if (h.d != 1 || h.N % 4 != 0 || h.M % 4 != 0) return false;
    }
    return v2_plan(h, call.B, 148, call.knobs).BN != 0;
}

cudaError_t tf32v2_launch(const ks_handle_s& h, const KsCall& call) {
    const V2Plan p = v2_plan(h, call.B, ks::num_sms(h.device), call.knobs);
    if (p.BN == 0) return cudaErrorInvalidValue;
    if (call.layout == KS_LAYOUT_BSL) return v2_launch_layout<KS_LAYOUT_BSL>(h, call, p);
    return v2_launch_layout<KS_LAYOUT_BSF>(h, call, p);
}

}  // namespace ks
