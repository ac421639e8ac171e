// Half-precision (BF16 / FP16, tcgen05.mma.kind::f16, FP32 accumulation) KS
// kernel for the BSL layout, NEXT-3 (the paper's FP16 study,
// PAPER.md:1597-1618, ran CUDA-core half2 only).
//
// "Swap-AB" form of the output-stationary tile (Alg. 3):
// in BSL, X is [N][B] and Y is [M][B] (batch last), so for one KS block (i, j)
//     Y[row_ij[k0:k0+BN], n0:n0+NT] = K[row_ij[k0:..], col_ij] . X[col_ij, n0:n0+NT]
// is a GEMM whose B operand X[col_ij, n-range] is already MN-major in memory
// (n contiguous).  kind::f16 takes MN-major operands directly, so:
//   * A = K tile  [BN rows k][64 l]: TMA 2-D box from the packed k_tile rows
//     (K-major, SWIZZLE_128B); UMMA M = 128 (rows >= BN are never stored);
//   * B = X tile  [64 l][NT n]: TMA 3-D boxes {64 n, 1 j, 64 l} of X viewed as
//     [a c][d][B] (MN-major, SWIZZLE_128B, one 8 KB box per 64 n);
//   * D in TMEM: lane = output row k, column = batch n, double-buffered.
// No transposer warps and no permutation pass: the strided
// column gather col_ij is the 3-D TMA box.  The epilogue thread owning row k
// stores 16 consecutive n of output row r = i b d + k d + j as 32 contiguous
// bytes, so every store writes whole sectors.
// Warps: 0 = TMA producer, 1 = TMEM allocator + MMA issuer, 2-5 = epilogue.
#include "ks_umma.cuh"

namespace {

constexpr int HB_THREADS = 192;
constexpr int HB_BK = 64;                      // l per stage (one 128-byte row of halves)
constexpr int HB_A_BYTES = 128 * HB_BK * 2;    // 16 KB (room for UMMA M = 128 rows)
constexpr int HB_NEPI = 128;

template <int NT>
struct HalfBslCfg {
    static constexpr int B_BYTES = NT * HB_BK * 2;       // NT/64 boxes of 8 KB
    static constexpr int SLOT = HB_A_BYTES + B_BYTES;
    static constexpr int CTAS = NT <= 128 ? 2 : 1;
    static constexpr int BUDGET = CTAS == 2 ? 110 * 1024 : 210 * 1024;
    static constexpr int S_FIT = BUDGET / SLOT;
    static constexpr int S = S_FIT > 6 ? 6 : S_FIT;
    static constexpr int BAR_OFF = S * SLOT;
    static constexpr int SMEM = BAR_OFF + 256 + 1024;
    static constexpr int TMEM_COLS = 2 * NT <= 256 ? 256 : 512;
    static_assert(NT % 64 == 0 && NT <= 256 && S >= 2, "tile");
};

// MN-major, 128-byte-swizzled operand: atoms of 64 MN elements x 8 K rows (1 KB);
// LBO = stride between 64-element MN blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t mn_sw128_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

struct HbTile {
    int i, j, q, k0;
    int64_t n0;
};

__device__ __forceinline__ HbTile hb_decode(int64_t tile, int nkc, int64_t nnb, int d, int BN, int NT) {
    HbTile t;
    t.k0 = (int)(tile % nkc) * BN;          // k-chunks of one (q, n-block) back to back: X tile reused via L2
    tile /= nkc;
    t.n0 = (tile % nnb) * NT;
    t.q = (int)(tile / nnb);
    t.i = t.q / d;
    t.j = t.q % d;
    return t;
}

template <typename T, int NT, bool ACT = false>
__global__ void __launch_bounds__(HB_THREADS, HalfBslCfg<NT>::CTAS)
ks_half_bsl_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                   T* __restrict__ Y, const T* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d, int BN,
                   int64_t ntiles) {
    using C = HalfBslCfg<NT>;
    constexpr int S = C::S;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    // [0,S) full  [S,2S) empty  [2S,2S+2) acc_full  [2S+2,2S+4) acc_empty, then the TMEM slot
    const uint32_t full0 = smem_u32(&bars[0]);
    const uint32_t empty0 = smem_u32(&bars[S]);
    const uint32_t accf0 = smem_u32(&bars[2 * S]);
    const uint32_t acce0 = smem_u32(&bars[2 * S + 2]);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 4]);
    const uint32_t slot0 = smem_u32(smem);        // S x (A 16 KB | B NT*128 B), 1 KB aligned

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int nkc = b / BN;
    const int64_t nnb = (B + NT - 1) / NT;
    const int nk = (c + HB_BK - 1) / HB_BK;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(accf0 + 8 * s, 1);
            mbar_init(acce0 + 8 * s, HB_NEPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    }
    if (warp == 1) {
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
            const uint32_t tx = (uint32_t)BN * HB_BK * 2 + C::B_BYTES;
            int64_t g = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const HbTile tc = hb_decode(tile, nkc, nnb, d, BN, NT);
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    if (g >= S) mbar_wait(empty0 + 8 * st, (uint32_t)(((g / S) - 1) & 1));
                    const uint32_t sa = slot0 + st * C::SLOT;
                    mbar_expect_tx(full0 + 8 * st, tx);
                    tma_2d(sa, &kmap, t * HB_BK, tc.q * b + tc.k0, full0 + 8 * st);
#pragma unroll
                    for (int h = 0; h < NT / 64; ++h)
                        tma_3d(sa + HB_A_BYTES + h * 8192, &xmap, (int)tc.n0 + 64 * h, tc.j, tc.i * c + t * HB_BK,
                               full0 + 8 * st);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_t<T>(NT) | (1u << 16);    // B (X) MN-major
            int64_t g = 0, it = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int ab = (int)(it & 1);
                if (it >= 2) mbar_wait(acce0 + 8 * ab, (uint32_t)(((it / 2) - 1) & 1));
                tc_fence_after();
                const uint32_t dtm = tmem + (uint32_t)(ab * NT);
                for (int t = 0; t < nk; ++t, ++g) {
                    const int st = (int)(g % S);
                    mbar_wait(full0 + 8 * st, (uint32_t)((g / S) & 1));
                    tc_fence_after();
                    const uint32_t sa = slot0 + st * C::SLOT;
                    const uint32_t sb = sa + HB_A_BYTES;
                    const int ksteps = min(HB_BK / 16, (c - t * HB_BK) / 16);
                    for (int s = 0; s < ksteps; ++s)
                        mma_f16(dtm, sw128_desc(sa + 32 * s), mn_sw128_desc(sb + 2048 * s, 8192, 1024), idesc,
                                (t > 0 || s > 0) ? 1u : 0u);
                    mma_commit(empty0 + 8 * st);
                }
                mma_commit(accf0 + 8 * ab);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: TMEM lane quarter lq = rows k in [32 lq, 32 lq + 32) ----------------
        const int lq = warp & 3;
        const int k = lq * 32 + lane;
        const bool active = lq * 32 < BN;           // warp-uniform
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const HbTile tc = hb_decode(tile, nkc, nnb, d, BN, NT);
            const int ab = (int)(it & 1);
            mbar_wait(accf0 + 8 * ab, (uint32_t)((it / 2) & 1));
            tc_fence_after();
            if (active) {
                const int64_t r = (int64_t)tc.i * b * d + (int64_t)(tc.k0 + k) * d + tc.j;
                const float bv = (bias && k < BN) ? ElemTraits<T>::to_f(bias[r]) : 0.f;   // NEXT-2
                const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * NT);
#pragma unroll 1
                for (int col = 0; col < NT; col += 16) {
                    float v[16];
                    tmem_ld16(tbase + col, v);
                    const int64_t n = tc.n0 + col;
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float y0 = v[2 * e] + bv, y1 = v[2 * e + 1] + bv;
                        if constexpr (ACT) {                 // epilogue activation (compile-time switch)
                            y0 = ks_act(y0, act);
                            y1 = ks_act(y1, act);
                        }
                        const T lo = ElemTraits<T>::from_f(y0), hi = ElemTraits<T>::from_f(y1);
                        pk[e] = (uint32_t)reinterpret_cast<const uint16_t&>(lo) |
                                ((uint32_t)reinterpret_cast<const uint16_t&>(hi) << 16);
                    }
                    // Lane pair (k even, k+1) writes whole 32-byte sectors: store 1 puts
                    // the even row's two 16-byte halves, store 2 the odd row's (each lane
                    // hands its partner the half it does not store itself).
                    const bool odd = lane & 1;
                    uint32_t x[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[e] = __shfl_xor_sync(0xffffffffu, odd ? pk[e] : pk[4 + e], 1);
                    const int64_t re = odd ? r - d : r, ro = odd ? r : r + d;     // rows of k even / k odd
                    const int64_t h = odd ? 8 : 0;                                 // this lane's half
                    if (k < BN && n + h < B) {                                     // BN even, B % 8 == 0
                        __stcs(reinterpret_cast<uint4*>(Y + re * B + n + h),
                               odd ? make_uint4(x[0], x[1], x[2], x[3]) : make_uint4(pk[0], pk[1], pk[2], pk[3]));
                        __stcs(reinterpret_cast<uint4*>(Y + ro * B + n + h),
                               odd ? make_uint4(pk[4], pk[5], pk[6], pk[7]) : make_uint4(x[0], x[1], x[2], x[3]));
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acce0 + 8 * ab);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    }
}

// Rows per tile: the whole block when b <= 128, else the largest multiple-of-16
// divisor <= 128 (the k-chunks of one X tile run back to back, sharing it via L2).
int hb_pick_bn(int64_t b) {
    if (b <= 128 && b % 16 == 0) return (int)b;
    for (int bn : {128, 112, 96, 80, 64, 48, 32, 16})
        if (b % bn == 0) return bn;
    return 0;
}

template <typename T, int NT, bool ACT = false>
cudaError_t launch_hb(const ks_handle_s& h, const KsCall& call) {
    using C = HalfBslCfg<NT>;
    const CUtensorMapDataType dt = ElemTraits<T>::tma;
    const int BN = hb_pick_bn(h.b);
    CUtensorMap xmap, kmap;
    {
        const cuuint64_t kd[2] = {(cuuint64_t)h.c, (cuuint64_t)(h.a * h.d * h.b)};
        const cuuint64_t ks[1] = {(cuuint64_t)h.c * 2};
        const cuuint32_t kb[2] = {HB_BK, (cuuint32_t)BN};
        if (!encode(&kmap, h.k_tf32, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_128B, dt)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t xd[3] = {(cuuint64_t)call.B, (cuuint64_t)h.d, (cuuint64_t)(h.a * h.c)};
        const cuuint64_t xs[2] = {(cuuint64_t)call.B * 2, (cuuint64_t)(h.d * call.B) * 2};
        const cuuint32_t xb[3] = {64, 1, HB_BK};
        if (!encode(&xmap, call.X, 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B, dt)) return cudaErrorInvalidValue;
    }
    auto kern = ks_half_bsl_kernel<T, NT, ACT>;
    static bool attr[64] = {false};
    if (!attr[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr[h.device & 63] = true;
    }
    const int64_t ntiles = (h.b / BN) * ((call.B + NT - 1) / NT) * (h.a * h.d);
    int64_t slots = (int64_t)ks::num_sms(h.device) * C::CTAS;
    if (max_grid() > 0) slots = max_grid();
    const int64_t grid = ntiles < slots ? ntiles : slots;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)grid), dim3(HB_THREADS), C::SMEM, call.stream, xmap,
                                         kmap, reinterpret_cast<T*>(call.Y), reinterpret_cast<const T*>(call.bias),
                                         call.act, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d, BN, ntiles);
    ks::count_launch();
    return e;
}

}  // namespace

namespace ks {

bool half_bsl_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (h.b < 16 || h.c < 16 || h.c % 16 != 0 || hb_pick_bn(h.b) == 0) return false;
    if (h.a * h.d * h.b >= (int64_t(1) << 31) || h.a * h.c >= (int64_t(1) << 31)) return false;
    if (call.B >= (int64_t(1) << 31) || call.B % 8 != 0) return false;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(call.X), ya = reinterpret_cast<uintptr_t>(call.Y);
    return (xa & 15) == 0 && (ya & 15) == 0;
}

cudaError_t half_bsl_launch(const ks_handle_s& h, const KsCall& call) {
    static const int nt = [] {
        const char* e = getenv("KS_HB_NT");          // experiments only: batch columns per tile
        return e ? atoi(e) : 128;
    }();
    const bool bf = h.dtype == KS_DTYPE_BF16;
    if (call.act) {
        if (nt == 256) return bf ? launch_hb<__nv_bfloat16, 256, true>(h, call) : launch_hb<__half, 256, true>(h, call);
        return bf ? launch_hb<__nv_bfloat16, 128, true>(h, call) : launch_hb<__half, 128, true>(h, call);
    }
    if (nt == 256) return bf ? launch_hb<__nv_bfloat16, 256>(h, call) : launch_hb<__half, 256>(h, call);
    return bf ? launch_hb<__nv_bfloat16, 128>(h, call) : launch_hb<__half, 128>(h, call);
}

}  // namespace ks
