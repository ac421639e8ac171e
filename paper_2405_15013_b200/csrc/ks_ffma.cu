// Register-tiled FP32 (CUDA-core FFMA) KS kernel for the GEMM-like patterns
// (b a multiple of 8 -- widest tiles for 24 / 32 multiples -- c a multiple of 8): the paper's sweep
// (b = c in {48..128}), ViT-S/16 and GPT-2 KSLinear factors.
//
// Alg. 3, re-tiled for sm_100a: each CTA owns the output
// tile Y[n0:n0+BMJ, row_{i,j}[k0:k0+BN]] for J consecutive j of one
// super-block i (output-stationary, written exactly once, no atomics,
// PAPER.md:1172-1184).  It streams the reduction over col_{i,j} in BK = 8
// chunks: X[:, col_{i,j}] is gathered straight from the caller's layout
// (no permutation pass) into shared memory as A[l][j][n],
// the pre-packed K^T tile (k_tile) into B[l][j][k];
// register double-buffering overlaps the next chunk's global loads with the
// current chunk's FFMA.
//
//  * Warp tile 64 (batch rows) x 4*TN (outputs), thread micro-tile 8 x TN,
//    the 8 rows split 4 + 4 at stride 32 so A-fragment LDS.128 are
//    conflict-free; B fragments are warp broadcasts (4 distinct addresses).
//  * BSF, d > 1: J in {2, 4} consecutive j are gathered together so each X
//    load is a J-wide vector (d-strided sectors are shared, SURVEY §7 hard
//    part 1); the epilogue goes through shared memory and writes J-wide runs
//    ("structured epilogue").
//  * BSL: rows of X / Y are contiguous along the batch: float4 loads/stores
//    straight to/from registers.
// Reduction order: l ascending, one FP32 FMA chain per output -- the same
// arithmetic as the generic and streaming kernels (bit-identical results).
#include "ks_internal.h"

#include <cstdlib>

#ifndef KS_FFMA_MINB
#define KS_FFMA_MINB 2      // CTAs per SM the register allocation targets (experiments: -DKS_FFMA_MINB=1)
#endif

namespace {

constexpr int TM = 8;

template <int J> struct VecJ;
template <> struct VecJ<1> { using T = float; };
template <> struct VecJ<2> { using T = float2; };
template <> struct VecJ<4> { using T = float4; };

template <int LAYOUT, int J, int WPJM, int WPJN, int TN, int KBK>
struct Cfg {
    static constexpr int BK = KBK;                   // l per pipeline chunk
    static constexpr int WARPS = J * WPJM * WPJN;
    static constexpr int THREADS = WARPS * 32;
    static constexpr int BMJ = 64 * WPJM;            // batch rows per j
    static constexpr int BN = 4 * TN * WPJN;         // outputs (k) per j
    static constexpr int LDA = J * BMJ;              // A row (one l): [j][n]
    static constexpr int LDB = J * BN;               // B row (one l): [j][k]
    static constexpr int A_ELEMS = BK * LDA;
    static constexpr int B_ELEMS = BK * LDB;
    // per-thread global loads per BK chunk
    static constexpr int A_VECS = (LAYOUT == KS_LAYOUT_BSL) ? (BK * BMJ / 4) : (BK * BMJ);
    static constexpr int A_PER_T = (A_VECS + THREADS - 1) / THREADS;
    static constexpr int B_VECS = B_ELEMS / 4;
    static constexpr int B_PER_T = (B_VECS + THREADS - 1) / THREADS;
    static constexpr bool SMEM_EPI = (LAYOUT == KS_LAYOUT_BSF);   // used only when d > 1
    static constexpr int BNP = BN + 4;                // epilogue plane pitch
    static constexpr int C_ELEMS = BMJ * BNP * J;
    static constexpr int PIPE_ELEMS = 2 * (A_ELEMS + B_ELEMS);
    static constexpr int SMEM_ELEMS = (SMEM_EPI && C_ELEMS > PIPE_ELEMS) ? C_ELEMS : PIPE_ELEMS;
    static constexpr int SMEM_BYTES = SMEM_ELEMS * 4;
    static_assert(LAYOUT == KS_LAYOUT_BSF || J == 1, "BSL uses J = 1");
    static_assert(WARPS <= 8, "at most 8 warps");
};

// SC (scalar): X loads and Y stores element by element with predicated tails, for
// BSL batches with B % 4 != 0 and for X / Y views that are only 4-byte aligned
// (the vector path needs 16 bytes); the arithmetic (l ascending, one FMA chain per
// output) is the same, so the results are bit-identical to the vector path.
template <int LAYOUT, int J, int WPJM, int WPJN, int TN, int KBK, bool SC = false>
__global__ void __launch_bounds__(Cfg<LAYOUT, J, WPJM, WPJN, TN, KBK>::THREADS, KS_FFMA_MINB)
ks_ffma_kernel(const float* __restrict__ X, const float* __restrict__ Kt, float* __restrict__ Y,
               const float* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d) {
    static_assert(!SC || J == 1, "scalar path: one j per CTA");
    using C = Cfg<LAYOUT, J, WPJM, WPJN, TN, KBK>;
    constexpr int BK = C::BK;
    using VT = typename VecJ<J>::T;
    pdl_wait();
    pdl_launch_dependents();
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                         // [2][BK][J][BMJ]
    float* Bs = smem + 2 * C::A_ELEMS;        // [2][BK][J][BN]

    const int tid = threadIdx.x;
    const int nkc = b / C::BN;
    const int64_t nnb = (B + C::BMJ - 1) / C::BMJ;
    int64_t bid = blockIdx.x;
    const int kc = (int)(bid % nkc);
    bid /= nkc;
    const int64_t nb = bid % nnb;
    const int64_t g = bid / nnb;
    const int dj = d / J;
    const int i = (int)(g / dj);
    const int j0 = (int)(g % dj) * J;
    const int k0 = kc * C::BN;
    const int64_t n0 = nb * C::BMJ;
    const int64_t N = (int64_t)a * c * d, M = (int64_t)a * b * d;
    const int nk = c / BK;

    // ---- warp / thread coordinates --------------------------------------
    const int warp = tid >> 5, lane = tid & 31;
    const int wj = warp / (WPJM * WPJN);
    const int wr = warp % (WPJM * WPJN);
    const int wm = wr / WPJN, wn = wr % WPJN;
    const int ty = lane >> 2, tx = lane & 3;
    const int rowA = wm * 64 + ty * 4;        // rows rowA..+3 and rowA+32..+35
    const int colB = wn * 4 * TN + tx * TN;   // cols colB..colB+TN-1

    // ---- global -> register staging ---------------------------------------
    float4 ra[C::A_PER_T * (LAYOUT == KS_LAYOUT_BSL ? 1 : 0) + 1];
    VT rv[(LAYOUT == KS_LAYOUT_BSF) ? C::A_PER_T : 1];
    float4 rb[C::B_PER_T];

    const float* kt_base = Kt + ((int64_t)i * d + j0) * c * b + k0;   // + jj*c*b + l*b + k

    // Batch rows past B (last tile) load a clamped, valid row instead of a
    // conditional zero: their outputs are never stored, and an unconditional
    // load needs no select after it -- measured: the zero/select form made the
    // compiler wait for the prefetch at the top of the FFMA loop (36% of the
    // BSF kernel's stall samples on one MOV).
    auto load_tile = [&](int t) {
        const int l0 = t * BK;
        if (LAYOUT == KS_LAYOUT_BSL) {
#pragma unroll
            for (int r = 0; r < C::A_PER_T; ++r) {
                const int idx = tid + r * C::THREADS;
                if (idx < C::A_VECS) {
                    const int l = idx / (C::BMJ / 4);
                    const int n4 = idx % (C::BMJ / 4);
                    const int64_t s = (int64_t)i * c * d + (int64_t)(l0 + l) * d + j0;
                    if constexpr (SC) {               // any B, 4-byte alignment: clamped scalar loads
                        const int64_t n = n0 + 4 * n4;
                        const float* xs = X + s * B;
                        ra[r] = make_float4(__ldg(xs + min(n, B - 1)), __ldg(xs + min(n + 1, B - 1)),
                                            __ldg(xs + min(n + 2, B - 1)), __ldg(xs + min(n + 3, B - 1)));
                    } else {
                        const int64_t n = min(n0 + 4 * n4, B - 4);          // B % 4 == 0
                        ra[r] = __ldg(reinterpret_cast<const float4*>(X + s * B + n));
                    }
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < C::A_PER_T; ++r) {
                const int idx = tid + r * C::THREADS;
                if (idx < C::A_VECS) {
                    const int n = idx % C::BMJ;
                    const int l = idx / C::BMJ;
                    const int64_t nn = min(n0 + n, B - 1);
                    const float* p = X + nn * N + (int64_t)i * c * d + (int64_t)(l0 + l) * d + j0;
                    rv[r] = __ldg(reinterpret_cast<const VT*>(p));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < C::B_PER_T; ++r) {
            const int idx = tid + r * C::THREADS;
            if (idx < C::B_VECS) {
                const int l = idx / (C::LDB / 4);
                const int rem = idx % (C::LDB / 4);
                const int jj = rem / (C::BN / 4);
                const int k4 = rem % (C::BN / 4);
                rb[r] = __ldg(reinterpret_cast<const float4*>(
                    kt_base + (int64_t)jj * c * b + (int64_t)(l0 + l) * b + 4 * k4));
            }
        }
    };

    auto store_tile = [&](int buf) {
        float* as = As + buf * C::A_ELEMS;
        float* bs = Bs + buf * C::B_ELEMS;
        if (LAYOUT == KS_LAYOUT_BSL) {
#pragma unroll
            for (int r = 0; r < C::A_PER_T; ++r) {
                const int idx = tid + r * C::THREADS;
                if (idx < C::A_VECS) {
                    const int l = idx / (C::BMJ / 4);
                    const int n4 = idx % (C::BMJ / 4);
                    *reinterpret_cast<float4*>(as + l * C::LDA + 4 * n4) = ra[r];
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < C::A_PER_T; ++r) {
                const int idx = tid + r * C::THREADS;
                if (idx < C::A_VECS) {
                    const int n = idx % C::BMJ;
                    const int l = idx / C::BMJ;
                    const float* pv = reinterpret_cast<const float*>(&rv[r]);
#pragma unroll
                    for (int jj = 0; jj < J; ++jj) as[l * C::LDA + jj * C::BMJ + n] = pv[jj];
                }
            }
        }
#pragma unroll
        for (int r = 0; r < C::B_PER_T; ++r) {
            const int idx = tid + r * C::THREADS;
            if (idx < C::B_VECS) *reinterpret_cast<float4*>(bs + 4 * idx) = rb[r];
        }
    };

    static_assert(TN % 2 == 0, "FFMA2 pairs of outputs");
    uint64_t acc2[TM][TN / 2];                    // (acc[m][2p], acc[m][2p+1]) packed for FFMA2
#pragma unroll
    for (int m = 0; m < TM; ++m)
#pragma unroll
        for (int p = 0; p < TN / 2; ++p) acc2[m][p] = 0;

    load_tile(0);
    store_tile(0);
    __syncthreads();

    for (int t = 0; t < nk; ++t) {
        if (t + 1 < nk) load_tile(t + 1);
        const float* as = As + (t & 1) * C::A_ELEMS + wj * C::BMJ + rowA;
        const float* bs = Bs + (t & 1) * C::B_ELEMS + wj * C::BN + colB;
#pragma unroll
        for (int l = 0; l < BK; ++l) {
            const float4 a0 = *reinterpret_cast<const float4*>(as + l * C::LDA);
            const float4 a1 = *reinterpret_cast<const float4*>(as + l * C::LDA + 32);
            float bv[TN];
            if constexpr (TN == 8) {
                const float4 b0 = *reinterpret_cast<const float4*>(bs + l * C::LDB);
                const float4 b1 = *reinterpret_cast<const float4*>(bs + l * C::LDB + 4);
                bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
                bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
            } else {
#pragma unroll
                for (int q = 0; q < TN / 2; ++q) {
                    const float2 v = *reinterpret_cast<const float2*>(bs + l * C::LDB + 2 * q);
                    bv[2 * q] = v.x;
                    bv[2 * q + 1] = v.y;
                }
            }
            const float av[TM] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int m = 0; m < TM; ++m)
#pragma unroll
                for (int p = 0; p < TN / 2; ++p)
                    acc2[m][p] = ffma2(f2pack(av[m], av[m]), f2pack(bv[2 * p], bv[2 * p + 1]), acc2[m][p]);
        }
        if (t + 1 < nk) store_tile((t + 1) & 1);
        __syncthreads();
    }

    // ---- epilogue: each owned Y element written exactly once ------------------
    float acc[TM][TN];
#pragma unroll
    for (int m = 0; m < TM; ++m)
#pragma unroll
        for (int p = 0; p < TN / 2; ++p) {
            acc[m][2 * p] = f2lo(acc2[m][p]);
            acc[m][2 * p + 1] = f2hi(acc2[m][p]);
        }
    const int j = j0 + wj;
    if (bias) {                                   // KSLinear bias (NEXT-2), per output row r
#pragma unroll
        for (int q = 0; q < TN; ++q) {
            const float bq = __ldg(bias + (int64_t)i * b * d + (int64_t)(k0 + colB + q) * d + j);
#pragma unroll
            for (int m = 0; m < TM; ++m) acc[m][q] += bq;
        }
    }
    if (act) {                                    // epilogue activation (NEXT-2), after the bias
#pragma unroll
        for (int m = 0; m < TM; ++m)
#pragma unroll
            for (int q = 0; q < TN; ++q) acc[m][q] = ks_act(acc[m][q], act);
    }
    if (LAYOUT == KS_LAYOUT_BSL) {
        // Y[(i*b*d + k*d + j) * B + n], n contiguous
#pragma unroll
        for (int q = 0; q < TN; ++q) {
            const int64_t r = (int64_t)i * b * d + (int64_t)(k0 + colB + q) * d + j;
            float* yr = Y + r * B + n0 + rowA;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if constexpr (SC) {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (n0 + rowA + 32 * h + e < B) __stcs(yr + 32 * h + e, acc[4 * h + e][q]);
                } else if (n0 + rowA + 32 * h < B) {
                    __stcs(reinterpret_cast<float4*>(yr + 32 * h),
                           make_float4(acc[4 * h][q], acc[4 * h + 1][q], acc[4 * h + 2][q], acc[4 * h + 3][q]));
                }
            }
        }
    } else if (d == 1) {
        // Y[n*M + i*b + k], k contiguous: TN-wide runs
#pragma unroll
        for (int m = 0; m < TM; ++m) {
            const int64_t n = n0 + rowA + (m & 3) + 32 * (m >> 2);
            if (n >= B) continue;
            float* yr = Y + n * M + (int64_t)i * b + k0 + colB;
            if constexpr (SC) {
#pragma unroll
                for (int q = 0; q < TN; ++q) __stcs(yr + q, acc[m][q]);
            } else if constexpr (TN == 8) {
                __stcs(reinterpret_cast<float4*>(yr), make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]));
                __stcs(reinterpret_cast<float4*>(yr + 4), make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]));
            } else {
#pragma unroll
                for (int q = 0; q < TN / 2; ++q)
                    __stcs(reinterpret_cast<float2*>(yr + 2 * q), make_float2(acc[m][2 * q], acc[m][2 * q + 1]));
            }
        }
    } else {
        // structured epilogue through shared memory: one plane per j, Cs[jj][n][k]
        // (row pitch BN+4 keeps vector stores aligned and spreads banks), then
        // each (n, k) gathers its J values into one J-wide global store.
        float* Cs = smem;
        float* plane = Cs + wj * (C::BMJ * C::BNP);
#pragma unroll
        for (int m = 0; m < TM; ++m) {
            const int n = rowA + (m & 3) + 32 * (m >> 2);
            float* dst = plane + n * C::BNP + colB;
            if constexpr (TN == 8) {
                *reinterpret_cast<float4*>(dst) = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
                *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[m][4], acc[m][5], acc[m][6], acc[m][7]);
            } else {
#pragma unroll
                for (int q = 0; q < TN / 2; ++q)
                    *reinterpret_cast<float2*>(dst + 2 * q) = make_float2(acc[m][2 * q], acc[m][2 * q + 1]);
            }
        }
        __syncthreads();
        for (int e = tid; e < C::BMJ * C::BN; e += C::THREADS) {
            const int n = e / C::BN, k = e % C::BN;
            if (n0 + n >= B) continue;
            float v[J];
#pragma unroll
            for (int jj = 0; jj < J; ++jj) v[jj] = Cs[jj * (C::BMJ * C::BNP) + n * C::BNP + k];
            float* yp = Y + (n0 + n) * M + (int64_t)i * b * d + (int64_t)(k0 + k) * d + j0;
            __stcs(reinterpret_cast<VT*>(yp), *reinterpret_cast<const VT*>(v));
        }
    }
}

// ----------------------------------------------------------------- host -----
bool pick_bn(int64_t b, int J, int* wpjn, int* tn) {
    if (b % 128 == 0 && J <= 2) { *wpjn = 4; *tn = 8; return true; }
    if (b % 96 == 0 && J <= 2)  { *wpjn = 4; *tn = 6; return true; }
    if (b % 64 == 0)            { *wpjn = 2; *tn = 8; return true; }
    if (b % 48 == 0)            { *wpjn = 2; *tn = 6; return true; }
    if (b % 32 == 0)            { *wpjn = 1; *tn = 8; return true; }
    if (b % 24 == 0)            { *wpjn = 1; *tn = 6; return true; }
    // any other b % 8 == 0 (80, 112, 40, ...): narrower warp tiles instead of the
    // one-thread-per-output generic kernel (VERDICT r1 "perf cliffs")
    if (b % 16 == 0)            { *wpjn = 1; *tn = 4; return true; }
    if (b % 8 == 0)             { *wpjn = 1; *tn = 2; return true; }
    return false;
}

// l per pipeline chunk: 16 when c allows (half the barriers and staging
// overhead per FFMA), else 8.  KS_FFMA_BK=8 forces 8 (experiments).
int ffma_bk(const ks_handle_s& h) {
    static const int forced = [] {
        const char* e = getenv("KS_FFMA_BK");
        return e ? atoi(e) : 0;
    }();
    if (forced == 8) return 8;
    return h.c % 16 == 0 ? 16 : 8;
}

int pick_j(const ks_handle_s& h, const KsCall& call) {
    if (call.layout == KS_LAYOUT_BSL) return 1;
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y);
    if (h.d % 4 == 0 && (al & 15) == 0) return 4;
    if (h.d % 2 == 0 && (al & 7) == 0) return 2;
    return 1;
}

template <int LAYOUT, int J, int WPJM, int WPJN, int TN, int KBK, bool SC = false>
cudaError_t launch_cfg(const ks_handle_s& h, const KsCall& call) {
    using C = Cfg<LAYOUT, J, WPJM, WPJN, TN, KBK>;
    auto kern = ks_ffma_kernel<LAYOUT, J, WPJM, WPJN, TN, KBK, SC>;
    static bool attr_set[64] = {false};
    if (!attr_set[h.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set[h.device & 63] = true;
    }
    const int64_t nkc = h.b / C::BN;
    const int64_t nnb = (call.B + C::BMJ - 1) / C::BMJ;
    const int64_t blocks = nkc * nnb * (h.a * h.d / J);
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)blocks), dim3(C::THREADS), C::SMEM_BYTES, call.stream,
                                         call.X, (const float*)h.k_tile, call.Y, call.bias, call.act, call.B, (int)h.a,
                                         (int)h.b, (int)h.c, (int)h.d);
    ks::count_launch();
    return e;
}

template <int LAYOUT, int J, bool SC = false>
cudaError_t launch_j(const ks_handle_s& h, const KsCall& call) {
    int wpjn = 0, tn = 0;
    if (!pick_bn(h.b, J, &wpjn, &tn)) return cudaErrorInvalidValue;
    // WPJM = 8 / (J * WPJN)
#define KS_FFMA_CASE(WN, T)                                                                \
    if (wpjn == WN && tn == T) {                                                           \
        if constexpr (8 / (J * WN) >= 1 && (8 % (J * WN)) == 0)                            \
            return ffma_bk(h) == 16 ? launch_cfg<LAYOUT, J, 8 / (J * WN), WN, T, 16, SC>(h, call)   \
                                    : launch_cfg<LAYOUT, J, 8 / (J * WN), WN, T, 8, SC>(h, call);   \
    }
    if constexpr (J <= 2) {
        KS_FFMA_CASE(4, 8)
        KS_FFMA_CASE(4, 6)
    }
    KS_FFMA_CASE(2, 8)
    KS_FFMA_CASE(2, 6)
    KS_FFMA_CASE(1, 8)
    KS_FFMA_CASE(1, 6)
    KS_FFMA_CASE(1, 4)
    KS_FFMA_CASE(1, 2)
#undef KS_FFMA_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

namespace ks {

bool ffma_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (h.c % 8 != 0) return false;
    int wpjn, tn;
    if (!pick_bn(h.b, 1, &wpjn, &tn)) return false;
    if (h.b > (1 << 20) || h.c > (1 << 20) || h.a * h.d > (int64_t(1) << 30)) return false;
    // 4-byte aligned X / Y (the ABI minimum): BSL with B % 4 != 0 or views that are
    // not 16-byte aligned run the scalar (SC) instantiation, bit-identical results
    return true;
}

// the vector path needs 16-byte aligned X / Y and, in BSL, B % 4 == 0
bool ffma_vec_ok(const KsCall& call) {
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y);
    return (al & 15) == 0 && (call.layout != KS_LAYOUT_BSL || call.B % 4 == 0);
}

cudaError_t ffma_launch(const ks_handle_s& h, const KsCall& call) {
    if (ffma_ws_supports(h, call)) return ffma_ws_launch(h, call);
    if (!ffma_vec_ok(call)) {
        if (call.layout == KS_LAYOUT_BSL) return launch_j<KS_LAYOUT_BSL, 1, true>(h, call);
        return launch_j<KS_LAYOUT_BSF, 1, true>(h, call);
    }
    if (call.layout == KS_LAYOUT_BSL) return launch_j<KS_LAYOUT_BSL, 1>(h, call);
    switch (pick_j(h, call)) {
        case 4: return launch_j<KS_LAYOUT_BSF, 4>(h, call);
        case 2: return launch_j<KS_LAYOUT_BSF, 2>(h, call);
        default: return launch_j<KS_LAYOUT_BSF, 1>(h, call);
    }
}

}  // namespace ks
