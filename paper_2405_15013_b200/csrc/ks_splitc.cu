// Small-batch split-c kernel ("Small B: lanes split c and
// combine with __shfl_xor_sync in a fixed butterfly order", the
// kernel's warp-level parallelism; north star "warp-shuffle reductions").
//
// For B <= KS_SPLITC_MAX_B a 128-row output tile leaves most of a tensor-core or
// register-tiled FFMA tile empty; here the parallelism comes from the reduction
// instead.  One warp owns a 4-row x 8-output block of one KS block (i, j):
//   * lane t takes the l in {t, t + 32, ...} (c split across the 32 lanes), keeps
//     its 8 K^T values per l in registers (k_tile[(i d + j)][l][k0 .. k0+8), one
//     32-byte sector per lane) and its X values of the 4 rows, and accumulates
//     32 partial sums acc[row][k] (l ascending within the lane);
//   * one reduce-transpose butterfly of 31 __shfl_xor_sync (offsets 16, 8, 4, 2, 1)
//     sums the 32 partial sums across lanes so that lane t ends with output
//     t = row * 8 + k: a fixed order, so the result is deterministic run to run.
// Each Y element is written once (no atomics).  The summation order differs
// from the l-ascending FP32 kernels (R11): results agree to FP32
// rounding, and are bit-exact on small-integer data (exact arithmetic).
#include "ks_internal.h"

namespace {

constexpr int SC_ROWS = 4;     // batch rows per warp
constexpr int SC_K = 8;        // outputs (k) per warp
constexpr int SC_WARPS = 4;    // warps per CTA

template <int LAYOUT, int CL>
__global__ void __launch_bounds__(SC_WARPS * 32)
ks_splitc_kernel(const float* __restrict__ X, const float* __restrict__ Kt, float* __restrict__ Y,
                 const float* __restrict__ bias, int act, int64_t B, int a, int b, int c, int d) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * SC_WARPS + (threadIdx.x >> 5);
    const int nkc = b / SC_K;
    const int64_t nrb = (B + SC_ROWS - 1) / SC_ROWS;
    const int64_t total = (int64_t)a * d * nkc * nrb;
    pdl_wait();
    pdl_launch_dependents();
    if (wid >= total) return;
    const int kc = (int)(wid % nkc);
    const int64_t rb = (wid / nkc) % nrb;
    const int q = (int)(wid / ((int64_t)nkc * nrb));      // i * d + j
    const int i = q / d, j = q % d;
    const int k0 = kc * SC_K;
    const int64_t n0 = rb * SC_ROWS;
    const int64_t N = (int64_t)a * c * d, M = (int64_t)a * b * d;

    float acc[SC_ROWS][SC_K];
#pragma unroll
    for (int r = 0; r < SC_ROWS; ++r)
#pragma unroll
        for (int k = 0; k < SC_K; ++k) acc[r][k] = 0.f;
#pragma unroll
    for (int u = 0; u < CL; ++u) {
        const int l = lane + 32 * u;
        if (l < c) {
            // K^T row l of block q: 8 consecutive k (one 32-byte sector)
            const float4* wp = reinterpret_cast<const float4*>(Kt + ((int64_t)q * c + l) * b + k0);
            const float4 w0 = __ldg(wp), w1 = __ldg(wp + 1);
            const float w[SC_K] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            const int64_t s = ((int64_t)i * c + l) * d + j;         // column of X
#pragma unroll
            for (int r = 0; r < SC_ROWS; ++r) {
                const int64_t n = n0 + r;
                const float x = n < B ? __ldg(LAYOUT == KS_LAYOUT_BSL ? X + s * B + n : X + n * N + s) : 0.f;
#pragma unroll
                for (int k = 0; k < SC_K; ++k) acc[r][k] = fmaf(x, w[k], acc[r][k]);
            }
        }
    }
    // reduce-transpose: after the step with offset `off`, a lane keeps the half of its
    // values whose index bit log2(off) equals its own lane bit; it ends with index = lane
    float v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = acc[t / SC_K][t % SC_K];
#pragma unroll
    for (int off = 16, half = 16; off >= 1; off >>= 1, half >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int t = 0; t < half; ++t) {
            const float send = up ? v[t] : v[t + half];
            const float keep = up ? v[t + half] : v[t];
            v[t] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    const int r = lane / SC_K, k = lane % SC_K;
    const int64_t n = n0 + r;
    if (n < B) {
        const int64_t row = (int64_t)i * b * d + (int64_t)(k0 + k) * d + j;
        float y = v[0];
        if (bias) y += __ldg(bias + row);
        y = ks_act(y, act);
        if (LAYOUT == KS_LAYOUT_BSL)
            Y[row * B + n] = y;
        else
            Y[n * M + row] = y;
    }
}

template <int LAYOUT>
cudaError_t launch_splitc(const ks_handle_s& h, const KsCall& call) {
    const int cl = (int)((h.c + 31) / 32);
    const int64_t warps = h.a * h.d * (h.b / SC_K) * ((call.B + SC_ROWS - 1) / SC_ROWS);
    const dim3 grid((unsigned)((warps + SC_WARPS - 1) / SC_WARPS)), block(SC_WARPS * 32);
    cudaError_t e = cudaErrorInvalidValue;
#define KS_SC_CASE(n)                                                                                     \
    case n:                                                                                               \
        e = ks::launch_pdl(ks_splitc_kernel<LAYOUT, n>, grid, block, 0, call.stream, call.X, h.k_tile, call.Y, \
                           call.bias, call.act, call.B, (int)h.a, (int)h.b, (int)h.c, (int)h.d);          \
        break;
    switch (cl) {
        KS_SC_CASE(1) KS_SC_CASE(2) KS_SC_CASE(3) KS_SC_CASE(4) KS_SC_CASE(5) KS_SC_CASE(6) KS_SC_CASE(7)
        KS_SC_CASE(8)
    }
#undef KS_SC_CASE
    ks::count_launch();
    return e;
}

}  // namespace

namespace ks {

// FP32 handles, 1 <= B <= KS_SPLITC_MAX_B, GEMM-like blocks (b a multiple of 8,
// 16 <= c <= 256), 32-byte aligned packed K^T rows (b % 8 == 0 gives that).
// Measured against the FFMA / generic families (device time per call from CUDA-graph
// replay, profiles/r02/small_b.jsonl): 2-8x faster for every BSF case B <= 64 and for
// BSL up to B = 16; in BSL a warp's 4 rows are 16-byte pieces of each X row, so at
// B >= 32 with more than 8 M multiply-adds per call the FFMA / generic kernels win.
bool splitc_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (h.dtype != KS_DTYPE_F32 || call.B < 1 || call.B > KS_SPLITC_MAX_B) return false;
    if (h.b % SC_K != 0 || h.c < 16 || h.c > 256) return false;
    if (h.a * h.d * h.c >= (int64_t(1) << 31) || h.a * h.d * h.b >= (int64_t(1) << 31)) return false;
    return true;
}

bool splitc_preferred(const ks_handle_s& h, const KsCall& call) {
    if (!splitc_supports(h, call)) return false;
    return !(call.layout == KS_LAYOUT_BSL && call.B > 16 && call.B * h.nnz > (int64_t(8) << 20));
}

cudaError_t splitc_launch(const ks_handle_s& h, const KsCall& call) {
    if (call.layout == KS_LAYOUT_BSL) return launch_splitc<KS_LAYOUT_BSL>(h, call);
    return launch_splitc<KS_LAYOUT_BSF>(h, call);
}

}  // namespace ks
