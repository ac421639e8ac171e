// Generic KS kernel: one thread per output element, any pattern, any layout,
// any B.  The correctness floor of the library and the
// fallback for shapes no specialised family covers.
//
// For output (n, r) with r = i*b*d + k*d + j (row_{i,j}[k], Alg. 2 line 3,
// PAPER.md:356) the reduction runs over col_{i,j} = {i*c*d + l*d + j}
// (Alg. 2 line 4), l ascending, FP32 FMA:
//     Y(n, r) = sum_l X(n, i*c*d + l*d + j) * K4[i][k][l][j].
// Every output is written exactly once (row sets partition [0,M)).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ks_internal.h"

namespace {

// XL / YL: layouts of X and Y (equal except for ks_matmul_io and mixed-layout
// chain intermediates); outputs are enumerated in Y's order.
template <int XL, int YL>
__global__ void __launch_bounds__(256) ks_generic_kernel(
    const float* __restrict__ X, const float* __restrict__ K4, float* __restrict__ Y,
    const float* __restrict__ bias, int act, int64_t B, int64_t a, int64_t b, int64_t c, int64_t d) {
    pdl_wait();
    pdl_launch_dependents();
    const int64_t M = a * b * d, N = a * c * d;
    const int64_t total = B * M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t n, r;
        if (YL == KS_LAYOUT_BSF) { n = e / M; r = e - n * M; }
        else                         { r = e / B; n = e - r * B; }
        const int64_t i = r / (b * d);
        const int64_t rem = r - i * b * d;
        const int64_t k = rem / d;
        const int64_t j = rem - k * d;
        const int64_t s0 = i * c * d + j;                // col_{i,j}[0]
        const float* kp = K4 + ((i * b + k) * c) * d + j;  // K4[i][k][0][j]
        float acc = 0.f;
        for (int64_t l = 0; l < c; ++l) {
            const int64_t s = s0 + l * d;
            const float x = XL == KS_LAYOUT_BSF ? X[n * N + s] : X[s * B + n];
            acc = fmaf(x, kp[l * d], acc);
        }
        Y[e] = ks_act(bias ? acc + bias[r] : acc, act);
    }
}

// Half-precision generic kernel: same reduction order, FP32 accumulation,
// output rounded to nearest-even (half handles whose pattern the tensor-core
// kernel cannot take).
template <typename T, int XL, int YL>
__global__ void __launch_bounds__(256) ks_generic_half_kernel(
    const T* __restrict__ X, const T* __restrict__ K4, T* __restrict__ Y, const T* __restrict__ bias, int act,
    int64_t B, int64_t a, int64_t b, int64_t c, int64_t d) {
    pdl_wait();
    pdl_launch_dependents();
    const int64_t M = a * b * d, N = a * c * d;
    const int64_t total = B * M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t n, r;
        if (YL == KS_LAYOUT_BSF) { n = e / M; r = e - n * M; }
        else                         { r = e / B; n = e - r * B; }
        const int64_t i = r / (b * d);
        const int64_t rem = r - i * b * d;
        const int64_t k = rem / d;
        const int64_t j = rem - k * d;
        const int64_t s0 = i * c * d + j;
        const T* kp = K4 + ((i * b + k) * c) * d + j;
        float acc = 0.f;
        for (int64_t l = 0; l < c; ++l) {
            const int64_t s = s0 + l * d;
            const float x = (float)(XL == KS_LAYOUT_BSF ? X[n * N + s] : X[s * B + n]);
            acc = fmaf(x, (float)kp[l * d], acc);
        }
        if (bias) acc += (float)bias[r];
        Y[e] = T(ks_act(acc, act));
    }
}

template <typename T>
cudaError_t launch_generic_half(const ks_handle_s& h, const KsCall& call) {
    const int threads = 256;
    const int64_t total = call.B * h.M;
    int64_t blocks = (total + threads - 1) / threads;
    const int64_t cap = (int64_t)ks::num_sms(h.device) * 8 * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const T* X = reinterpret_cast<const T*>(call.X);
    T* Y = reinterpret_cast<T*>(call.Y);
    const T* K = reinterpret_cast<const T*>(h.k_canon);
    const T* bias = reinterpret_cast<const T*>(call.bias);
    constexpr int F = KS_LAYOUT_BSF, L = KS_LAYOUT_BSL;
    const bool xf = call.layout == F, yf = call.ylayout() == F;
    auto kern = xf ? (yf ? ks_generic_half_kernel<T, F, F> : ks_generic_half_kernel<T, F, L>)
                   : (yf ? ks_generic_half_kernel<T, L, F> : ks_generic_half_kernel<T, L, L>);
    const cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), 0, call.stream, X, K, Y, bias, call.act,
                                         call.B, (int64_t)h.a, (int64_t)h.b, (int64_t)h.c, (int64_t)h.d);
    ks::count_launch();
    return e;
}

}  // namespace

namespace ks {

cudaError_t generic_half_launch(const ks_handle_s& h, const KsCall& call) {
    return h.dtype == KS_DTYPE_BF16 ? launch_generic_half<__nv_bfloat16>(h, call)
                                    : launch_generic_half<__half>(h, call);
}

bool generic_supports(const ks_handle_s&, const KsCall&) { return true; }

cudaError_t generic_launch(const ks_handle_s& h, const KsCall& call) {
    const int threads = 256;
    const int64_t total = call.B * h.M;
    int64_t blocks = (total + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms(h.device) * 8 * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    constexpr int F = KS_LAYOUT_BSF, L = KS_LAYOUT_BSL;
    const bool xf = call.layout == F, yf = call.ylayout() == F;
    auto kern = xf ? (yf ? ks_generic_kernel<F, F> : ks_generic_kernel<F, L>)
                   : (yf ? ks_generic_kernel<L, F> : ks_generic_kernel<L, L>);
    const cudaError_t e = launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), 0, call.stream, call.X,
                                     (const float*)h.k_canon, call.Y, call.bias, call.act, call.B, (int64_t)h.a, (int64_t)h.b,
                                     (int64_t)h.c, (int64_t)h.d);
    count_launch();
    return e;
}

}  // namespace ks
