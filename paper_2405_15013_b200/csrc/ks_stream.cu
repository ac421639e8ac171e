// Streaming KS kernel for small blocks (b, c in {1, 2, 4}): the FFT / square
// dyadic butterfly factors (b = c = 2) and other
// low-arithmetic-intensity patterns.  AI = bc / (2(b+c)) flop/byte <= 1, so
// the roofline is HBM; the kernel is a vectorised, coalesced stream with the
// b x c block of each (i, j) held in registers (output-stationary: each Y
// element is written once, no shared memory needed).
//
// BSF (X is B x N): item = (i, j-vector of V consecutive j); the thread keeps
//   K4[i][k][l][j..j+V) (contiguous in the canonical order: d is fastest) in
//   registers and streams RT batch rows:
//     Y[n, i*b*d + k*d + j..] = sum_l X[n, i*c*d + l*d + j..] * K4[i][k][l][j..]
//   Consecutive threads walk j then i, i.e. along the row: loads of a warp for
//   fixed l cover one contiguous run when d >= 4V*32 and interleave with the
//   l+1 run otherwise (L1/L2 merge the halves; DRAM sees each sector once).
// BSL (X is N x B): item = (i, j, V consecutive batch columns); the b*c
//   weights are warp-uniform scalars, every row load/store is a fully
//   coalesced V-wide vector along the batch.
// Reduction order: l ascending with FP32 FMA, identical in both layouts.
#include "ks_internal.h"

namespace {

template <int V> struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };

template <int V> __device__ __forceinline__ typename Vec<V>::T vzero();
template <> __device__ __forceinline__ float vzero<1>() { return 0.f; }
template <> __device__ __forceinline__ float2 vzero<2>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ float4 vzero<4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ float vfma(float x, float k, float acc) { return fmaf(x, k, acc); }
__device__ __forceinline__ float2 vfma(float2 x, float2 k, float2 acc) {
    return make_float2(fmaf(x.x, k.x, acc.x), fmaf(x.y, k.y, acc.y));
}
__device__ __forceinline__ float4 vfma(float4 x, float4 k, float4 acc) {
    return make_float4(fmaf(x.x, k.x, acc.x), fmaf(x.y, k.y, acc.y), fmaf(x.z, k.z, acc.z),
                       fmaf(x.w, k.w, acc.w));
}
__device__ __forceinline__ float2 vfmas(float2 x, float k, float2 acc) {
    return make_float2(fmaf(x.x, k, acc.x), fmaf(x.y, k, acc.y));
}
__device__ __forceinline__ float4 vfmas(float4 x, float k, float4 acc) {
    return make_float4(fmaf(x.x, k, acc.x), fmaf(x.y, k, acc.y), fmaf(x.z, k, acc.z),
                       fmaf(x.w, k, acc.w));
}
__device__ __forceinline__ float vfmas(float x, float k, float acc) { return fmaf(x, k, acc); }

__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float vadds(float a, float s) { return a + s; }
__device__ __forceinline__ float2 vadds(float2 a, float s) { return make_float2(a.x + s, a.y + s); }
__device__ __forceinline__ float4 vadds(float4 a, float s) { return make_float4(a.x + s, a.y + s, a.z + s, a.w + s); }
__device__ __forceinline__ float vact(float a, int act) { return ks_act(a, act); }
__device__ __forceinline__ float2 vact(float2 a, int act) { return make_float2(ks_act(a.x, act), ks_act(a.y, act)); }
__device__ __forceinline__ float4 vact(float4 a, int act) {
    return make_float4(ks_act(a.x, act), ks_act(a.y, act), ks_act(a.z, act), ks_act(a.w, act));
}

// ---------------------------------------------------------------- BSF ------
template <int BB, int CC, int V, int RT, bool ACT = false>
__global__ void __launch_bounds__(256) ks_stream_bsf(
    const float* __restrict__ X, const float* __restrict__ K4, float* __restrict__ Y,
    const float* __restrict__ bias, int act, int64_t B, int a, int d) {
    using T = typename Vec<V>::T;
    pdl_wait();
    pdl_launch_dependents();
    const int dv = d / V;
    const int64_t P = (int64_t)a * dv;                 // items per batch row
    const int64_t chunks = (B + RT - 1) / RT;
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it >= P * chunks) return;
    const int64_t p = it % P;
    const int64_t chunk = it / P;
    const int i = (int)(p / dv);
    const int j = (int)(p - (int64_t)i * dv) * V;
    const int64_t N = (int64_t)a * CC * d, M = (int64_t)a * BB * d;

    T kr[BB][CC];
#pragma unroll
    for (int k = 0; k < BB; ++k)
#pragma unroll
        for (int l = 0; l < CC; ++l)
            kr[k][l] = __ldg(reinterpret_cast<const T*>(K4 + ((int64_t)(i * BB + k) * CC + l) * d + j));

    T br[BB];                                          // bias of row_{i,j}[k], j..j+V
#pragma unroll
    for (int k = 0; k < BB; ++k)
        br[k] = bias ? __ldg(reinterpret_cast<const T*>(bias + (int64_t)i * BB * d + k * d + j)) : vzero<V>();

    const int64_t n0 = chunk * RT;
    const float* xb = X + n0 * N + (int64_t)i * CC * d + j;
    float* yb = Y + n0 * M + (int64_t)i * BB * d + j;
    T xr[RT][CC];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int l = 0; l < CC; ++l)
            xr[r][l] = (n0 + r < B) ? __ldcs(reinterpret_cast<const T*>(xb + r * N + l * d)) : vzero<V>();
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        if (n0 + r >= B) break;
#pragma unroll
        for (int k = 0; k < BB; ++k) {
            T acc = vzero<V>();
#pragma unroll
            for (int l = 0; l < CC; ++l) acc = vfma(xr[r][l], kr[k][l], acc);
            if (bias) acc = vadd(acc, br[k]);
            if constexpr (ACT) acc = vact(acc, act);     // epilogue activation (compile-time switch)
            __stcs(reinterpret_cast<T*>(yb + r * M + k * d), acc);
        }
    }
}

// ---------------------------------------------------------------- BSL ------
template <int BB, int CC, int V, int RT, bool ACT = false>
__global__ void __launch_bounds__(256) ks_stream_bsl(
    const float* __restrict__ X, const float* __restrict__ K4, float* __restrict__ Y,
    const float* __restrict__ bias, int act, int64_t B, int a, int d, int64_t nblocks) {
    using T = typename Vec<V>::T;
    pdl_wait();
    pdl_launch_dependents();
    const int64_t NV = B / V;
    const int64_t q = blockIdx.x / nblocks;          // q = i*d + j
    const int64_t nb = blockIdx.x - q * nblocks;
    const int i = (int)(q / d);
    const int j = (int)(q - (int64_t)i * d);

    float kr[BB][CC];
#pragma unroll
    for (int k = 0; k < BB; ++k)
#pragma unroll
        for (int l = 0; l < CC; ++l)
            kr[k][l] = __ldg(K4 + ((int64_t)(i * BB + k) * CC + l) * d + j);

    const float* xb = X + ((int64_t)i * CC * d + j) * B;
    float* yb = Y + ((int64_t)i * BB * d + j) * B;
    const int64_t rowx = (int64_t)d * B;             // stride between l (and k) rows
    T xr[RT][CC];
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int64_t nv = (nb * RT + r) * blockDim.x + threadIdx.x;
#pragma unroll
        for (int l = 0; l < CC; ++l)
            xr[r][l] = nv < NV ? __ldcs(reinterpret_cast<const T*>(xb + l * rowx) + nv) : vzero<V>();
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int64_t nv = (nb * RT + r) * blockDim.x + threadIdx.x;
        if (nv >= NV) break;
#pragma unroll
        for (int k = 0; k < BB; ++k) {
            T acc = vzero<V>();
#pragma unroll
            for (int l = 0; l < CC; ++l) acc = vfmas(xr[r][l], kr[k][l], acc);
            if (bias) acc = vadds(acc, __ldg(bias + (int64_t)i * BB * d + k * d + j));
            if constexpr (ACT) acc = vact(acc, act);     // epilogue activation (compile-time switch)
            __stcs(reinterpret_cast<T*>(yb + k * rowx) + nv, acc);
        }
    }
}

// Rows per thread (BSF): measured on the FFT chain, RT = 2, 4, 8 reach the same
// ~90% of copy bandwidth per factor; 8 keeps the fewest threads in flight.
template <int BB, int CC, int V>
cudaError_t launch_bsf(const ks_handle_s& h, const KsCall& call) {
    constexpr int RT = (BB * CC <= 4) ? 8 : 4;
    const int threads = 256;
    const int64_t P = h.a * (h.d / V);
    const int64_t items = P * ((call.B + RT - 1) / RT);
    const int64_t blocks = (items + threads - 1) / threads;
    auto kern = call.act ? ks_stream_bsf<BB, CC, V, RT, true> : ks_stream_bsf<BB, CC, V, RT, false>;
    cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), 0, call.stream,
                                   call.X, (const float*)h.k_canon, call.Y, call.bias, call.act, call.B, (int)h.a, (int)h.d);
    ks::count_launch();
    return e;
}

template <int BB, int CC, int V>
cudaError_t launch_bsl(const ks_handle_s& h, const KsCall& call) {
    constexpr int RT = (BB * CC <= 4) ? 4 : 2;
    const int64_t NV = call.B / V;
    int threads = 256;
    if (NV < 256) threads = (int)((NV + 31) / 32 * 32);
    const int64_t nblocks = (NV + (int64_t)threads * RT - 1) / ((int64_t)threads * RT);
    const int64_t blocks = h.a * h.d * nblocks;
    auto kern = call.act ? ks_stream_bsl<BB, CC, V, RT, true> : ks_stream_bsl<BB, CC, V, RT, false>;
    cudaError_t e = ks::launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), 0, call.stream,
                                   call.X, (const float*)h.k_canon, call.Y, call.bias, call.act, call.B, (int)h.a,
                                   (int)h.d, nblocks);
    ks::count_launch();
    return e;
}

int pick_vec(const ks_handle_s& h, const KsCall& call) {
    const int64_t span = call.layout == KS_LAYOUT_BSF ? h.d : call.B;
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y) |
                         (call.layout == KS_LAYOUT_BSF ? reinterpret_cast<uintptr_t>(call.bias) : 0);
    if (span % 4 == 0 && (al & 15) == 0) return 4;
    if (span % 2 == 0 && (al & 7) == 0) return 2;
    return 1;
}

bool small_bc(int64_t v) { return v == 1 || v == 2 || v == 4; }

template <int BB, int CC>
cudaError_t dispatch_v(const ks_handle_s& h, const KsCall& call) {
    const int V = pick_vec(h, call);
    if (call.layout == KS_LAYOUT_BSF) {
        if (V == 4) return launch_bsf<BB, CC, 4>(h, call);
        if (V == 2) return launch_bsf<BB, CC, 2>(h, call);
        return launch_bsf<BB, CC, 1>(h, call);
    }
    if (V == 4) return launch_bsl<BB, CC, 4>(h, call);
    if (V == 2) return launch_bsl<BB, CC, 2>(h, call);
    return launch_bsl<BB, CC, 1>(h, call);
}

template <int BB>
cudaError_t dispatch_c(const ks_handle_s& h, const KsCall& call) {
    switch (h.c) {
        case 1: return dispatch_v<BB, 1>(h, call);
        case 2: return dispatch_v<BB, 2>(h, call);
        case 4: return dispatch_v<BB, 4>(h, call);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

namespace ks {

bool stream_supports(const ks_handle_s& h, const KsCall& call) {
    if (call.mixed()) return false;
    if (!small_bc(h.b) || !small_bc(h.c)) return false;
    if (h.a > (int64_t(1) << 30) || h.d > (int64_t(1) << 30)) return false;
    if (call.layout == KS_LAYOUT_BSL && h.a * h.d > (int64_t(1) << 31) / 64) return false;
    return true;
}

cudaError_t stream_launch(const ks_handle_s& h, const KsCall& call) {
    switch (h.b) {
        case 1: return dispatch_c<1>(h, call);
        case 2: return dispatch_c<2>(h, call);
        case 4: return dispatch_c<4>(h, call);
    }
    return cudaErrorInvalidValue;
}
}  // namespace ks
