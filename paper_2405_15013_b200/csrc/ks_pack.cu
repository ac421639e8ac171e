// Offline repacking of a KS factor (ks_pack_weights).  An integer permutation
// of the abcd canonical values into the layouts the kernels read:
//   k_tile[(i*d+j)][l][k]  = K4[i][k][l][j]   K^T[col_ij, row_ij] contiguous per
//                                            tile, k fastest
//   k_tf32[(i*d+j)][k][l]  = rna_tf32(K4[i][k][l][j])   K-major B operand of the
//                                            tcgen05 TF32 kernel, pre-rounded
//   k_lo  [(i*d+j)][k][l]  = rna_tf32(K4[i][k][l][j] - k_tf32[...]) -- the low
//                                            part of the 3xTF32 split (F32X3)
//   k_dense[i][k*d+j][l*d+j'] = rna_tf32(K4[i][k][l][j]) if j == j' else 0 --
//                                            densified super-blocks (TF32, small d)
// Excluded from timing.
#include "ks_internal.h"

namespace {

__device__ __forceinline__ float round_tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void pack_kernel(const float* __restrict__ k4, float* __restrict__ tile,
                            float* __restrict__ tf32, int64_t a, int64_t b, int64_t c,
                            int64_t d) {
    const int64_t nnz = a * b * c * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        // e = ((i*b + k)*c + l)*d + j
        const int64_t j = e % d;
        int64_t t = e / d;
        const int64_t l = t % c;
        t /= c;
        const int64_t k = t % b;
        const int64_t i = t / b;
        const float v = k4[e];
        const int64_t q = i * d + j;
        tile[(q * c + l) * b + k] = v;
        tf32[(q * b + k) * c + l] = round_tf32_rna(v);
    }
}

__global__ void pack_lo_kernel(const float* __restrict__ k4, float* __restrict__ lo, int64_t a, int64_t b,
                               int64_t c, int64_t d) {
    const int64_t nnz = a * b * c * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e % d;
        int64_t t = e / d;
        const int64_t l = t % c;
        t /= c;
        const int64_t k = t % b;
        const int64_t i = t / b;
        const float v = k4[e];
        lo[((i * d + j) * b + k) * c + l] = round_tf32_rna(v - round_tf32_rna(v));
    }
}

// Densified super-blocks (TF32 BSF, small d): block i of K as a dense
// (b d) x (c d) matrix, D_i[k*d + j][l*d + j'] = K4[i][k][l][j] if j == j' else 0
// (Def. 1: supp(K) within I_a (x) 1_{bd x cd}), RNA-rounded.
__global__ void pack_dense_kernel(const float* __restrict__ k4, float* __restrict__ dense, int64_t a, int64_t b,
                                  int64_t c, int64_t d) {
    const int64_t bd = b * d, cd = c * d, tot = a * bd * cd;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e % cd;           // l*d + j'
        const int64_t r = (e / cd) % bd;    // k*d + j
        const int64_t i = e / (cd * bd);
        const int64_t j = r % d, k = r / d, jp = s % d, l = s / d;
        dense[e] = (j == jp) ? round_tf32_rna(k4[((i * b + k) * c + l) * d + j]) : 0.0f;
    }
}

// Half handles: a pure permutation of the 16-bit values into [i*d+j][k][l]
// (the tensor-core weight tiles); no rounding.
__global__ void pack_half_kernel(const uint16_t* __restrict__ k4, uint16_t* __restrict__ mma, int64_t a,
                                 int64_t b, int64_t c, int64_t d) {
    const int64_t nnz = a * b * c * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e % d;
        int64_t t = e / d;
        const int64_t l = t % c;
        t /= c;
        const int64_t k = t % b;
        const int64_t i = t / b;
        mma[((i * d + j) * b + k) * c + l] = k4[e];
    }
}

}  // namespace

namespace ks {

cudaError_t pack_half(const ks_handle_s& h, cudaStream_t s) {
    const int threads = 256;
    int64_t blocks = (h.nnz + threads - 1) / threads;
    if (blocks > 65535 * 8) blocks = 65535 * 8;
    pack_half_kernel<<<(unsigned)blocks, threads, 0, s>>>(reinterpret_cast<const uint16_t*>(h.k_canon),
                                                          reinterpret_cast<uint16_t*>(h.k_tf32), h.a, h.b, h.c, h.d);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pack_lo(const ks_handle_s& h, cudaStream_t s) {
    const int threads = 256;
    int64_t blocks = (h.nnz + threads - 1) / threads;
    if (blocks > 65535 * 8) blocks = 65535 * 8;
    pack_lo_kernel<<<(unsigned)blocks, threads, 0, s>>>(h.k_canon, h.k_lo, h.a, h.b, h.c, h.d);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pack_dense(const ks_handle_s& h, cudaStream_t s) {
    const int threads = 256;
    const int64_t tot = h.nnz * h.d;
    int64_t blocks = (tot + threads - 1) / threads;
    if (blocks > 65535 * 8) blocks = 65535 * 8;
    pack_dense_kernel<<<(unsigned)blocks, threads, 0, s>>>(h.k_canon, h.k_dense, h.a, h.b, h.c, h.d);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pack_tiles(const ks_handle_s& h, cudaStream_t s) {
    const int threads = 256;
    int64_t blocks = (h.nnz + threads - 1) / threads;
    if (blocks > 65535 * 8) blocks = 65535 * 8;
    pack_kernel<<<(unsigned)blocks, threads, 0, s>>>(h.k_canon, h.k_tile, h.k_tf32, h.a, h.b, h.c, h.d);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ks
