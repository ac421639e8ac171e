// Fused multi-factor chain kernel: applies every factor of
// a square small-block chain (b_l = c_l = BB in {2, 4}, all dimensions equal,
// e.g. the FFT / square dyadic butterfly, Table 3)
// to R batch rows held in shared memory, so X is read once and Y written once
// instead of one HBM round trip per factor.
//
// Why it is legal in place: with b = c the output rows row_{i,j} (Alg. 2 line 3,
// PAPER.md:356) and input columns col_{i,j} (line 4) of a block are the same
// index set {i*b*d + l*d + j}, and the blocks partition [0, N),
// so each (i, j) block of each row is read and rewritten by exactly one thread.
//
// Arithmetic per output: l ascending, one FP32 FMA chain starting from 0 -- the
// exact operation sequence of the per-factor kernels, so the fused chain is
// bit-identical to L separate ks_matmul launches (tested).
//
// Passes: consecutive square-dyadic factors whose d doubles (the DIT order of
// the chain application, K_L first) are grouped up to 3 per shared-memory pass
// ("radix-8"): a thread loads the 8 values {base + m*d0}, applies the 2-3
// factors in registers and writes them back, cutting shared-memory traffic 3x.
// Other factor sequences run one factor per pass.
//
// Bank-conflict-free rows (SWZ): when N % 256 == 0 the row groups move by
// tensor TMA with SWIZZLE_128B, so float e of a row sits at e ^ (((e >> 5) & 7) << 2)
// (16-byte chunks XOR-permuted within each 128-byte segment).  Every pass's
// warp accesses then hit 32 distinct banks: the d0 = 8 radix-8 pass (lanes
// 8 j x 4 blocks, addresses 64 blk + 8 m + j) was 4-way conflicted and the d0 = 1
// pass (32-byte per-lane runs) 2-way -- half of all shared-memory wavefronts
// were conflicts (ncu, profiles/r02/fused_*).  The arithmetic is unchanged.
#include "ks_umma.cuh"

#include <cstdlib>

namespace {

constexpr int MAXF = 32;
constexpr int THREADS = 512;

// position of float e of a row in the SWIZZLE_128B layout (an involution)
template <bool SWZ>
__device__ __forceinline__ uint32_t rpos(uint32_t e) {
    if constexpr (SWZ) return e ^ (((e >> 5) & 7u) << 2);
    else return e;
}

struct FusedFactor {
    const float* k;   // canonical K4 of the factor
    int a, d;
};

struct FusedParams {
    FusedFactor f[MAXF];   // application order (K_L first)
    int pass_len[MAXF];    // number of factors in each pass (1..3), passes in order
    int pass_first[MAXF];  // index in f of each pass's first factor
    int npass;
    int N;                 // row length (all dims equal)
    int resident;          // number of radix-8 passes whose weights live in TMEM (0..2)
    int res_pass[2];       // which passes (the TMEM slot is the index in this list)
    int part_pass;         // a third pass whose first two factors live in the last 128 columns, or -1
    int act;               // epilogue activation after the bias (ks_activation_t, NEXT-2)
    int pf_pass;           // the next group's load is issued after this pass (-1: before the first)
};

// Weights of one radix-2^T item (T consecutive dyadic factors, b = c = 2, with
// d0, 2 d0, 4 d0): kw[t][p][kl] = K4[i][k][l][jt] of factor t, pair p (bit t of
// the element index m cleared), kl = 2k + l.
// T0: load only factors t >= T0 (the others come from tensor memory).
template <int T, int T0 = 0>
__device__ __forceinline__ void dyadic_load(const FusedFactor* F, int it, float (&kw)[T][(1 << T) / 2][4]) {
    constexpr int E = 1 << T;
    const int d0 = F[0].d;
    const int j = it % d0;
    const int blk = it / d0;                      // super-block of size E*d0
    if (d0 == 1) {
        // the item's weights of factor t are one 2^(T+1)-float run starting at
        // blk * 2^(T+1): vector loads; offset of (pair p, k, l) inside the run is
        // (p >> t) * 4 * 2^t + (2k + l) * 2^t + (p mod 2^t)
#pragma unroll
        for (int t = T0; t < T; ++t) {
            float kk[2 * E];
            const float4* src = reinterpret_cast<const float4*>(F[t].k + (int64_t)blk * (2 * E));
#pragma unroll
            for (int q = 0; q < E / 2; ++q) {
                const float4 w = __ldg(src + q);
                kk[4 * q] = w.x; kk[4 * q + 1] = w.y; kk[4 * q + 2] = w.z; kk[4 * q + 3] = w.w;
            }
#pragma unroll
            for (int p = 0; p < E / 2; ++p)
#pragma unroll
                for (int kl = 0; kl < 4; ++kl)
                    kw[t][p][kl] = kk[(p >> t) * 4 * (1 << t) + kl * (1 << t) + (p & ((1 << t) - 1))];
        }
    } else {
#pragma unroll
        for (int t = T0; t < T; ++t) {
            const int dt = d0 << t;
#pragma unroll
            for (int p = 0; p < E / 2; ++p) {
                // p enumerates m with bit t cleared; s = base + m*d0 = d0*(blk*E + m) + j
                // with j < d0, so for factor t (d_t = d0 * 2^t, super-block 2*d_t):
                //   i  = s / (2 d_t) = (blk*E + m) >> (t+1),  j_t = s % d_t = d0*(m mod 2^t) + j
                const int lo = p & ((1 << t) - 1);
                const int m = ((p >> t) << (t + 1)) | lo;
                const int i = (blk << (T - t - 1)) + (m >> (t + 1));
                const int jt = d0 * (m & ((1 << t) - 1)) + j;
                const float* kp = F[t].k + ((int64_t)(i * 2) * 2) * dt + jt;   // K4[i][0][0][jt]
                kw[t][p][0] = __ldg(kp);              // k=0,l=0
                kw[t][p][1] = __ldg(kp + dt);         // k=0,l=1
                kw[t][p][2] = __ldg(kp + 2 * dt);     // k=1,l=0
                kw[t][p][3] = __ldg(kp + 3 * dt);     // k=1,l=1
            }
        }
    }
}

// Apply an item's T factors to its E elements {base + m*d0} of every row.
template <int T, bool SWZ = false>
__device__ __forceinline__ void dyadic_apply(float* sm, int rows, int N, int d0, int it,
                                             const float (&kw)[T][(1 << T) / 2][4]) {
    constexpr int E = 1 << T;
    const int base = (it / d0) * (E * d0) + it % d0;
    for (int r = 0; r < rows; ++r) {
        float* row = sm + (size_t)r * N;
        float v[E];
        if (d0 == 1) {                             // E consecutive floats: vector shared loads
#pragma unroll
            for (int m = 0; m < E; m += 4) {
                const float4 q = *reinterpret_cast<const float4*>(row + rpos<SWZ>(base + m));
                v[m] = q.x; v[m + 1] = q.y; v[m + 2] = q.z; v[m + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = row[rpos<SWZ>(base + m * d0)];
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
#pragma unroll
            for (int p = 0; p < E / 2; ++p) {
                const int lo = p & ((1 << t) - 1);
                const int m0 = ((p >> t) << (t + 1)) | lo;
                const int m1 = m0 | (1 << t);
                const float x0 = v[m0], x1 = v[m1];
                v[m0] = fmaf(x1, kw[t][p][1], fmaf(x0, kw[t][p][0], 0.f));
                v[m1] = fmaf(x1, kw[t][p][3], fmaf(x0, kw[t][p][2], 0.f));
            }
        }
        if (d0 == 1) {
#pragma unroll
            for (int m = 0; m < E; m += 4)
                *reinterpret_cast<float4*>(row + rpos<SWZ>(base + m)) = make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]);
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) row[rpos<SWZ>(base + m * d0)] = v[m];
        }
    }
}

// dyadic_apply with the stride d0 = 2^LD0 a compile-time constant: the E
// element offsets m*d0 fold into the shared-memory instructions' immediates
// (the runtime-stride form spends ~2 integer instructions per element on
// addresses -- measured: 56% of the fused kernel's instructions were not FFMA),
// and rows are processed two at a time (both rows' loads issue before either
// row's FMAs) for instruction-level parallelism.  Same operations, same order
// per output as dyadic_apply: bit-identical.
template <int T, int LD0, bool SWZ>
__device__ __forceinline__ void dyadic_row_load(const float* row, uint32_t base, float (&v)[1 << T]) {
    constexpr int E = 1 << T, D0 = 1 << LD0;
    if constexpr (D0 == 1) {
#pragma unroll
        for (int m = 0; m < E; m += 4) {
            const float4 q = *reinterpret_cast<const float4*>(row + rpos<SWZ>(base + m));
            v[m] = q.x; v[m + 1] = q.y; v[m + 2] = q.z; v[m + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = row[rpos<SWZ>(base + m * D0)];
    }
}
template <int T, int LD0, bool SWZ>
__device__ __forceinline__ void dyadic_row_store(float* row, uint32_t base, const float (&v)[1 << T]) {
    constexpr int E = 1 << T, D0 = 1 << LD0;
    if constexpr (D0 == 1) {
#pragma unroll
        for (int m = 0; m < E; m += 4)
            *reinterpret_cast<float4*>(row + rpos<SWZ>(base + m)) = make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]);
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) row[rpos<SWZ>(base + m * D0)] = v[m];
    }
}
template <int T>
__device__ __forceinline__ void dyadic_row_math(float (&v)[1 << T], const float (&kw)[T][(1 << T) / 2][4]) {
    constexpr int E = 1 << T;
#pragma unroll
    for (int t = 0; t < T; ++t) {
#pragma unroll
        for (int p = 0; p < E / 2; ++p) {
            const int lo = p & ((1 << t) - 1);
            const int m0 = ((p >> t) << (t + 1)) | lo;
            const int m1 = m0 | (1 << t);
            const float x0 = v[m0], x1 = v[m1];
            v[m0] = fmaf(x1, kw[t][p][1], fmaf(x0, kw[t][p][0], 0.f));
            v[m1] = fmaf(x1, kw[t][p][3], fmaf(x0, kw[t][p][2], 0.f));
        }
    }
}
template <int T, int LD0, bool SWZ>
__device__ __forceinline__ void dyadic_apply_c(float* sm, int rows, int N, int it,
                                               const float (&kw)[T][(1 << T) / 2][4]) {
    constexpr int E = 1 << T, D0 = 1 << LD0;
    const uint32_t base = (uint32_t)((it >> LD0) * (E * D0) + (it & (D0 - 1)));
    float* row = sm;
    int r = 0;
    for (; r + 1 < rows; r += 2, row += 2 * N) {
        // two rows at once with FFMA2: lane 0 = row r, lane 1 = row r+1, the weight a
        // broadcast scalar -- per lane exactly dyadic_row_math's fmaf chain (bit-identical)
        float v0[E], v1[E];
        dyadic_row_load<T, LD0, SWZ>(row, base, v0);
        dyadic_row_load<T, LD0, SWZ>(row + N, base, v1);
        uint64_t v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = f2pack(v0[m], v1[m]);
#pragma unroll
        for (int t = 0; t < T; ++t) {
#pragma unroll
            for (int p = 0; p < E / 2; ++p) {
                const int lo = p & ((1 << t) - 1);
                const int m0 = ((p >> t) << (t + 1)) | lo;
                const int m1 = m0 | (1 << t);
                const uint64_t x0 = v[m0], x1 = v[m1];
                const float* k = kw[t][p];
                v[m0] = ffma2(x1, f2pack(k[1], k[1]), ffma2(x0, f2pack(k[0], k[0]), 0));
                v[m1] = ffma2(x1, f2pack(k[3], k[3]), ffma2(x0, f2pack(k[2], k[2]), 0));
            }
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            v0[m] = f2lo(v[m]);
            v1[m] = f2hi(v[m]);
        }
        dyadic_row_store<T, LD0, SWZ>(row, base, v0);
        dyadic_row_store<T, LD0, SWZ>(row + N, base, v1);
    }
    if (r < rows) {
        float v0[E];
        dyadic_row_load<T, LD0, SWZ>(row, base, v0);
        dyadic_row_math<T>(v0, kw);
        dyadic_row_store<T, LD0, SWZ>(row, base, v0);
    }
}

// runtime d0 (a power of two, d0 * 2^T <= N) -> the compile-time form; d0 up to 2^13
template <int T, bool SWZ>
__device__ __forceinline__ void dyadic_apply_any(float* sm, int rows, int N, int d0, int it,
                                                 const float (&kw)[T][(1 << T) / 2][4]) {
    switch (__ffs(d0) - 1) {
#define KS_FUSED_D0(L) \
    case L: dyadic_apply_c<T, L, SWZ>(sm, rows, N, it, kw); return;
        KS_FUSED_D0(0) KS_FUSED_D0(1) KS_FUSED_D0(2) KS_FUSED_D0(3) KS_FUSED_D0(4) KS_FUSED_D0(5) KS_FUSED_D0(6)
        KS_FUSED_D0(7) KS_FUSED_D0(8) KS_FUSED_D0(9) KS_FUSED_D0(10) KS_FUSED_D0(11) KS_FUSED_D0(12)
        KS_FUSED_D0(13)
#undef KS_FUSED_D0
    }
    dyadic_apply<T, SWZ>(sm, rows, N, d0, it, kw);
}

// One radix-2^T pass over all rows of the tile, T consecutive dyadic factors
// (b = c = 2) with d, 2d, 4d: weights loaded (from L2) per item, then applied to
// every row of the group.
template <int T, bool SWZ>
__device__ __forceinline__ void dyadic_pass(float* sm, int rows, int N, const FusedFactor* F) {
    constexpr int E = 1 << T;
    const int nitem = N / E;                      // (super-block of the last factor, j) pairs
    for (int it = threadIdx.x; it < nitem; it += THREADS) {
        float kw[T][E / 2][4];
        dyadic_load<T>(F, it, kw);
        dyadic_apply_any<T, SWZ>(sm, rows, N, F[0].d, it, kw);
    }
}

// ---- TMEM-resident weights (P.resident radix-8 passes) -----------------------
// A pass's weights are re-read from L2 for every group of R rows (they do not fit
// beside the row buffers in shared memory); P.resident passes (<= 2; the d0 = 1
// pass, whose weight loads are the least coalesced, first) keep them in tensor memory
// instead, loaded once per CTA: thread t (one item
// per thread, N / 8 == THREADS) owns 96 columns of TMEM lane (warp % 4) * 32 +
// lane -- 4 warps share a lane quarter, 4 x 96 = 384 of the 512 columns -- and
// reads its 48 weights back with three tcgen05.ld .x16 per pass and row group.
__device__ __forceinline__ uint32_t tmem_w_addr(uint32_t tmem, int ps, int q) {
    const int warp = threadIdx.x >> 5;
    return tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 96 + ps * 48 + 16 * q);
}
// the 128 columns left after two resident passes: 32 per thread, factors 0-1 of a third pass
__device__ __forceinline__ uint32_t tmem_part_addr(uint32_t tmem, int q) {
    const int warp = threadIdx.x >> 5;
    return tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(384 + (warp >> 2) * 32 + 16 * q);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
          "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
          "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
          "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
          "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
          "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_ld16f(uint32_t taddr, float* v) {
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

// One factor with b = c = BB (any a, d) per pass.
template <int BB, bool SWZ>
__device__ __forceinline__ void block_pass(float* sm, int rows, int N, const FusedFactor& F) {
    const int d = F.d;
    const int nblk = F.a * d;
    for (int blk = threadIdx.x; blk < nblk; blk += THREADS) {
        const int i = blk / d, j = blk % d;
        float kr[BB][BB];
#pragma unroll
        for (int k = 0; k < BB; ++k)
#pragma unroll
            for (int l = 0; l < BB; ++l) kr[k][l] = __ldg(F.k + ((int64_t)(i * BB + k) * BB + l) * d + j);
        const int base = i * BB * d + j;
        for (int r = 0; r < rows; ++r) {
            float* row = sm + (size_t)r * N;
            float x[BB];
#pragma unroll
            for (int l = 0; l < BB; ++l) x[l] = row[rpos<SWZ>(base + l * d)];
#pragma unroll
            for (int k = 0; k < BB; ++k) {
                float acc = 0.f;
#pragma unroll
                for (int l = 0; l < BB; ++l) acc = fmaf(x[l], kr[k][l], acc);
                row[rpos<SWZ>(base + k * d)] = acc;
            }
        }
    }
}


// Row groups move by bulk asynchronous copies (TMA engine; SWZ: tensor copies of
// a {32, N/32, R} box with SWIZZLE_128B, else cp.async.bulk): the next group
// streams into the second buffer while this one is computed, and the finished
// group drains to HBM in the background.
template <int BB, bool SWZ>
__global__ void __launch_bounds__(THREADS, 1)
ks_chain_fused_kernel(const float* __restrict__ X, float* __restrict__ Y, const float* __restrict__ bias, int64_t B,
                      const __grid_constant__ FusedParams P, int R, const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ CUtensorMap ymap) {
    extern __shared__ __align__(1024) float4 sm4[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ uint32_t tmem_slot;
    if (BB == 2 && P.resident > 0) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    pdl_wait();
    pdl_launch_dependents();
    if (BB == 2 && P.resident > 0) {                // stage the resident passes' weights once
        for (int slot = 0; slot < P.resident; ++slot) {
            float kw[3][4][4];
            dyadic_load<3>(&P.f[P.pass_first[P.res_pass[slot]]], threadIdx.x, kw);
            const float* flat = &kw[0][0][0];
#pragma unroll
            for (int q = 0; q < 3; ++q) tmem_st16(tmem_w_addr(tmem, slot, q), flat + 16 * q);
        }
        if (P.part_pass >= 0) {                       // factors 0-1 of a third pass: 32 columns
            float kw[3][4][4];
            dyadic_load<3>(&P.f[P.pass_first[P.part_pass]], threadIdx.x, kw);
            const float* flat = &kw[0][0][0];
#pragma unroll
            for (int q = 0; q < 2; ++q) tmem_st16(tmem_part_addr(tmem, q), flat + 16 * q);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const int N = P.N;
    // buffer b at smf + b*R*N: indexing the shared symbol directly (not through an
    // array of pointers) keeps the accesses in the shared window (LDS/STS, not
    // generic LD/ST -- measured: the pointer array made every row access generic)
    // 1024-byte aligned (the SWIZZLE_128B pattern repeats every 1 KB of address)
    float* const smf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm4) + 1023) & ~uintptr_t(1023));
    auto buf = [&](int64_t k) { return smf + (size_t)(k & 1) * R * N; };
    const int64_t ngroups = (B + R - 1) / R;
    const int64_t mine = ngroups > blockIdx.x ? (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto group_rows = [&](int64_t k) {
        const int64_t row0 = ((int64_t)blockIdx.x + k * gridDim.x) * R;
        return (int)((B - row0) < R ? (B - row0) : R);
    };
    auto issue_load = [&](int64_t k) {          // thread 0 only
        const int64_t row0 = ((int64_t)blockIdx.x + k * gridDim.x) * R;
        const uint32_t bar = smem_u32(&full[k & 1]);
        if constexpr (SWZ) {                    // R-row box; rows past B arrive zero-filled
            mbar_expect_tx(bar, (uint32_t)R * (uint32_t)N * 4u);
            tma_3d(smem_u32(buf(k)), &xmap, 0, 0, (int)row0, bar);
        } else {
            const uint32_t bytes = (uint32_t)group_rows(k) * (uint32_t)N * 4u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(buf(k))), "l"(X + row0 * N), "r"(bytes), "r"(bar) : "memory");
        }
    };
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (mine > 0) issue_load(0);
    }
    __syncthreads();
    for (int64_t k = 0; k < mine; ++k) {
        // Prefetch of group k+1 into the other buffer, whose previous contents (group
        // k-1) must have left for HBM first: thread 0 waits for that store's reads
        // after the second pass of group k (KS_FUSED_PF_PASS), not before it, so the
        // whole CTA does not idle while the store drains.
        auto prefetch = [&]() {
            if (threadIdx.x == 0 && k + 1 < mine) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue_load(k + 1);
            }
        };
        if (P.pf_pass < 0) prefetch();
        {
            const uint32_t bar = smem_u32(&full[k & 1]);
            const uint32_t par = (uint32_t)((k >> 1) & 1);
            asm volatile(
                "{\n.reg .pred P1;\nLAB_WAIT:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(bar), "r"(par) : "memory");
        }
        float* sm = buf(k);
        const int rows = group_rows(k);
        int f = 0;
        for (int ps = 0; ps < P.npass; ++ps) {
            const int len = P.pass_len[ps];
            const int slot = P.resident > 0 && P.res_pass[0] == ps ? 0 : P.resident > 1 && P.res_pass[1] == ps ? 1 : -1;
            if (BB == 2 && slot >= 0) {              // weights from TMEM
                float kw[3][4][4];
                float* flat = &kw[0][0][0];
#pragma unroll
                for (int q = 0; q < 3; ++q) tmem_ld16f(tmem_w_addr(tmem, slot, q), flat + 16 * q);
                dyadic_apply_any<3, SWZ>(sm, rows, N, P.f[f].d, threadIdx.x, kw);
            } else if (BB == 2 && ps == P.part_pass) {   // factors 0-1 from TMEM, factor 2 from L2
                float kw[3][4][4];
                float* flat = &kw[0][0][0];
#pragma unroll
                for (int q = 0; q < 2; ++q) tmem_ld16f(tmem_part_addr(tmem, q), flat + 16 * q);
                dyadic_load<3, 2>(&P.f[f], threadIdx.x, kw);
                dyadic_apply_any<3, SWZ>(sm, rows, N, P.f[f].d, threadIdx.x, kw);
            } else if (BB == 2 && len == 3) dyadic_pass<3, SWZ>(sm, rows, N, &P.f[f]);
            else if (BB == 2 && len == 2) dyadic_pass<2, SWZ>(sm, rows, N, &P.f[f]);
            else block_pass<BB, SWZ>(sm, rows, N, P.f[f]);
            f += len;
            if (ps == P.pf_pass) prefetch();
            __syncthreads();
        }
        if (bias || P.act) {                        // KSLinear bias / activation after the last factor (NEXT-2)
            for (int e = threadIdx.x; e < rows * N / 4; e += THREADS) {
                float4 q = reinterpret_cast<float4*>(sm)[e];
                if (bias) {
                    // logical column of this (physical) 16-byte chunk: rpos is an involution
                    const float4 bb = __ldg(reinterpret_cast<const float4*>(bias) + rpos<SWZ>(4 * (e % (N / 4))) / 4);
                    q.x += bb.x; q.y += bb.y; q.z += bb.z; q.w += bb.w;
                }
                if (P.act) {
                    q.x = ks_act(q.x, P.act); q.y = ks_act(q.y, P.act);
                    q.z = ks_act(q.z, P.act); q.w = ks_act(q.w, P.act);
                }
                reinterpret_cast<float4*>(sm)[e] = q;
            }
            __syncthreads();
        }
        // generic writes/reads of this buffer before the async-proxy store (and the
        // later refill of the buffer)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t row0 = ((int64_t)blockIdx.x + k * gridDim.x) * R;
            if constexpr (SWZ)                  // rows past B are clipped by the tensor map
                tma_store_3d(&ymap, 0, 0, (int)row0, smem_u32(sm));
            else
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(Y + row0 * N), "r"(smem_u32(sm)), "r"((uint32_t)rows * (uint32_t)N * 4u) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (BB == 2 && P.resident > 0) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        }
    }
}

constexpr int SMEM_BUDGET = 224 * 1024;      // two row-group buffers (double-buffered); 227 KB opt-in max
constexpr int SMEM_ALIGN_PAD = 1024;         // the kernel aligns the buffers to 1 KB

}  // namespace

namespace ks {

// Eligibility: BSF, L <= 32, every factor square with b = c = BB in {2, 4},
// all dimensions equal to N, N % 4 == 0, at least one row fits in shared
// memory, 16-byte aligned X and Y.
bool fused_chain_supports(const ks_handle_t* hs, int L, const KsCall& call) {
    if (call.mixed()) return false;
    if (call.layout != KS_LAYOUT_BSF || L < 2 || L > MAXF) return false;
    const int64_t bb = hs[0]->b;
    if (bb != 2 && bb != 4) return false;
    const int64_t N = hs[0]->N;
    for (int l = 0; l < L; ++l) {
        if (hs[l]->b != bb || hs[l]->c != bb || hs[l]->N != N || hs[l]->M != N) return false;
    }
    if (N % 4 != 0 || 2 * N * 4 > SMEM_BUDGET || N > (int64_t(1) << 24)) return false;
    const uintptr_t al = reinterpret_cast<uintptr_t>(call.X) | reinterpret_cast<uintptr_t>(call.Y);
    return ((al | reinterpret_cast<uintptr_t>(call.bias)) & 15) == 0;
}

bool resident_partial() {                           // KS_FUSED_TMEM_PART=0 disables (experiments)
    static const bool on = [] {
        const char* e = getenv("KS_FUSED_TMEM_PART");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

cudaError_t fused_chain_launch(const ks_handle_t* hs, int L, const KsCall& call) {
    FusedParams P{};
    const int64_t N = hs[0]->N;
    P.N = (int)N;
    P.act = call.act;
    // application order: K_L first (handles[L-1])
    for (int t = 0; t < L; ++t) {
        const ks_handle_s& h = *hs[L - 1 - t];
        P.f[t] = FusedFactor{h.k_canon, (int)h.a, (int)h.d};
    }
    // group dyadic runs (b = c = 2, d doubling, a halving) into passes of <= 3
    int t = 0;
    P.npass = 0;
    const bool dyadic = hs[0]->b == 2;
    static const int max_len = [] {           // KS_FUSED_RADIX (experiments): 2, 4 or 8
        const char* e = getenv("KS_FUSED_RADIX");
        const int r = e ? atoi(e) : 8;
        return r >= 8 ? 3 : r >= 4 ? 2 : 1;
    }();
    while (t < L) {
        int len = 1;
        if (dyadic) {
            while (len < max_len && t + len < L && P.f[t + len].d == 2 * P.f[t + len - 1].d &&
                   2 * P.f[t + len].a == P.f[t + len - 1].a)
                ++len;
        }
        P.pass_first[P.npass] = t;
        P.pass_len[P.npass++] = len;
        t += len;
    }
    // TMEM-resident weights for up to two leading radix-8 passes: one item per thread
    static const int resident_max = [] {            // KS_FUSED_TMEM (experiments): 0..2
        const char* e = getenv("KS_FUSED_TMEM");
        const int v = e ? atoi(e) : 2;
        return v < 0 ? 0 : v > 2 ? 2 : v;
    }();
    P.resident = 0;
    P.part_pass = -1;
    if (dyadic && N / 8 == THREADS) {
        // the d0 = 1 pass first: its per-thread float4 weight loads are 64 B apart
        // (half of every sector wasted), the d0 > 1 passes' loads are coalesced --
        // measured: TMEM for passes {0, 1} 129 us, for {3, 2} 156 us, none 172 us
        for (int pass_d1 = 0; pass_d1 < 2; ++pass_d1)
            for (int ps = 0; ps < P.npass && P.resident < resident_max; ++ps) {
                const bool d1 = P.f[P.pass_first[ps]].d == 1;
                if (P.pass_len[ps] == 3 && d1 == (pass_d1 == 0)) P.res_pass[P.resident++] = ps;
            }
        if (P.resident == 2 && resident_max >= 2 && resident_partial())
            for (int ps = 0; ps < P.npass; ++ps)
                if (P.pass_len[ps] == 3 && ps != P.res_pass[0] && ps != P.res_pass[1]) {
                    P.part_pass = ps;
                    break;
                }
    }
    int64_t R = SMEM_BUDGET / (2 * N * 4);                      // rows per buffer
    if (R > 16) R = 16;
    const int64_t sms = num_sms(hs[0]->device);
    // enough row groups to fill the machine
    while (R > 1 && (call.B + R - 1) / R < sms) R /= 2;
    const size_t smem = (size_t)2 * R * N * 4 + SMEM_ALIGN_PAD;
    int64_t groups = (call.B + R - 1) / R;
    const int64_t grid = groups < sms ? groups : sms;             // persistent, one CTA per SM
    // bank-conflict-free swizzled rows: whole 1 KB swizzle periods per row, box dims <= 256
    static const bool swz_on = [] {                 // KS_FUSED_SWZ=0 disables (experiments)
        const char* e = getenv("KS_FUSED_SWZ");
        return !(e && atoi(e) == 0);
    }();
    CUtensorMap xmap{}, ymap{};
    bool swz = swz_on && N % 256 == 0 && N / 32 <= 256 && call.B < (int64_t(1) << 31);
    if (swz) {
        const cuuint64_t dims[3] = {32, (cuuint64_t)(N / 32), (cuuint64_t)call.B};
        const cuuint64_t strides[2] = {128, (cuuint64_t)N * 4};
        const cuuint32_t box[3] = {32, (cuuint32_t)(N / 32), (cuuint32_t)R};
        swz = encode(&xmap, call.X, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B) &&
              encode(&ymap, call.Y, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    static const int pf_pass = [] {                 // KS_FUSED_PF_PASS (experiments): -1 = before pass 0
        const char* e = getenv("KS_FUSED_PF_PASS");
        return e ? atoi(e) : 1;     // measured (N = 4096, L = 12): -1 111.7 us, 0 / 1 107.5, 2 115.6
    }();
    P.pf_pass = pf_pass < P.npass ? pf_pass : P.npass - 1;
    cudaError_t e;
    auto kern = hs[0]->b == 2 ? (swz ? ks_chain_fused_kernel<2, true> : ks_chain_fused_kernel<2, false>)
                              : (swz ? ks_chain_fused_kernel<4, true> : ks_chain_fused_kernel<4, false>);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kern, dim3((unsigned)grid), dim3(THREADS), smem, call.stream, call.X, call.Y, call.bias, call.B, P,
                   (int)R, xmap, ymap);
    count_launch();
    return e;
}

}  // namespace ks
