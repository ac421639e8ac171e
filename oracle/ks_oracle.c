/*
 * ks_oracle.c -- CPU ORACLE FOR THE KS MATMUL.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2405_15013_b200/).
 *
 * What it computes is the plain definition, deliberately slow:
 *
 *  O-1  ks_oracle_dense: the masked dense K in FP64.  Def. 1
 *       fixes the support I_a (x) 1_{bxc} (x) I_d; the values come in the
 *       canonical (a,b,c,d) order with d fastest (einsum packing,
 *       PAPER.md:860-869):  K4[i][k][l][j] is the entry of row i*b*d + k*d + j
 *       and column i*c*d + l*d + j  (SURVEY.md §0 "Index form").
 *
 *  O-2  ks_oracle_matmul_dense: Y = X K^T (§1 "Scope") as a
 *       naive triple loop  Y(n,r) = sum_{s=0}^{N-1} X(n,s) * D[r][s]  with s
 *       ascending, accumulated in FP64, over the DENSE matrix (zeros included).
 *       X(n,s) is addressed through the layout: batch-size-first X[n*N+s],
 *       batch-size-last X[s*B+n] (§2.2).  It also returns
 *       the error envelope  A(n,r) = sum_s |X(n,s)| |D[r][s]|.
 *       OpenMP over the (n, r) output elements; each element has one owner
 *       and a fixed summation order, so the result is independent of the
 *       thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KS_ORACLE_OK 0
#define KS_ORACLE_EINVAL 1

/* O-1: materialise the masked dense M x N matrix (row-major), M=abd, N=acd. */
int ks_oracle_dense(int64_t a, int64_t b, int64_t c, int64_t d,
                    const double* K4, double* D)
{
    if (a < 1 || b < 1 || c < 1 || d < 1 || !K4 || !D) return KS_ORACLE_EINVAL;
    const int64_t M = a * b * d, N = a * c * d;
    memset(D, 0, sizeof(double) * (size_t)(M * N));
    for (int64_t i = 0; i < a; ++i)
        for (int64_t k = 0; k < b; ++k)
            for (int64_t l = 0; l < c; ++l)
                for (int64_t j = 0; j < d; ++j) {
                    const int64_t row = i * b * d + k * d + j;
                    const int64_t col = i * c * d + l * d + j;
                    D[row * N + col] = K4[((i * b + k) * c + l) * d + j];
                }
    return KS_ORACLE_OK;
}

/* O-2: naive triple loop over the dense matrix.
 *   X      : input, layout 0 = BSF (B x N), 1 = BSL (N x B)
 *   rows   : which batch rows n to compute (nrows of them); NULL = 0..B-1
 *   Y      : nrows x M, batch-size-first, row t holds batch row rows[t]
 *   absY   : same shape, the envelope sum_s |X||D|; may be NULL
 *   threads: OpenMP threads (<= 0 : runtime default)                        */
int ks_oracle_matmul_dense(int64_t M, int64_t N, const double* D,
                           const double* X, int64_t B, int layout,
                           const int64_t* rows, int64_t nrows,
                           double* Y, double* absY, int threads)
{
    if (M < 1 || N < 1 || B < 0 || !D || !X || !Y) return KS_ORACLE_EINVAL;
    if (layout != 0 && layout != 1) return KS_ORACLE_EINVAL;
    if (!rows) nrows = B;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    int bad = 0;
    for (int64_t t = 0; t < nrows; ++t) {
        const int64_t n = rows ? rows[t] : t;
        if (n < 0 || n >= B) bad = 1;
    }
    if (bad) return KS_ORACLE_EINVAL;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t t = 0; t < nrows; ++t) {
        for (int64_t r = 0; r < M; ++r) {
            const int64_t n = rows ? rows[t] : t;
            double acc = 0.0, env = 0.0;
            for (int64_t s = 0; s < N; ++s) {
                const double x = layout == 0 ? X[n * N + s] : X[s * B + n];
                const double k = D[r * N + s];
                acc += x * k;
                env += fabs(x) * fabs(k);
            }
            Y[t * M + r] = acc;
            if (absY) absY[t * M + r] = env;
        }
    }
    return bad ? KS_ORACLE_EINVAL : KS_ORACLE_OK;
}

int ks_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
