/*
 * ks.h -- C ABI of the B200-native Kronecker-sparse (KS) matmul library
 *         (libks.so, built from paper_2405_15013_b200/csrc/).
 *
 * The operation (§1 "Scope of This Work"):
 *
 *     Y = X K^T,    K in R^{M x N},  M = a b d,  N = a c d,
 *
 * where K is (a,b,c,d)-Kronecker-sparse: supp(K) is contained in
 * I_a (x) 1_{b x c} (x) I_d  (Def. 1).  K is fixed and may be
 * preprocessed offline (ks_pack_weights); X and Y are dense and keep the
 * caller's layout, batch-size-first or batch-size-last
 * (§2.2).  Chains K_1 ... K_L (Table 3,
 * PAPER.md:936-962) are applied as Y = X K_L^T ... K_1^T.
 *
 * Conventions shared by every entry point
 *  - Element type: IEEE float32 for X, K, Y.  Arithmetic is FP32 FFMA on
 *    CUDA cores (KS_MATH_FP32, default) or TF32 tensor cores with FP32
 *    accumulation (KS_MATH_TF32; only where b,c >= 16), or FP32 accuracy on
 *    the tensor cores through the 3xTF32 split x k ~ x_lo k_hi + x_hi k_lo +
 *    x_hi k_hi (KS_MATH_F32X3; b,c >= 16; not in the paper -- see DESIGN.md).
 *  - Indexing is 64-bit throughout.  B = 0 is a no-op returning KS_OK.
 *  - Pointers named X / Y below are CUDA DEVICE pointers (e.g. a torch
 *    tensor's data_ptr()) on the device the handle was packed on, contiguous,
 *    at least 4-byte aligned (16-byte alignment enables the vector paths).
 *    X and Y must not overlap.  Y is fully overwritten (every element written
 *    exactly once; PAPER.md:354-374 row sets partition [0, M)).
 *  - Streams: ks_stream_t is a cudaStream_t passed as void*; NULL is the
 *    legacy default stream.  Calls are asynchronous w.r.t. the host unless
 *    stated; launch errors are reported by the return value, asynchronous
 *    device faults surface at the caller's next synchronisation.
 *  - Errors: every call returns a ks_status_t and never aborts; the status
 *    and a message are also kept per host thread (ks_last_error*).
 *  - Threading: handles are immutable after ks_pack_weights (ks_set_math /
 *    ks_set_kernel excepted: do not call them concurrently with a matmul on
 *    the same handle); concurrent ks_matmul / ks_chain calls on different
 *    streams are safe.
 */
#ifndef KS_H_
#define KS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_ABI_VERSION 1

typedef struct ks_handle_s* ks_handle_t;   /* opaque packed factor           */
typedef void* ks_stream_t;                 /* cudaStream_t                    */

/* Batch layouts.
 *  BSF: X is B x N row-major, X(n,s) = X[n*N + s];  Y(n,r) = Y[n*M + r].
 *  BSL: X is N x B row-major, X(n,s) = X[s*B + n];  Y(n,r) = Y[r*B + n].      */
typedef enum { KS_LAYOUT_BSF = 0, KS_LAYOUT_BSL = 1 } ks_layout_t;

/* Arithmetic.  TF32: operands rounded to TF32 (K: round-to-nearest-away at
 * pack time; X: per kernel), products accumulated in FP32. */
typedef enum { KS_MATH_FP32 = 0, KS_MATH_TF32 = 1, KS_MATH_F32X3 = 2 } ks_math_t;

/* Storage / operand type of a handle and of the X, Y, bias it is used with.
 * F32 handles follow ks_math_t.  BF16 / F16 handles (the
 * paper's FP16 study PAPER.md:1597-1696) multiply on tcgen05 tensor cores
 * (kind::f16) with FP32 accumulation and round the output to nearest-even;
 * patterns the tensor-core kernel cannot take run a generic half kernel with
 * FP32 accumulation.                                                         */
typedef enum { KS_DTYPE_F32 = 0, KS_DTYPE_BF16 = 1, KS_DTYPE_F16 = 2 } ks_dtype_t;

/* Epilogue activation of ks_matmul_act / ks_chain_act (the
 * "+ GELU" of the FFN row): applied in FP32 to each output after
 * the bias, in the epilogue of the last factor applied (K_1).  GELU is the exact
 * form 0.5 y (1 + erf(y / sqrt 2)) (erff).                                   */
typedef enum { KS_ACT_NONE = 0, KS_ACT_GELU = 1 } ks_activation_t;

/* Kernel families; KS_KERNEL_AUTO lets the plan table choose (default).    */
typedef enum {
    KS_KERNEL_AUTO = 0,
    KS_KERNEL_GENERIC = 1,  /* one thread per output element, any pattern   */
    KS_KERNEL_STREAM = 2,   /* vectorised streaming kernel, b,c in {1,2,4}  */
    KS_KERNEL_FFMA = 3,     /* register-tiled FP32 kernel, larger b,c       */
    KS_KERNEL_TF32 = 4,     /* tcgen05 TF32 tensor-core kernel              */
    KS_KERNEL_FUSED_CHAIN = 5, /* whole chain in one launch (trace records only) */
    KS_KERNEL_SPLITC = 6       /* small B (<= 64): lanes split c, warp-shuffle
                                  butterfly reduction           */
} ks_kernel_t;

typedef enum {
    KS_OK = 0,
    KS_ERR_INVALID_ARG = 1,  /* null pointer, negative size, overlap, bad enum */
    KS_ERR_PATTERN = 2,      /* a,b,c,d < 1 or sizes overflow 64-bit           */
    KS_ERR_CHAIN_SHAPE = 3,  /* a_l c_l d_l != a_{l+1} b_{l+1} d_{l+1}         */
    KS_ERR_UNSUPPORTED = 4,  /* requested kernel/math cannot run this pattern  */
    KS_ERR_DEVICE = 5,       /* no CUDA device / wrong current device / not sm_100 */
    KS_ERR_ALIGNMENT = 6,    /* pointer not 4-byte aligned                     */
    KS_ERR_OOM = 7,          /* device or pinned allocation failed             */
    KS_ERR_CUDA = 8          /* any other CUDA runtime error (see message)     */
} ks_status_t;

/* ---------------------------------------------------------------------------
 * ks_pack_weights -- offline preprocessing of one KS factor (PAPER.md:434-436:
 * "preprocessed and stored so that every tile K^T[col_ij, row_ij] is already
 * contiguous"; excluded from timing).
 *   a,b,c,d : the pattern (Def. 1), each >= 1.
 *   K       : a*b*c*d floats in canonical order (a,b,c,d), d fastest
 *             (einsum packing): K[((i*b+k)*c+l)*d+j] is
 *             the entry at row i*b*d + k*d + j, column i*c*d + l*d + j.
 *             Host or device memory (copied through UVA).  Not retained.
 * Synchronous.  The handle owns device copies of K in every layout the
 * kernels read (canonical, tile-contiguous K^T, TF32 operand tiles) on the
 * device current at call time.  Returns NULL on error (see ks_last_error).
 * ------------------------------------------------------------------------- */
ks_handle_t ks_pack_weights(int64_t a, int64_t b, int64_t c, int64_t d, const float* K);

/* Same with an explicit element type: K holds a*b*c*d values of `dtype`
 * (host or device).  A handle's dtype is fixed; use it with ks_matmul_any /
 * ks_chain_any (ks_matmul / ks_chain / ks_chain_ex / ks_*_bias accept only
 * F32 handles and return KS_ERR_INVALID_ARG otherwise).                     */
ks_handle_t ks_pack_weights_ex(int64_t a, int64_t b, int64_t c, int64_t d, const void* K,
                               ks_dtype_t dtype);
ks_status_t ks_get_dtype(ks_handle_t h, ks_dtype_t* out);

/* Release a handle (NULL is ignored).  Synchronises the handle's device. */
void ks_free(ks_handle_t h);

/* Pattern of a handle: out[0..3] = a,b,c,d.                               */
ks_status_t ks_get_pattern(ks_handle_t h, int64_t out[4]);

/* Select the arithmetic.  KS_MATH_TF32 and KS_MATH_F32X3 need b >= 16 and
 * c >= 16 (north star: tensor cores only where each block is a dense
 * contraction); otherwise KS_ERR_UNSUPPORTED and the math is unchanged.
 * KS_MATH_F32X3 allocates and packs the low halves rna_tf32(K - rna_tf32(K)) on the
 * handle's device the first time (synchronous).  Calls the F32X3 tensor-core
 * kernels cannot take (BSF with d > 4 and d % 4 != 0, c % 16 != 0) run the
 * FP32 CUDA-core kernels.                                                  */
ks_status_t ks_set_math(ks_handle_t h, ks_math_t m);

/* Force a kernel family (tests / benchmarks).  KS_KERNEL_AUTO restores the
 * plan table.  A forced family that cannot run a given call makes that call
 * return KS_ERR_UNSUPPORTED (no silent fallback).                          */
ks_status_t ks_set_kernel(ks_handle_t h, ks_kernel_t k);

/* The kernel family ks_matmul would launch for (B, layout) on this handle. */
ks_status_t ks_plan(ks_handle_t h, int64_t B, ks_layout_t layout, ks_kernel_t* out);

/* Launch-plan knobs (the paper's per-pattern "presets",
 * PAPER.md:735, auto-tuned per pattern and GPU).  Every
 * kernel family exposes its measured design alternatives as one bit each; the
 * library takes them, per call, from a compiled-in table generated by an
 * offline B200 autotune over the configs[2] sweep and configs[3]/[4] factors
 * (key: a, b, c, d, layout, math, floor(log2 B)), else from its rules.  No knob
 * changes the result beyond FP rounding order (FP32 kernels: bit-identical).  */
typedef enum {
    KS_KNOB_TF32_V2 = 1 << 0,    /* TF32 BSL / BSF d=1: resident-weight, TMA-store kernel  */
    KS_KNOB_V2_NKB2 = 1 << 1,    /*   ... with double-buffered weight segments             */
    KS_KNOB_DENSIFY = 1 << 2,    /* TF32 BSF 2<=d<=8: super-blocks as dense (bd x cd)       */
    KS_KNOB_J8 = 1 << 3,         /* TF32 BSF J-gather: 32-byte runs also for b > 64        */
    KS_KNOB_BN256 = 1 << 4,      /* TF32 BSF J=2: 256-wide output tiles                    */
    KS_KNOB_KB32 = 1 << 5,       /* FFMA TMA ring: 32 l per chunk for b = 96 tiles          */
    KS_KNOB_FFMA_WS = 1 << 6,    /* FFMA: warp-specialised TMA-fed kernels                 */
    KS_KNOB_FFMA_WSG = 1 << 7,   /* FFMA BSF d>1: four-j / all-j TMA kernels               */
    KS_KNOB_TF32_MN = 1 << 8,    /* TF32 BSL in: A MN-major by TMA (no transposer warps)   */
    KS_KNOB_FFMA_WSL = 1 << 9    /* FFMA BSF d%4==0: one j per lane, FFMA2 (else four-j)   */
} ks_knob_t;

/* Force the knobs of every call on this handle (autotuning, A/B tests): a
 * mask of KS_KNOB_* bits, or -1 to return to the preset table / rules.
 * KS_ERR_INVALID_ARG for anything else.  Not thread-safe against concurrent
 * calls on the same handle. */
ks_status_t ks_set_knobs(ks_handle_t h, int64_t knobs);

/* The knobs a call with (B, layout) would use, and where they come from:
 * *source = 0 rules, 1 preset table, 2 ks_set_knobs override (may be NULL). */
ks_status_t ks_plan_knobs(ks_handle_t h, int64_t B, ks_layout_t layout, uint32_t* knobs, int* source);

/* Number of entries in the compiled preset table. */
int         ks_preset_count(void);

/* ---------------------------------------------------------------------------
 * ks_matmul -- Y = X K^T for one factor: ONE fused kernel launch on `stream`,
 * no permutation passes (Alg. 2/3).
 *   X : device, B*N floats in `layout`;  Y : device, B*M floats in `layout`.
 * ------------------------------------------------------------------------- */
ks_status_t ks_matmul(ks_handle_t h, const float* X, float* Y, int64_t B,
                      ks_layout_t layout, ks_stream_t stream);

/* ---------------------------------------------------------------------------
 * ks_chain -- Y = X K_L^T ... K_1^T (PAPER.md:53-54 with the Y = X K^T form of
 * PAPER.md:86), batch-size-first.  handles[0] = K_1, ..., handles[L-1] = K_L
 * (paper order); K_L is applied first.  Requires N(K_l) == M(K_{l+1}), i.e.
 * a_l c_l d_l == a_{l+1} b_{l+1} d_{l+1} (Table 3), else
 * KS_ERR_CHAIN_SHAPE.  X: B*N(K_L) floats, Y: B*M(K_1) floats, device.
 * Intermediates live in a stream-ordered workspace owned by the library
 * (allocated and freed on `stream`).  L launches.
 * ------------------------------------------------------------------------- */
ks_status_t ks_chain(const ks_handle_t* handles, int L, const float* X, float* Y,
                     int64_t B, ks_stream_t stream);

/* Same as ks_chain with an explicit layout for X, Y and the intermediates. */
ks_status_t ks_chain_ex(const ks_handle_t* handles, int L, const float* X, float* Y,
                        int64_t B, ks_layout_t layout, ks_stream_t stream);

/* ---------------------------------------------------------------------------
 * KSLinear bias (the "+bias" rows of Table 7, PAPER.md:1563;
 * S:406-415): the same operations with Y += 1 * bias^T fused into the epilogue of
 * the last factor applied (K_1), i.e. Y(n, r) = (X K_L^T ... K_1^T)(n, r) + bias[r].
 *   bias : device, M(K_1) floats, 4-byte aligned (16-byte alignment keeps the
 *          vector paths), or NULL for no bias (then identical to ks_matmul /
 *          ks_chain_ex).  The bias is added after the FP32 reduction.
 * ------------------------------------------------------------------------- */
ks_status_t ks_matmul_bias(ks_handle_t h, const float* X, float* Y, const float* bias,
                           int64_t B, ks_layout_t layout, ks_stream_t stream);
ks_status_t ks_chain_bias(const ks_handle_t* handles, int L, const float* X, float* Y,
                          const float* bias, int64_t B, ks_layout_t layout, ks_stream_t stream);

/* Type-generic forms: X, Y, bias (may be NULL) are device arrays of the
 * handles' dtype (all handles of a chain must share it; intermediates use it
 * too).  Semantics otherwise as ks_matmul_bias / ks_chain_bias.             */
ks_status_t ks_matmul_any(ks_handle_t h, const void* X, void* Y, const void* bias, int64_t B,
                          ks_layout_t layout, ks_stream_t stream);
ks_status_t ks_chain_any(const ks_handle_t* handles, int L, const void* X, void* Y,
                         const void* bias, int64_t B, ks_layout_t layout, ks_stream_t stream);

/* Same as ks_matmul_any / ks_chain_any with an epilogue activation applied to
 * every output after the bias (NEXT-2; FFN "2 x Linear + GELU"):
 * Y = act(X K^T + bias), for a chain act(X K_L^T ... K_1^T + bias), fused into
 * the epilogue of the last factor applied (K_1) in every kernel family (and of
 * the fused chain kernel).  act: KS_ACT_NONE or KS_ACT_GELU (exact erf form,
 * FP32 erff), else KS_ERR_INVALID_ARG.  Half handles: applied in FP32 before
 * the output is rounded.                                                     */
ks_status_t ks_matmul_act(ks_handle_t h, const void* X, void* Y, const void* bias, ks_activation_t act,
                          int64_t B, ks_layout_t layout, ks_stream_t stream);
ks_status_t ks_chain_act(const ks_handle_t* handles, int L, const void* X, void* Y, const void* bias,
                         ks_activation_t act, int64_t B, ks_layout_t layout, ks_stream_t stream);

/* ---------------------------------------------------------------------------
 * Chain fusion policy (process-wide, default on).  When on, ks_chain /
 * ks_chain_ex / ks_chain_host run an eligible chain -- BSF, 2 <= L <= 32,
 * every factor square with b = c in {2, 4} (e.g. the FFT / square dyadic
 * butterfly) and FP32 math -- as ONE kernel that keeps R batch rows
 * in shared memory across all factors: X is read and Y
 * written once instead of one HBM round trip per factor.  The result is
 * bit-identical to the per-factor launches.  Off: one launch per factor.
 * ks_chain_fusion_eligible reports whether a call would fuse (1) or not (0).
 * ------------------------------------------------------------------------- */
ks_status_t ks_set_chain_fusion(int enable);
int ks_chain_fusion_eligible(const ks_handle_t* handles, int L, int64_t B, ks_layout_t layout);

/* ---------------------------------------------------------------------------
 * Mixed layouts.  The paper fixes one layout per call (BSF: X is B x N
 * row-major; BSL: X^T, N x B, the layout its kernel favours,
 * PAPER.md:631-641 "batch-size-last").  Inside a chain the intermediates are
 * the library's own buffers, so their layout is free.
 *
 * ks_matmul_io -- Y = X K^T with X in x_layout and Y in y_layout (X: device,
 *   B*N floats; Y: device, B*M floats; 4-byte aligned, no overlap).  FP32
 *   handles only.  x_layout == y_layout is ks_matmul.  Mixed pairs run the
 *   TF32 tensor-core kernel (math KS_MATH_TF32: BSF in / BSL out for any
 *   pattern it supports in BSF; BSL in / BSF out for d = 1 and d in
 *   {2,3,4,6,8} or d % 4 == 0, B % 4 == 0, Y 16-byte aligned), else the
 *   generic kernel (FP32, any pattern).  Errors as ks_matmul.
 *
 * ks_set_chain_mixed_layouts -- process-wide policy (default on): a BSF chain
 *   of TF32 factors keeps each intermediate next to a factor with d > 8 in
 *   BSL, so that factor's d-strided BSF gather or store is
 *   replaced by unit-stride batch runs; used only when every call of the chain
 *   then runs the TF32 kernel.  X and Y keep the caller's layout; results
 *   are those of the per-factor calls in the chosen layouts.
 * ks_chain_layouts -- the plan a ks_chain_ex call would use: out[t] = layout
 *   of the output of handles[t] (out[0] = Y's, the caller's), out[L] = X's
 *   (L+1 ints); handles[t] reads out[t+1] and writes out[t].
 *   Returns 1 if any intermediate is mixed, 0 if uniform, -1 on bad arguments.
 * ------------------------------------------------------------------------- */
ks_status_t ks_matmul_io(ks_handle_t h, const float* X, ks_layout_t x_layout, float* Y, ks_layout_t y_layout,
                         int64_t B, ks_stream_t stream);
ks_status_t ks_set_chain_mixed_layouts(int enable);
int ks_chain_layouts(const ks_handle_t* handles, int L, int64_t B, ks_layout_t layout, int* out);

/* ---------------------------------------------------------------------------
 * ks_chain_host -- end-to-end form of ks_chain_ex for HOST buffers: X_host and
 * Y_host are host memory (pinned for full PCIe speed and copy/compute
 * overlap; pageable works but the copies then serialise).  The batch is cut
 * into chunks of ~16 MB of X + Y (at most 16) and pipelined over three
 * library-internal streams: the host->device copy of chunk k+1 and the
 * device->host copy of chunk k-1 overlap the chain on chunk k.  Ordered after
 * prior work on `stream`, and later work on `stream` waits for all of it;
 * device buffers come from the library's stream-ordered pool.  Asynchronous:
 * Y_host is valid after the caller synchronises `stream`.  Each row equals
 * ks_chain_ex's result bit for bit whenever the chunks run the same kernel
 * families as the whole batch (always under KS_MATH_FP32, whose kernels are
 * bit-identical; a ragged BSL chunk may move a TF32 call to FP32 FFMA).  A
 * single factor is L = 1.
 * ------------------------------------------------------------------------- */
ks_status_t ks_chain_host(const ks_handle_t* handles, int L, const float* X_host,
                          float* Y_host, int64_t B, ks_layout_t layout, ks_stream_t stream);

/* ---------------------------------------------------------------------------
 * CUDA-graph form of a chain ("optional CUDA-graph
 * capture"): ks_chain_graph records exactly the launches ks_chain_any would
 * make for (handles, L, X, Y, bias, B, layout) -- per-factor kernels with
 * their programmatic-dependent-launch edges, or the one fused-chain kernel --
 * into an executable CUDA graph; ks_graph_launch replays it on `stream` with a
 * single cudaGraphLaunch (no per-launch host work).
 *   X, Y, bias, B, layout: baked into the graph (same meaning, layout and
 *            alignment rules as ks_chain_any); the caller keeps them alive and
 *            may change their CONTENTS between launches.
 *   handles: must outlive the graph; their math / kernel / fusion settings are
 *            those at capture time.
 * The graph owns its intermediate workspace (2 x B x max(M_l) elements,
 * allocated at capture, freed by ks_graph_free).  ks_chain_graph is
 * synchronous; returns NULL on error (see ks_last_error).  Replays are ordered
 * on `stream` like any kernel launch; concurrent replays of ONE graph on
 * different streams are not allowed (they share the workspace).            */
typedef struct ks_graph_s* ks_graph_t;
ks_graph_t  ks_chain_graph(const ks_handle_t* handles, int L, const void* X, void* Y, const void* bias,
                           int64_t B, ks_layout_t layout);
ks_status_t ks_graph_launch(ks_graph_t g, ks_stream_t stream);
int         ks_graph_kernel_count(ks_graph_t g);          /* kernels one replay launches; -1 on NULL */
void        ks_graph_free(ks_graph_t g);                   /* NULL is ignored; synchronises */

/* Copy one packed variant of K back to host (tests check the index maps
 * bit-exactly).  variant 0: canonical a*b*c*d;  1: tile-contiguous K^T,
 * [i*d+j][l][k] (a*d*c*b floats);  2: TF32-rounded tiles [i*d+j][k][l]
 * (a*d*b*c floats);  3: the F32X3 low halves rna_tf32(K - rna_tf32(K)), same order
 * as 2 (only after ks_set_math(h, KS_MATH_F32X3));  4: the densified TF32
 * super-blocks [i][k*d+j][l*d+j'] = rna_tf32(K4[i][k][l][j]) if j == j' else 0,
 * a*(b*d)*(c*d) floats (only after ks_set_math(h, KS_MATH_TF32) with
 * 2 <= d <= 8: the BSF tensor-core path may contract a super-block as one dense
 * (bd x cd) block, Def. 1).  count must equal the
 * variant's element count.  Half
 * handles copy elements of their dtype (2 bytes each): variant 0 canonical,
 * 2 tensor-core tiles [i*d+j][k][l] (unrounded); variant 1 does not exist.  */
ks_status_t ks_read_packed(ks_handle_t h, int variant, float* dst_host, int64_t count);

/* ---------------------------------------------------------------------------
 * Launch tracing (profiling aid, off by default).  While enabled, every
 * kernel launch the library makes is bracketed by a pair of CUDA events
 * recorded on the launch stream, together with its kernel family and its
 * algorithmic bytes 4*(B*N + a*b*c*d + B*M) (the paper's byte model, read X +
 * nnz(K) + write Y).  ks_trace_enable(1) clears the buffer.
 * ks_trace_read synchronises on the recorded events and copies up to `max`
 * records (oldest first) into the caller's host arrays (any may be NULL),
 * stores the number available in *count, then clears the buffer.           */
ks_status_t ks_trace_enable(int on);
ks_status_t ks_trace_read(int64_t max, int64_t* count, float* ms, int* family,
                          double* model_bytes);

/* Diagnostics. */
ks_status_t ks_last_error(void);                /* per host thread           */
const char* ks_last_error_message(void);        /* per host thread, static   */
const char* ks_status_string(ks_status_t s);
uint64_t    ks_kernel_launch_count(void);       /* kernels launched so far   */
int         ks_abi_version(void);               /* KS_ABI_VERSION            */

/* Measurement aid (not on the KS path): the FP32 FFMA throughput of the
 * current device, measured by an FFMA-loop kernel (8 independent chains per
 * thread, 2 x 512 threads per SM, best of 5 event-timed launches on `stream`;
 * synchronous).  The "alu" roofline denominator of the FP32 CUDA-core kernels
 * (SURVEY.md §8d "Peaks": "an FFMA loop for FP32").  *tflops receives TFLOP/s
 * (2 flops per FMA).  KS_ERR_INVALID_ARG if tflops is NULL; KS_ERR_CUDA /
 * KS_ERR_OOM on CUDA failures. */
ks_status_t ks_peak_ffma(ks_stream_t stream, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* KS_H_ */
