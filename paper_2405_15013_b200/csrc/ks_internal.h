// Internal interfaces between the host runtime (ks_runtime.cpp) and the
// kernel translation units.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ks.h"

struct ks_handle_s {
    int64_t a, b, c, d;   // pattern (Def. 1)
    int64_t M, N, nnz;    // abd, acd, abcd
    int device;
    float* k_canon;       // [a][b][c][d]            (boundary order)
    float* k_tile;        // [i*d+j][l][k]  = K^T tiles
    float* k_tf32;        // [i*d+j][k][l]  TF32-rounded, K-major B operand
    float* k_lo;          // [i*d+j][k][l]  rna_tf32(K - k_tf32) (3xTF32 low part), from ks_set_math(F32X3)
    float* k_dense = nullptr;   // [i][k*d+j][l*d+j'] rna_tf32(K4[i][k][l][j]) if j == j' else 0: the
                                // super-block i of K as a dense (bd x cd) TF32 block, from ks_set_math(TF32)
                                // for 2 <= d <= KS_DENSE_MAX_D (BSF "densified" tensor-core path)
    ks_math_t math;
    ks_kernel_t forced;
    int dtype = KS_DTYPE_F32;   // element type of K, X, Y (half handles: k_canon / k_tf32
                                // hold half values, k_tile is unused)
    int64_t knobs_override = -1;  // ks_set_knobs: launch-plan knobs forced for this handle (-1: plan)
    int esize() const { return dtype == KS_DTYPE_F32 ? 4 : 2; }
};

// Launch-plan knobs: the KS_KNOB_* bits of include/ks.h.  The
// runtime fills KsCall::knobs from the compiled per-pattern preset table
// (ks_presets.inc, generated from an offline B200 autotune,
// scripts/autotune.py), else from the rules (ks::rule_knobs).
struct KsCall {
    const float* X;
    float* Y;
    int64_t B;
    int layout;           // ks_layout_t
    cudaStream_t stream;
    const float* bias = nullptr;   // optional length-M vector added in the epilogue
    uint32_t knobs = 0;            // KsKnob bits (ks::plan_knobs)
    int out_layout = -1;           // layout of Y (ks_matmul_io / chain intermediates); -1: `layout`
    int act = KS_ACT_NONE;         // epilogue activation after the bias (ks_activation_t)
    int ylayout() const { return out_layout < 0 ? layout : out_layout; }
    bool mixed() const { return ylayout() != layout; }
};

namespace ks {

// Process-wide launch counter (ks_kernel_launch_count).
void count_launch();

// ---- packing (ks_pack.cu) --------------------------------------------------
cudaError_t pack_tiles(const ks_handle_s& h, cudaStream_t s);
cudaError_t pack_lo(const ks_handle_s& h, cudaStream_t s);        // fills h.k_lo
cudaError_t pack_dense(const ks_handle_s& h, cudaStream_t s);     // fills h.k_dense
constexpr int64_t KS_DENSE_MAX_D = 8;

// ---- kernel families ---------------------------------------------------------
// Each family exposes `supports` (pure host predicate, no CUDA calls) and
// `launch` (exactly one kernel launch on call.stream).
bool generic_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t generic_launch(const ks_handle_s& h, const KsCall& call);

bool stream_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t stream_launch(const ks_handle_s& h, const KsCall& call);

bool ffma_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t ffma_launch(const ks_handle_s& h, const KsCall& call);
// warp-specialised TMA-fed FFMA kernel (ks_ffma_ws.cu): BSL, and BSF with d = 1;
// ffma_launch routes there when it supports the call
bool ffma_ws_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t ffma_ws_launch(const ks_handle_s& h, const KsCall& call);

// small-batch split-c warp-shuffle kernel (ks_splitc.cu): FP32, B <= KS_SPLITC_MAX_B
constexpr int64_t KS_SPLITC_MAX_B = 64;
bool splitc_supports(const ks_handle_s& h, const KsCall& call);
bool splitc_preferred(const ks_handle_s& h, const KsCall& call);   // the auto plan's rule
cudaError_t splitc_launch(const ks_handle_s& h, const KsCall& call);

bool tf32_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t tf32_launch(const ks_handle_s& h, const KsCall& call);
// round-2 TF32 kernel (ks_tf32_v2.cu): BSL and BSF d = 1, MN-major A by TMA,
// resident weights, TMA-store epilogue; tf32_launch routes there when it applies
bool tf32v2_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t tf32v2_launch(const ks_handle_s& h, const KsCall& call);

// half precision handles (NEXT-3): tcgen05 kind::f16 kernel and a generic one
bool half_supports(const ks_handle_s& h, const KsCall& call);
cudaError_t half_launch(const ks_handle_s& h, const KsCall& call);
bool half_bsl_supports(const ks_handle_s& h, const KsCall& call);      // ks_half_bsl.cu (swap-AB)
cudaError_t half_bsl_launch(const ks_handle_s& h, const KsCall& call);
cudaError_t generic_half_launch(const ks_handle_s& h, const KsCall& call);
cudaError_t pack_half(const ks_handle_s& h, cudaStream_t s);

// Fused multi-factor chain (ks_chain_fused.cu): one launch for a whole chain.
bool fused_chain_supports(const ks_handle_t* hs, int L, const KsCall& call);
cudaError_t fused_chain_launch(const ks_handle_t* hs, int L, const KsCall& call);

int num_sms(int device);

// Launch-plan knobs of a call (ks_presets.cpp): the handle's ks_set_knobs
// override, else the preset table entry for (pattern, layout, math, log2 B),
// else the rules.  *source (optional): 0 rules, 1 preset table, 2 override.
uint32_t plan_knobs(const ks_handle_s& h, const KsCall& call, int* source = nullptr);
uint32_t rule_knobs(const ks_handle_s& h, const KsCall& call);
int preset_count();

}  // namespace ks

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels launched through launch_pdl may be scheduled while the previous
// kernel in the stream drains (its CTAs exit); each such kernel calls
// pdl_wait() before its first global-memory access, which returns once the
// previous grid has completed and its writes are visible.  Only the prologue
// (launch, shared-memory carve-out, barrier init, TMEM alloc) overlaps.
// KS_PDL=0 disables it (experiments).
namespace ks {
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace ks

#ifdef __CUDACC__
// Packed FP32 pairs for FFMA2 (fma.rn.f32x2, sm_100a): two independent
// correctly rounded FMAs per instruction -- each lane is exactly fmaf, so FFMA2
// kernels stay bit-identical to the FFMA ones (measured: 0 mismatches in 1.3e8,
// scripts/probe_ffma2.cu) at the same 74 TF/s peak, with half the issue slots.
// A scalar broadcast operand (f2pack(x, x)) folds into FFMA2's .F32 operand form.
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

// Epilogue activation (NEXT-2): the exact GELU 0.5 y (1 + erf(y / sqrt 2)), FP32.
__device__ __forceinline__ float ks_act(float y, int act) {
    return act == KS_ACT_GELU ? 0.5f * y * (1.f + erff(y * 0.7071067811865476f)) : y;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
