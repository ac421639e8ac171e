// Host runtime behind the C ABI of include/ks.h: validation, handles and
// packing, per-call plan selection, chain orchestration with a stream-ordered
// workspace, error state.  Every compute step runs in the kernels of the
// other translation units; nothing here touches X, K or Y on the host.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ks_internal.h"

namespace {

thread_local ks_status_t t_status = KS_OK;
thread_local char t_msg[512] = "ok";
thread_local bool t_capturing = false;   // inside ks_chain_graph's stream capture: no trace events

std::atomic<uint64_t> g_launches{0};

// ---- launch tracing -----------------------------------------------------------
struct TraceRec {
    cudaEvent_t start, stop;
    int family;
    double bytes;
};
std::mutex g_trace_mu;
std::atomic<bool> g_trace_on{false};
std::vector<TraceRec> g_trace;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t trace_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

ks_status_t fail(ks_status_t s, const char* fmt, ...) {
    t_status = s;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_msg, sizeof(t_msg), fmt, ap);
    va_end(ap);
    return s;
}

ks_status_t ok() {
    t_status = KS_OK;
    std::snprintf(t_msg, sizeof(t_msg), "ok");
    return KS_OK;
}

ks_status_t fail_cuda(cudaError_t e, const char* where) {
    if (e == cudaErrorMemoryAllocation)
        return fail(KS_ERR_OOM, "%s: %s", where, cudaGetErrorString(e));
    return fail(KS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool mul_ok(int64_t x, int64_t y, int64_t* out) {
    return !__builtin_mul_overflow(x, y, out) && *out < (int64_t(1) << 62);
}

// ---- per-device stream-ordered memory pool (chain workspace, host staging) ---
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;

// Per-device internal streams of ks_chain_host's copy / compute pipeline.
struct HostStreams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
};
std::mutex g_hs_mu;
std::vector<HostStreams*> g_hs;

cudaError_t host_streams(int dev, HostStreams** out) {
    std::lock_guard<std::mutex> lk(g_hs_mu);
    if ((int)g_hs.size() <= dev) g_hs.resize(dev + 1, nullptr);
    if (!g_hs[dev]) {
        auto* h = new HostStreams();
        cudaError_t e = cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->comp, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete h;
            return e;
        }
        g_hs[dev] = h;
    }
    *out = g_hs[dev];
    return cudaSuccess;
}

cudaError_t get_pool(int dev, cudaMemPool_t* out) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if ((int)g_pools.size() <= dev) g_pools.resize(dev + 1, nullptr);
    if (!g_pools[dev]) {
        cudaMemPoolProps props;
        std::memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p;
        cudaError_t e = cudaMemPoolCreate(&p, &props);
        if (e != cudaSuccess) return e;
        uint64_t keep = ~uint64_t(0);   // keep freed blocks: steady state is allocation-free
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        g_pools[dev] = p;
    }
    *out = g_pools[dev];
    return cudaSuccess;
}

ks_status_t check_device(const ks_handle_s* h) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail_cuda(e, "cudaGetDevice");
    if (dev != h->device)
        return fail(KS_ERR_DEVICE, "handle packed on device %d but current device is %d",
                    h->device, dev);
    return KS_OK;
}

bool overlap(const void* x, int64_t xbytes, const void* y, int64_t ybytes) {
    auto xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
    return xa < ya + (uintptr_t)ybytes && ya < xa + (uintptr_t)xbytes;
}

ks_kernel_t choose(const ks_handle_s& h, const KsCall& call) {
    if (h.dtype != KS_DTYPE_F32) {           // half handles: tensor cores, else generic
        if (h.forced == KS_KERNEL_GENERIC) return KS_KERNEL_GENERIC;
        const bool tc = ks::half_supports(h, call);
        if (h.forced == KS_KERNEL_TF32) return tc ? KS_KERNEL_TF32 : KS_KERNEL_AUTO;
        if (h.forced != KS_KERNEL_AUTO) return KS_KERNEL_AUTO;
        return tc ? KS_KERNEL_TF32 : KS_KERNEL_GENERIC;
    }
    if (h.forced != KS_KERNEL_AUTO) {
        switch (h.forced) {
            case KS_KERNEL_GENERIC: return ks::generic_supports(h, call) ? KS_KERNEL_GENERIC : KS_KERNEL_AUTO;
            case KS_KERNEL_STREAM:  return ks::stream_supports(h, call) ? KS_KERNEL_STREAM : KS_KERNEL_AUTO;
            case KS_KERNEL_FFMA:    return ks::ffma_supports(h, call) ? KS_KERNEL_FFMA : KS_KERNEL_AUTO;
            case KS_KERNEL_TF32:    return ks::tf32_supports(h, call) ? KS_KERNEL_TF32 : KS_KERNEL_AUTO;
            case KS_KERNEL_SPLITC:  return ks::splitc_supports(h, call) ? KS_KERNEL_SPLITC : KS_KERNEL_AUTO;
            default: return KS_KERNEL_AUTO;
        }
    }
    if ((h.math == KS_MATH_TF32 || h.math == KS_MATH_F32X3) && ks::tf32_supports(h, call)) return KS_KERNEL_TF32;
    if (ks::stream_supports(h, call)) return KS_KERNEL_STREAM;
    if (ks::splitc_preferred(h, call)) return KS_KERNEL_SPLITC;
    if (ks::ffma_supports(h, call)) return KS_KERNEL_FFMA;
    return KS_KERNEL_GENERIC;
}

cudaError_t launch(ks_kernel_t k, const ks_handle_s& h, const KsCall& call) {
    if (h.dtype != KS_DTYPE_F32) {
        if (k == KS_KERNEL_TF32) return ks::half_launch(h, call);
        if (k == KS_KERNEL_GENERIC) return ks::generic_half_launch(h, call);
        return cudaErrorInvalidValue;
    }
    switch (k) {
        case KS_KERNEL_GENERIC: return ks::generic_launch(h, call);
        case KS_KERNEL_STREAM:  return ks::stream_launch(h, call);
        case KS_KERNEL_FFMA:    return ks::ffma_launch(h, call);
        case KS_KERNEL_TF32:    return ks::tf32_launch(h, call);
        case KS_KERNEL_SPLITC:  return ks::splitc_launch(h, call);
        default: return cudaErrorInvalidValue;
    }
}

// One factor, arguments already validated.
ks_status_t run_one(const ks_handle_s& h, const float* X, float* Y, int64_t B, int layout,
                    cudaStream_t s, const float* bias = nullptr, int out_layout = -1, int act = KS_ACT_NONE) {
    KsCall call{X, Y, B, layout, s, bias};
    call.out_layout = out_layout;
    call.act = act;
    call.knobs = ks::plan_knobs(h, call);
    ks_kernel_t k = choose(h, call);
    if (k == KS_KERNEL_AUTO)
        return fail(KS_ERR_UNSUPPORTED, "forced kernel %d cannot run pattern (%lld,%lld,%lld,%lld) "
                    "B=%lld layout=%d->%d", (int)h.forced, (long long)h.a, (long long)h.b,
                    (long long)h.c, (long long)h.d, (long long)B, layout, call.ylayout());
    TraceRec rec{nullptr, nullptr, (int)k, 0.0};
    const bool tracing = g_trace_on.load(std::memory_order_relaxed) && !t_capturing;
    if (tracing) {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        rec.start = trace_event();
        rec.stop = trace_event();
        rec.bytes = h.esize() * ((double)B * (double)h.N + (double)h.nnz + (double)B * (double)h.M);
        cudaEventRecord(rec.start, s);
    }
    cudaError_t e = launch(k, h, call);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (tracing) {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        cudaEventRecord(rec.stop, s);
        g_trace.push_back(rec);
    }
    if (e != cudaSuccess) return fail_cuda(e, "kernel launch");
    return KS_OK;
}

ks_status_t validate_chain(const ks_handle_t* hs, int L, int64_t B, int layout) {
    if (!hs || L < 1) return fail(KS_ERR_INVALID_ARG, "need L >= 1 handles");
    if (B < 0) return fail(KS_ERR_INVALID_ARG, "B must be >= 0");
    if (layout != KS_LAYOUT_BSF && layout != KS_LAYOUT_BSL)
        return fail(KS_ERR_INVALID_ARG, "bad layout %d", layout);
    for (int l = 0; l < L; ++l) {
        if (!hs[l]) return fail(KS_ERR_INVALID_ARG, "handles[%d] is NULL", l);
        ks_status_t s = check_device(hs[l]);
        if (s != KS_OK) return s;
        if (hs[l]->dtype != hs[0]->dtype) return fail(KS_ERR_INVALID_ARG, "handles of a chain must share a dtype");
    }
    for (int l = 0; l + 1 < L; ++l)
        if (hs[l]->N != hs[l + 1]->M)
            return fail(KS_ERR_CHAIN_SHAPE, "factor %d has N=%lld but factor %d has M=%lld "
                        "(need a_l c_l d_l == a_{l+1} b_{l+1} d_{l+1})", l + 1,
                        (long long)hs[l]->N, l + 2, (long long)hs[l + 1]->M);
    int64_t t;
    for (int l = 0; l < L; ++l)
        if (!mul_ok(B, hs[l]->M, &t) || !mul_ok(B, hs[l]->N, &t))
            return fail(KS_ERR_INVALID_ARG, "B * dim overflows");
    return KS_OK;
}

std::atomic<bool> g_fusion{true};
std::atomic<bool> g_mixed{true};

// Mixed-layout intermediates (BSF chains of TF32 factors): an intermediate next
// to a factor with d > 8 is kept batch-size-last, so that factor reads (BSL in:
// each j's operand rows are 512-byte runs, no d-strided gather) or writes
// (BSL out: 128-byte warp stores per output row) it without the BSF d > 1
// penalty of PAPER.md:641.  d > 8 because only there the BSF kernel gathers J < d
// columns per tile (32-byte runs); for d <= 8 (J = d, whole-row runs) measured
// on B200 the uniform plan is as fast or faster (profiles/r02/time_models_m1.jsonl:
// ViT-S chains 8-12% slower mixed, GPT-2 UP 13% faster).  lay[t] = layout of the output of hs[t] (lay[0] = Y's,
// the caller's); lay[L] = X's; so hs[t] reads lay[t + 1] and writes lay[t].
// Applied only when every resulting call runs the TF32 tensor-core family
// (pointers: the 256-byte aligned workspace, X and Y as given); else uniform.
bool plan_chain_layouts(const ks_handle_t* hs, int L, const float* X, float* Y, int64_t B, int layout,
                        int* lay) {
    for (int t = 0; t <= L; ++t) lay[t] = layout;
    if (!g_mixed.load(std::memory_order_relaxed) || layout != KS_LAYOUT_BSF || L < 2) return false;
    bool any = false;
    for (int t = 0; t + 1 < L; ++t)          // output of hs[t + 1] = input of hs[t]
        if (hs[t]->d > 8 || hs[t + 1]->d > 8) {
            lay[t + 1] = KS_LAYOUT_BSL;
            any = true;
        }
    if (!any) return false;
    const float* ws = reinterpret_cast<const float*>(uintptr_t(256));
    for (int t = 0; t < L; ++t) {
        const ks_handle_s& h = *hs[t];
        if (h.forced != KS_KERNEL_AUTO || h.math != KS_MATH_TF32 || h.dtype != KS_DTYPE_F32) break;
        KsCall call{t == L - 1 ? X : ws, t == 0 ? Y : const_cast<float*>(ws), B, lay[t + 1], nullptr};
        call.out_layout = lay[t];
        call.knobs = ks::plan_knobs(h, call);
        if (choose(h, call) != KS_KERNEL_TF32) break;
        if (t == L - 1) return true;
    }
    for (int t = 0; t <= L; ++t) lay[t] = layout;
    return false;
}

bool fusion_ok(const ks_handle_t* hs, int L, const KsCall& call) {
    if (!g_fusion.load(std::memory_order_relaxed) || L < 2) return false;
    for (int l = 0; l < L; ++l)
        if (hs[l]->forced != KS_KERNEL_AUTO || hs[l]->math != KS_MATH_FP32 || hs[l]->dtype != KS_DTYPE_F32)
            return false;
    return ks::fused_chain_supports(hs, L, call);
}

// Whole chain in one launch (validated arguments, fusion_ok true).
ks_status_t run_fused(const ks_handle_t* hs, int L, const KsCall& call) {
    TraceRec rec{nullptr, nullptr, (int)KS_KERNEL_FUSED_CHAIN, 0.0};
    const bool tracing = g_trace_on.load(std::memory_order_relaxed) && !t_capturing;
    if (tracing) {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        rec.start = trace_event();
        rec.stop = trace_event();
        double nnz = 0;
        for (int l = 0; l < L; ++l) nnz += (double)hs[l]->nnz;
        rec.bytes = 4.0 * ((double)call.B * (double)hs[L - 1]->N + nnz + (double)call.B * (double)hs[0]->M);
        cudaEventRecord(rec.start, call.stream);
    }
    cudaError_t e = ks::fused_chain_launch(hs, L, call);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (tracing) {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        cudaEventRecord(rec.stop, call.stream);
        g_trace.push_back(rec);
    }
    if (e != cudaSuccess) return fail_cuda(e, "fused chain launch");
    return KS_OK;
}

// Workspace a per-factor chain needs: nbuf buffers of `bytes` each.
void chain_workspace(const ks_handle_t* hs, int L, int64_t B, size_t* bytes, int* nbuf) {
    int64_t maxdim = 0;
    for (int l = 1; l < L; ++l) maxdim = hs[l]->M > maxdim ? hs[l]->M : maxdim;
    *bytes = (size_t)hs[0]->esize() * (size_t)(B * maxdim);
    *nbuf = L >= 3 ? 2 : (L == 2 ? 1 : 0);
}

// Chain on device buffers; X, Y validated by the caller.  `ws` (optional):
// caller-owned intermediate buffers (ks_chain_graph), else stream-ordered
// allocations from the device pool.
ks_status_t run_chain(const ks_handle_t* hs, int L, const float* X, float* Y, int64_t B,
                      int layout, cudaStream_t s, const float* bias = nullptr, void* const* ws = nullptr,
                      int act = KS_ACT_NONE) {
    if (L == 1) return run_one(*hs[0], X, Y, B, layout, s, bias, -1, act);
    {
        KsCall call{X, Y, B, layout, s, bias};
        call.act = act;
        if (fusion_ok(hs, L, call)) return run_fused(hs, L, call);
    }
    size_t bytes;
    int nbuf;
    chain_workspace(hs, L, B, &bytes, &nbuf);
    void* buf[2] = {nullptr, nullptr};
    if (ws) {
        for (int i = 0; i < nbuf; ++i) buf[i] = ws[i];
    } else {
        cudaMemPool_t pool;
        cudaError_t e = get_pool(hs[0]->device, &pool);
        if (e != cudaSuccess) return fail_cuda(e, "cudaMemPoolCreate");
        for (int i = 0; i < nbuf; ++i) {
            e = cudaMallocFromPoolAsync(&buf[i], bytes, pool, s);
            if (e != cudaSuccess) {
                for (int k = 0; k < i; ++k) cudaFreeAsync(buf[k], s);
                return fail_cuda(e, "chain workspace");
            }
        }
    }
    ks_status_t st = KS_OK;
    std::vector<int> lay(L + 1);
    plan_chain_layouts(hs, L, X, Y, B, layout, lay.data());
    const float* in = X;
    for (int l = L - 1; l >= 0 && st == KS_OK; --l) {
        float* out = (l == 0) ? Y : static_cast<float*>(buf[(L - 1 - l) % nbuf]);
        st = run_one(*hs[l], in, out, B, lay[l + 1], s, l == 0 ? bias : nullptr, lay[l], l == 0 ? act : KS_ACT_NONE);
        in = out;                                                    // bias after the last hop
    }
    if (!ws)
        for (int i = 0; i < nbuf; ++i) cudaFreeAsync(buf[i], s);
    return st;
}

}  // namespace

namespace ks {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms(int device) {
    static std::mutex mu;
    static std::vector<int> cache;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)cache.size() <= device) cache.resize(device + 1, 0);
    if (!cache[device]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cache[device] = n > 0 ? n : 148;
    }
    return cache[device];
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("KS_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace ks

extern "C" {

ks_handle_t ks_pack_weights(int64_t a, int64_t b, int64_t c, int64_t d, const float* K) {
    return ks_pack_weights_ex(a, b, c, d, K, KS_DTYPE_F32);
}

ks_handle_t ks_pack_weights_ex(int64_t a, int64_t b, int64_t c, int64_t d, const void* K, ks_dtype_t dtype) {
    if (dtype != KS_DTYPE_F32 && dtype != KS_DTYPE_BF16 && dtype != KS_DTYPE_F16) {
        fail(KS_ERR_INVALID_ARG, "bad dtype %d", (int)dtype);
        return nullptr;
    }
    if (a < 1 || b < 1 || c < 1 || d < 1) {
        fail(KS_ERR_PATTERN, "pattern entries must be >= 1, got (%lld,%lld,%lld,%lld)",
             (long long)a, (long long)b, (long long)c, (long long)d);
        return nullptr;
    }
    int64_t ab, abd, ac, acd, abc, nnz;
    if (!mul_ok(a, b, &ab) || !mul_ok(ab, d, &abd) || !mul_ok(a, c, &ac) || !mul_ok(ac, d, &acd) ||
        !mul_ok(ab, c, &abc) || !mul_ok(abc, d, &nnz) || nnz > (int64_t(1) << 40)) {
        fail(KS_ERR_PATTERN, "pattern sizes overflow");
        return nullptr;
    }
    if (!K) { fail(KS_ERR_INVALID_ARG, "K is NULL"); return nullptr; }
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { fail(KS_ERR_DEVICE, "no CUDA device: %s", cudaGetErrorString(e)); return nullptr; }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) {
        fail(KS_ERR_DEVICE, "libks is built for sm_100a (B200); device %d is sm_%d%d", dev, major, minor);
        return nullptr;
    }
    auto* h = new ks_handle_s();
    h->a = a; h->b = b; h->c = c; h->d = d;
    h->M = abd; h->N = acd; h->nnz = nnz;
    h->device = dev;
    h->math = KS_MATH_FP32;
    h->forced = KS_KERNEL_AUTO;
    h->dtype = dtype;
    const bool f32 = dtype == KS_DTYPE_F32;
    const size_t bytes = (size_t)h->esize() * (size_t)nnz;
    if ((e = cudaMalloc(&h->k_canon, bytes)) != cudaSuccess ||
        (f32 && (e = cudaMalloc(&h->k_tile, bytes)) != cudaSuccess) ||
        (e = cudaMalloc(&h->k_tf32, bytes)) != cudaSuccess) {
        fail_cuda(e, "ks_pack_weights alloc");
        ks_free(h);
        return nullptr;
    }
    if ((e = cudaMemcpy(h->k_canon, K, bytes, cudaMemcpyDefault)) != cudaSuccess ||
        (e = f32 ? ks::pack_tiles(*h, 0) : ks::pack_half(*h, 0)) != cudaSuccess ||
        (e = cudaStreamSynchronize(0)) != cudaSuccess) {
        fail_cuda(e, "ks_pack_weights copy/pack");
        ks_free(h);
        return nullptr;
    }
    ok();
    return h;
}

void ks_free(ks_handle_t h) {
    if (!h) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != h->device) cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    cudaFree(h->k_canon);
    cudaFree(h->k_tile);
    cudaFree(h->k_tf32);
    cudaFree(h->k_lo);
    cudaFree(h->k_dense);
    if (cur >= 0 && cur != h->device) cudaSetDevice(cur);
    delete h;
}

ks_status_t ks_get_pattern(ks_handle_t h, int64_t out[4]) {
    if (!h || !out) return fail(KS_ERR_INVALID_ARG, "NULL argument");
    out[0] = h->a; out[1] = h->b; out[2] = h->c; out[3] = h->d;
    return ok();
}

ks_status_t ks_set_math(ks_handle_t h, ks_math_t m) {
    if (!h) return fail(KS_ERR_INVALID_ARG, "NULL handle");
    if (m != KS_MATH_FP32 && m != KS_MATH_TF32 && m != KS_MATH_F32X3)
        return fail(KS_ERR_INVALID_ARG, "bad math %d", (int)m);
    if (m != KS_MATH_FP32 && h->dtype != KS_DTYPE_F32)
        return fail(KS_ERR_UNSUPPORTED, "math applies to F32 handles (half handles use kind::f16)");
    if (m != KS_MATH_FP32 && (h->b < 16 || h->c < 16))
        return fail(KS_ERR_UNSUPPORTED, "tensor-core math needs b,c >= 16 (pattern has b=%lld c=%lld)",
                    (long long)h->b, (long long)h->c);
    if (m == KS_MATH_F32X3 && !h->k_lo) {      // the low halves of the 3xTF32 split, once per handle
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != h->device) cudaSetDevice(h->device);
        float* lo = nullptr;
        cudaError_t e = cudaMalloc(&lo, sizeof(float) * (size_t)h->nnz);
        if (e == cudaSuccess) {
            h->k_lo = lo;
            if ((e = ks::pack_lo(*h, 0)) == cudaSuccess) e = cudaStreamSynchronize(0);
            if (e != cudaSuccess) { cudaFree(lo); h->k_lo = nullptr; }
        }
        if (cur >= 0 && cur != h->device) cudaSetDevice(cur);
        if (e != cudaSuccess) return fail_cuda(e, "ks_set_math(F32X3) pack");
    }
    if (m == KS_MATH_TF32 && !h->k_dense && h->d >= 2 && h->d <= ks::KS_DENSE_MAX_D &&
        (size_t)h->nnz * (size_t)h->d * sizeof(float) <= (size_t(256) << 20)) {
        // densified super-blocks for the BSF tensor-core path (see ks_tf32.cu), once per handle
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != h->device) cudaSetDevice(h->device);
        float* dn = nullptr;
        cudaError_t e = cudaMalloc(&dn, sizeof(float) * (size_t)h->nnz * (size_t)h->d);
        if (e == cudaSuccess) {
            h->k_dense = dn;
            if ((e = ks::pack_dense(*h, 0)) == cudaSuccess) e = cudaStreamSynchronize(0);
            if (e != cudaSuccess) { cudaFree(dn); h->k_dense = nullptr; }
        }
        if (cur >= 0 && cur != h->device) cudaSetDevice(cur);
        if (e != cudaSuccess) return fail_cuda(e, "ks_set_math(TF32) dense pack");
    }
    h->math = m;
    return ok();
}

ks_status_t ks_set_kernel(ks_handle_t h, ks_kernel_t k) {
    if (!h) return fail(KS_ERR_INVALID_ARG, "NULL handle");
    if (k < KS_KERNEL_AUTO || k > KS_KERNEL_SPLITC || k == KS_KERNEL_FUSED_CHAIN)
        return fail(KS_ERR_INVALID_ARG, "bad kernel %d", (int)k);
    h->forced = k;
    return ok();
}

ks_status_t ks_plan(ks_handle_t h, int64_t B, ks_layout_t layout, ks_kernel_t* out) {
    if (!h || !out || B < 0) return fail(KS_ERR_INVALID_ARG, "bad argument");
    if (layout != KS_LAYOUT_BSF && layout != KS_LAYOUT_BSL) return fail(KS_ERR_INVALID_ARG, "bad layout");
    // Plans assume 256-byte aligned (allocator) pointers.
    KsCall call{reinterpret_cast<const float*>(uintptr_t(256)), reinterpret_cast<float*>(uintptr_t(256)),
                B, (int)layout, nullptr};
    call.knobs = ks::plan_knobs(*h, call);
    ks_kernel_t k = choose(*h, call);
    if (k == KS_KERNEL_AUTO) return fail(KS_ERR_UNSUPPORTED, "forced kernel cannot run this call");
    *out = k;
    return ok();
}

ks_status_t ks_set_knobs(ks_handle_t h, int64_t knobs) {
    if (!h) return fail(KS_ERR_INVALID_ARG, "NULL handle");
    if (knobs < -1 || knobs > 0x3FF) return fail(KS_ERR_INVALID_ARG, "knobs must be -1 or a mask of KS_KNOB_* bits");
    h->knobs_override = knobs;
    return ok();
}

ks_status_t ks_plan_knobs(ks_handle_t h, int64_t B, ks_layout_t layout, uint32_t* knobs, int* source) {
    if (!h || !knobs || B < 0) return fail(KS_ERR_INVALID_ARG, "bad argument");
    if (layout != KS_LAYOUT_BSF && layout != KS_LAYOUT_BSL) return fail(KS_ERR_INVALID_ARG, "bad layout");
    KsCall call{reinterpret_cast<const float*>(uintptr_t(256)), reinterpret_cast<float*>(uintptr_t(256)),
                B, (int)layout, nullptr};
    int src = 0;
    *knobs = ks::plan_knobs(*h, call, &src);
    if (source) *source = src;
    return ok();
}

int ks_preset_count(void) { return ks::preset_count(); }

ks_status_t ks_matmul(ks_handle_t h, const float* X, float* Y, int64_t B, ks_layout_t layout,
                      ks_stream_t stream) {
    return ks_matmul_bias(h, X, Y, nullptr, B, layout, stream);
}

ks_status_t ks_matmul_act(ks_handle_t h, const void* X, void* Y, const void* bias, ks_activation_t act, int64_t B,
                          ks_layout_t layout, ks_stream_t stream) {
    if (!h) return fail(KS_ERR_INVALID_ARG, "NULL handle");
    if (act != KS_ACT_NONE && act != KS_ACT_GELU) return fail(KS_ERR_INVALID_ARG, "bad activation %d", (int)act);
    const uintptr_t amask = (uintptr_t)h->esize() - 1;
    if (reinterpret_cast<uintptr_t>(bias) & amask) return fail(KS_ERR_ALIGNMENT, "bias must be element-aligned");
    if (B < 0) return fail(KS_ERR_INVALID_ARG, "B must be >= 0");
    if (layout != KS_LAYOUT_BSF && layout != KS_LAYOUT_BSL) return fail(KS_ERR_INVALID_ARG, "bad layout %d", (int)layout);
    ks_status_t s = check_device(h);
    if (s != KS_OK) return s;
    if (B == 0) return ok();
    if (!X || !Y) return fail(KS_ERR_INVALID_ARG, "NULL X or Y");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & amask)
        return fail(KS_ERR_ALIGNMENT, "X and Y must be element-aligned");
    int64_t xb, yb;
    if (!mul_ok(B, h->N * h->esize(), &xb) || !mul_ok(B, h->M * h->esize(), &yb))
        return fail(KS_ERR_INVALID_ARG, "B too large");
    if (overlap(X, xb, Y, yb)) return fail(KS_ERR_INVALID_ARG, "X and Y overlap");
    s = run_one(*h, static_cast<const float*>(X), static_cast<float*>(Y), B, layout,
                static_cast<cudaStream_t>(stream), static_cast<const float*>(bias), -1, (int)act);
    return s == KS_OK ? ok() : s;
}

ks_status_t ks_matmul_any(ks_handle_t h, const void* X, void* Y, const void* bias, int64_t B,
                          ks_layout_t layout, ks_stream_t stream) {
    return ks_matmul_act(h, X, Y, bias, KS_ACT_NONE, B, layout, stream);
}

ks_status_t ks_matmul_bias(ks_handle_t h, const float* X, float* Y, const float* bias, int64_t B,
                           ks_layout_t layout, ks_stream_t stream) {
    if (h && h->dtype != KS_DTYPE_F32) return fail(KS_ERR_INVALID_ARG, "half handle: use ks_matmul_any");
    return ks_matmul_any(h, X, Y, bias, B, layout, stream);
}

ks_status_t ks_chain_ex(const ks_handle_t* hs, int L, const float* X, float* Y, int64_t B,
                        ks_layout_t layout, ks_stream_t stream) {
    return ks_chain_bias(hs, L, X, Y, nullptr, B, layout, stream);
}

ks_status_t ks_chain_act(const ks_handle_t* hs, int L, const void* X, void* Y, const void* bias,
                         ks_activation_t act, int64_t B, ks_layout_t layout, ks_stream_t stream) {
    if (act != KS_ACT_NONE && act != KS_ACT_GELU) return fail(KS_ERR_INVALID_ARG, "bad activation %d", (int)act);
    ks_status_t s = validate_chain(hs, L, B, (int)layout);
    if (s != KS_OK) return s;
    const int es = hs[0]->esize();
    const uintptr_t amask = (uintptr_t)es - 1;
    if (reinterpret_cast<uintptr_t>(bias) & amask) return fail(KS_ERR_ALIGNMENT, "bias must be element-aligned");
    if (B == 0) return ok();
    if (!X || !Y) return fail(KS_ERR_INVALID_ARG, "NULL X or Y");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & amask)
        return fail(KS_ERR_ALIGNMENT, "X and Y must be element-aligned");
    if (overlap(X, B * hs[L - 1]->N * es, Y, B * hs[0]->M * es)) return fail(KS_ERR_INVALID_ARG, "X and Y overlap");
    s = run_chain(hs, L, static_cast<const float*>(X), static_cast<float*>(Y), B, (int)layout,
                  static_cast<cudaStream_t>(stream), static_cast<const float*>(bias), nullptr, (int)act);
    return s == KS_OK ? ok() : s;
}

ks_status_t ks_chain_any(const ks_handle_t* hs, int L, const void* X, void* Y, const void* bias,
                         int64_t B, ks_layout_t layout, ks_stream_t stream) {
    return ks_chain_act(hs, L, X, Y, bias, KS_ACT_NONE, B, layout, stream);
}

ks_status_t ks_chain_bias(const ks_handle_t* hs, int L, const float* X, float* Y, const float* bias,
                          int64_t B, ks_layout_t layout, ks_stream_t stream) {
    if (hs && L >= 1 && hs[0] && hs[0]->dtype != KS_DTYPE_F32)
        return fail(KS_ERR_INVALID_ARG, "half handles: use ks_chain_any");
    return ks_chain_any(hs, L, X, Y, bias, B, layout, stream);
}

ks_status_t ks_get_dtype(ks_handle_t h, ks_dtype_t* out) {
    if (!h || !out) return fail(KS_ERR_INVALID_ARG, "NULL argument");
    *out = (ks_dtype_t)h->dtype;
    return ok();
}

ks_status_t ks_set_chain_fusion(int enable) {
    g_fusion.store(enable != 0);
    return ok();
}

ks_status_t ks_set_chain_mixed_layouts(int enable) {
    g_mixed.store(enable != 0);
    return ok();
}

int ks_chain_layouts(const ks_handle_t* hs, int L, int64_t B, ks_layout_t layout, int* out) {
    if (!out || validate_chain(hs, L, B, (int)layout) != KS_OK) return -1;
    const float* p = reinterpret_cast<const float*>(uintptr_t(256));
    const int mixed = plan_chain_layouts(hs, L, p, const_cast<float*>(p), B, (int)layout, out) ? 1 : 0;
    ok();
    return mixed;
}

ks_status_t ks_matmul_io(ks_handle_t h, const float* X, ks_layout_t x_layout, float* Y, ks_layout_t y_layout,
                         int64_t B, ks_stream_t stream) {
    if (!h) return fail(KS_ERR_INVALID_ARG, "NULL handle");
    if (h->dtype != KS_DTYPE_F32) return fail(KS_ERR_INVALID_ARG, "half handle: ks_matmul_io is FP32 / TF32 only");
    if (B < 0) return fail(KS_ERR_INVALID_ARG, "B must be >= 0");
    for (int l : {(int)x_layout, (int)y_layout})
        if (l != KS_LAYOUT_BSF && l != KS_LAYOUT_BSL) return fail(KS_ERR_INVALID_ARG, "bad layout %d", l);
    ks_status_t s = check_device(h);
    if (s != KS_OK) return s;
    if (B == 0) return ok();
    if (!X || !Y) return fail(KS_ERR_INVALID_ARG, "NULL X or Y");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 3)
        return fail(KS_ERR_ALIGNMENT, "X and Y must be 4-byte aligned");
    int64_t xb, yb;
    if (!mul_ok(B, h->N * 4, &xb) || !mul_ok(B, h->M * 4, &yb)) return fail(KS_ERR_INVALID_ARG, "B too large");
    if (overlap(X, xb, Y, yb)) return fail(KS_ERR_INVALID_ARG, "X and Y overlap");
    s = run_one(*h, X, Y, B, (int)x_layout, static_cast<cudaStream_t>(stream), nullptr, (int)y_layout);
    return s == KS_OK ? ok() : s;
}

int ks_chain_fusion_eligible(const ks_handle_t* hs, int L, int64_t B, ks_layout_t layout) {
    if (validate_chain(hs, L, B, (int)layout) != KS_OK) return 0;
    // plans assume 256-byte aligned (allocator) pointers
    KsCall call{reinterpret_cast<const float*>(uintptr_t(256)), reinterpret_cast<float*>(uintptr_t(256)), B,
                (int)layout, nullptr};
    ok();
    return fusion_ok(hs, L, call) ? 1 : 0;
}

ks_status_t ks_chain(const ks_handle_t* hs, int L, const float* X, float* Y, int64_t B,
                     ks_stream_t stream) {
    return ks_chain_ex(hs, L, X, Y, B, KS_LAYOUT_BSF, stream);
}

ks_status_t ks_chain_host(const ks_handle_t* hs, int L, const float* Xh, float* Yh, int64_t B,
                          ks_layout_t layout, ks_stream_t stream) {
    ks_status_t s = validate_chain(hs, L, B, (int)layout);
    if (s != KS_OK) return s;
    if (B == 0) return ok();
    if (!Xh || !Yh) return fail(KS_ERR_INVALID_ARG, "NULL X or Y");
    const int dev = hs[0]->device;
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    HostStreams* hsm = nullptr;
    cudaError_t e = host_streams(dev, &hsm);
    if (e != cudaSuccess) return fail_cuda(e, "internal streams");
    cudaMemPool_t pool;
    if ((e = get_pool(dev, &pool)) != cudaSuccess) return fail_cuda(e, "cudaMemPoolCreate");
    const int64_t es = hs[0]->esize();
    const int64_t N = hs[L - 1]->N, M = hs[0]->M;
    const size_t xbytes = (size_t)(es * B * N), ybytes = (size_t)(es * B * M);
    // Batch chunks of ~16 MB of X + Y, pipelined over three streams: the H2D copy
    // of chunk k+1 and the D2H copy of chunk k-1 overlap the chain on chunk k
    // (PCIe is full duplex; rows are independent).  BSL chunks are column
    // blocks (2-D copies into a contiguous N x Bc buffer), multiples of 4 columns.
    static const int64_t chunk_mb = [] {                 // KS_HOST_CHUNK_MB (experiments)
        const char* v = getenv("KS_HOST_CHUNK_MB");
        return (int64_t)(v && atoi(v) > 0 ? atoi(v) : 16);
    }();
    static const int64_t max_chunks = [] {               // KS_HOST_MAX_CHUNKS (experiments)
        const char* v = getenv("KS_HOST_MAX_CHUNKS");
        return (int64_t)(v && atoi(v) > 0 ? atoi(v) : 16);
    }();
    const int64_t per_row = es * (N + M);
    int64_t bc = (chunk_mb << 20) / (per_row > 0 ? per_row : 1);
    if (bc < 1) bc = 1;
    if (bc * max_chunks < B) bc = (B + max_chunks - 1) / max_chunks;
    if (layout == KS_LAYOUT_BSL) bc = (bc + 3) / 4 * 4;
    if (bc > B) bc = B;
    const int64_t nch = (B + bc - 1) / bc;
    void *dX = nullptr, *dY = nullptr;
    if ((e = cudaMallocFromPoolAsync(&dX, xbytes, pool, user)) != cudaSuccess) return fail_cuda(e, "staging X");
    if ((e = cudaMallocFromPoolAsync(&dY, ybytes, pool, user)) != cudaSuccess) {
        cudaFreeAsync(dX, user);
        return fail_cuda(e, "staging Y");
    }
    std::vector<cudaEvent_t> evs;
    auto event = [&](cudaEvent_t* ev) {
        cudaError_t r = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (r == cudaSuccess) evs.push_back(*ev);
        return r;
    };
    cudaEvent_t ev_start;
    if ((e = event(&ev_start)) == cudaSuccess) e = cudaEventRecord(ev_start, user);
    for (cudaStream_t t : {hsm->h2d, hsm->comp, hsm->d2h})
        if (e == cudaSuccess) e = cudaStreamWaitEvent(t, ev_start, 0);
    for (int64_t k = 0; k < nch && e == cudaSuccess && s == KS_OK; ++k) {
        const int64_t n0 = k * bc, nb = (B - n0) < bc ? (B - n0) : bc;
        // device chunk buffers: B x N / B x M (BSF) or N x nb / M x nb (BSL), contiguous
        char* xk = static_cast<char*>(dX) + es * n0 * N;
        char* yk = static_cast<char*>(dY) + es * n0 * M;
        // H2D of chunk k
        if (layout == KS_LAYOUT_BSF)
            e = cudaMemcpyAsync(xk, reinterpret_cast<const char*>(Xh) + es * n0 * N, (size_t)(es * nb * N),
                                cudaMemcpyHostToDevice, hsm->h2d);
        else   // column block [n0, n0 + nb) of the N x B host matrix -> contiguous N x nb
            e = cudaMemcpy2DAsync(xk, (size_t)(es * nb), reinterpret_cast<const char*>(Xh) + es * n0, (size_t)(es * B),
                                  (size_t)(es * nb), (size_t)N, cudaMemcpyHostToDevice, hsm->h2d);
        cudaEvent_t ev_in, ev_comp;
        if (e == cudaSuccess) e = event(&ev_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev_in, hsm->h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(hsm->comp, ev_in, 0);
        if (e != cudaSuccess) break;
        s = run_chain(hs, L, reinterpret_cast<const float*>(xk), reinterpret_cast<float*>(yk), nb, (int)layout,
                      hsm->comp);
        if (s != KS_OK) break;
        if ((e = event(&ev_comp)) == cudaSuccess) e = cudaEventRecord(ev_comp, hsm->comp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(hsm->d2h, ev_comp, 0);
        if (e != cudaSuccess) break;
        // D2H of chunk k
        if (layout == KS_LAYOUT_BSF)
            e = cudaMemcpyAsync(reinterpret_cast<char*>(Yh) + es * n0 * M, yk, (size_t)(es * nb * M),
                                cudaMemcpyDeviceToHost, hsm->d2h);
        else
            e = cudaMemcpy2DAsync(reinterpret_cast<char*>(Yh) + es * n0, (size_t)(es * B), yk, (size_t)(es * nb),
                                  (size_t)(es * nb), (size_t)M, cudaMemcpyDeviceToHost, hsm->d2h);
    }
    // join: the caller's stream waits for every internal stream (also on error paths)
    for (cudaStream_t t : {hsm->h2d, hsm->comp, hsm->d2h}) {
        cudaEvent_t ev_j;
        if (event(&ev_j) == cudaSuccess && cudaEventRecord(ev_j, t) == cudaSuccess) cudaStreamWaitEvent(user, ev_j, 0);
    }
    cudaFreeAsync(dX, user);
    cudaFreeAsync(dY, user);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);    // released once complete
    if (e != cudaSuccess) return fail_cuda(e, "host<->device pipeline");
    return s == KS_OK ? ok() : s;
}

}  // extern "C"

struct ks_graph_s {
    cudaGraphExec_t exec = nullptr;
    void* ws[2] = {nullptr, nullptr};
    int device = 0;
    int kernels = 0;
};

extern "C" {

ks_graph_t ks_chain_graph(const ks_handle_t* hs, int L, const void* X, void* Y, const void* bias, int64_t B,
                          ks_layout_t layout) {
    ks_status_t s = validate_chain(hs, L, B, (int)layout);
    if (s != KS_OK) return nullptr;
    if (B == 0 || !X || !Y) {
        fail(KS_ERR_INVALID_ARG, "ks_chain_graph needs B > 0 and non-NULL X, Y");
        return nullptr;
    }
    const int es = hs[0]->esize();
    const uintptr_t amask = (uintptr_t)es - 1;
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(bias)) & amask) {
        fail(KS_ERR_ALIGNMENT, "X, Y and bias must be element-aligned");
        return nullptr;
    }
    if (overlap(X, B * hs[L - 1]->N * es, Y, B * hs[0]->M * es)) {
        fail(KS_ERR_INVALID_ARG, "X and Y overlap");
        return nullptr;
    }
    auto* g = new ks_graph_s();
    g->device = hs[0]->device;
    size_t bytes;
    int nbuf;
    chain_workspace(hs, L, B, &bytes, &nbuf);
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < nbuf && e == cudaSuccess; ++i) e = cudaMalloc(&g->ws[i], bytes);
    cudaStream_t st = nullptr;
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGraph_t graph = nullptr;
    if (e == cudaSuccess) e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        const int64_t l0 = g_launches.load();
        t_capturing = true;
        s = run_chain(hs, L, static_cast<const float*>(X), static_cast<float*>(Y), B, (int)layout, st,
                      static_cast<const float*>(bias), g->ws);
        t_capturing = false;
        g->kernels = (int)(g_launches.load() - l0);
        g_launches.fetch_sub(g->kernels);              // counted again at every replay
        const cudaError_t e2 = cudaStreamEndCapture(st, &graph);
        if (s == KS_OK && e2 != cudaSuccess) e = e2;
    }
    if (e == cudaSuccess && s == KS_OK) e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (st) cudaStreamDestroy(st);
    if (e != cudaSuccess || s != KS_OK) {
        if (e != cudaSuccess) fail_cuda(e, "ks_chain_graph");
        ks_graph_free(g);
        return nullptr;
    }
    ok();
    return g;
}

ks_status_t ks_graph_launch(ks_graph_t g, ks_stream_t stream) {
    if (!g || !g->exec) return fail(KS_ERR_INVALID_ARG, "NULL graph");
    const cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail_cuda(e, "cudaGraphLaunch");
    g_launches.fetch_add(g->kernels, std::memory_order_relaxed);
    return ok();
}

int ks_graph_kernel_count(ks_graph_t g) { return g ? g->kernels : -1; }

void ks_graph_free(ks_graph_t g) {
    if (!g) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();
    if (g->exec) cudaGraphExecDestroy(g->exec);
    for (void* p : g->ws)
        if (p) cudaFree(p);
    cudaSetDevice(cur);
    delete g;
}

ks_status_t ks_read_packed(ks_handle_t h, int variant, float* dst, int64_t count) {
    if (!h || !dst) return fail(KS_ERR_INVALID_ARG, "NULL argument");
    const int64_t want = variant == 4 ? h->nnz * h->d : h->nnz;
    if (count != want) return fail(KS_ERR_INVALID_ARG, "count must be %lld for variant %d", (long long)want, variant);
    const float* src = variant == 0 ? h->k_canon : variant == 1 ? h->k_tile : variant == 2 ? h->k_tf32
                     : variant == 3 ? h->k_lo : variant == 4 ? h->k_dense : nullptr;
    if (!src) return fail(KS_ERR_INVALID_ARG, "variant must be 0, 1, 2, 3 (after ks_set_math(F32X3)) or 4 "
                          "(after ks_set_math(TF32), 2 <= d <= 8)");
    cudaError_t e = cudaMemcpy(dst, src, (size_t)h->esize() * (size_t)count, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail_cuda(e, "ks_read_packed");
    return ok();
}

ks_status_t ks_trace_enable(int on) {
    std::lock_guard<std::mutex> lk(g_trace_mu);
    for (auto& r : g_trace) {
        g_event_pool.push_back(r.start);
        g_event_pool.push_back(r.stop);
    }
    g_trace.clear();
    g_trace_on.store(on != 0);
    return ok();
}

ks_status_t ks_trace_read(int64_t max, int64_t* count, float* ms, int* family, double* bytes) {
    if (max < 0) return fail(KS_ERR_INVALID_ARG, "max must be >= 0");
    std::lock_guard<std::mutex> lk(g_trace_mu);
    if (count) *count = (int64_t)g_trace.size();
    ks_status_t st = KS_OK;
    for (size_t t = 0; t < g_trace.size(); ++t) {
        TraceRec& r = g_trace[t];
        if ((int64_t)t < max) {
            float v = 0.f;
            cudaError_t e = cudaEventSynchronize(r.stop);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&v, r.start, r.stop);
            if (e != cudaSuccess && st == KS_OK) st = fail_cuda(e, "ks_trace_read");
            if (ms) ms[t] = v;
            if (family) family[t] = r.family;
            if (bytes) bytes[t] = r.bytes;
        }
        g_event_pool.push_back(r.start);
        g_event_pool.push_back(r.stop);
    }
    g_trace.clear();
    return st == KS_OK ? ok() : st;
}

ks_status_t ks_last_error(void) { return t_status; }
const char* ks_last_error_message(void) { return t_msg; }

const char* ks_status_string(ks_status_t s) {
    switch (s) {
        case KS_OK: return "KS_OK";
        case KS_ERR_INVALID_ARG: return "KS_ERR_INVALID_ARG";
        case KS_ERR_PATTERN: return "KS_ERR_PATTERN";
        case KS_ERR_CHAIN_SHAPE: return "KS_ERR_CHAIN_SHAPE";
        case KS_ERR_UNSUPPORTED: return "KS_ERR_UNSUPPORTED";
        case KS_ERR_DEVICE: return "KS_ERR_DEVICE";
        case KS_ERR_ALIGNMENT: return "KS_ERR_ALIGNMENT";
        case KS_ERR_OOM: return "KS_ERR_OOM";
        case KS_ERR_CUDA: return "KS_ERR_CUDA";
    }
    return "KS_ERR_UNKNOWN";
}

uint64_t ks_kernel_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int ks_abi_version(void) { return KS_ABI_VERSION; }

}  // extern "C"
