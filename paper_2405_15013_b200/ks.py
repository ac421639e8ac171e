"""Thin Python binding of libks.so (include/ks.h).  Argument marshalling only:
every step of the KS path runs in the library's CUDA kernels.  PyTorch
supplies device memory and streams.

There is no CPU fallback: if libks.so is missing or cannot run on the current
device, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KS_LIB") or os.path.join(_PKG, "lib", "libks.so")   # KS_LIB: A/B experiments only

BSF, BSL = 0, 1
MATH_FP32, MATH_TF32, MATH_F32X3 = 0, 1, 2
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_STREAM, KERNEL_FFMA, KERNEL_TF32 = range(5)
KERNEL_SPLITC = 6
KERNEL_NAMES = {0: "auto", 1: "generic", 2: "stream", 3: "ffma", 4: "tf32", 5: "fused_chain", 6: "splitc"}
# launch-plan knobs (ks_knob_t, include/ks.h)
KNOB_TF32_V2, KNOB_V2_NKB2, KNOB_DENSIFY, KNOB_J8, KNOB_BN256, KNOB_KB32, KNOB_FFMA_WS, KNOB_FFMA_WSG, \
    KNOB_TF32_MN, KNOB_FFMA_WSL = (1 << i for i in range(10))
KNOB_NAMES = {1: "tf32_v2", 2: "v2_nkb2", 4: "densify", 8: "j8", 16: "bn256", 32: "kb32", 64: "ffma_ws",
              128: "ffma_wsg", 256: "tf32_mn", 512: "ffma_wsl"}


def preset_count() -> int:
    return int(load_library().ks_preset_count())

STATUS = {0: "KS_OK", 1: "KS_ERR_INVALID_ARG", 2: "KS_ERR_PATTERN", 3: "KS_ERR_CHAIN_SHAPE",
          4: "KS_ERR_UNSUPPORTED", 5: "KS_ERR_DEVICE", 6: "KS_ERR_ALIGNMENT", 7: "KS_ERR_OOM",
          8: "KS_ERR_CUDA"}

# Every symbol include/ks.h declares (tests check the .so exports them all).
DTYPE_F32, DTYPE_BF16, DTYPE_F16 = 0, 1, 2

EXPORTS = ["ks_pack_weights", "ks_pack_weights_ex", "ks_get_dtype", "ks_matmul_any", "ks_chain_any",
           "ks_free", "ks_get_pattern", "ks_set_math", "ks_set_kernel",
           "ks_plan", "ks_matmul", "ks_chain", "ks_chain_ex", "ks_matmul_bias", "ks_chain_bias",
           "ks_set_chain_fusion",
           "ks_chain_fusion_eligible", "ks_chain_host", "ks_read_packed",
           "ks_trace_enable", "ks_trace_read",
           "ks_last_error", "ks_last_error_message", "ks_status_string",
           "ks_kernel_launch_count", "ks_abi_version",
           "ks_chain_graph", "ks_graph_launch", "ks_graph_kernel_count", "ks_graph_free", "ks_peak_ffma",
           "ks_set_knobs", "ks_plan_knobs", "ks_preset_count",
           "ks_matmul_io", "ks_set_chain_mixed_layouts", "ks_chain_layouts", "ks_matmul_act", "ks_chain_act"]


class KSError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libks.so and declare the ABI.  Raises loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libks.so not built ({path}); run `python -m paper_2405_15013_b200.build`")
    lib = ctypes.CDLL(path)
    i64, vp, fp = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
    st = ctypes.c_int
    lib.ks_pack_weights.argtypes = [i64, i64, i64, i64, fp]
    lib.ks_pack_weights.restype = vp
    lib.ks_pack_weights_ex.argtypes = [i64, i64, i64, i64, fp, ctypes.c_int]
    lib.ks_pack_weights_ex.restype = vp
    lib.ks_get_dtype.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    lib.ks_get_dtype.restype = st
    lib.ks_matmul_any.argtypes = [vp, fp, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_matmul_any.restype = st
    lib.ks_chain_any.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_chain_any.restype = st
    lib.ks_free.argtypes = [vp]
    lib.ks_free.restype = None
    lib.ks_get_pattern.argtypes = [vp, ctypes.POINTER(i64)]
    lib.ks_get_pattern.restype = st
    lib.ks_set_math.argtypes = [vp, ctypes.c_int]
    lib.ks_set_math.restype = st
    lib.ks_set_kernel.argtypes = [vp, ctypes.c_int]
    lib.ks_set_kernel.restype = st
    lib.ks_plan.argtypes = [vp, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    lib.ks_plan.restype = st
    lib.ks_matmul.argtypes = [vp, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_matmul.restype = st
    lib.ks_chain.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, i64, vp]
    lib.ks_chain.restype = st
    lib.ks_chain_ex.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_chain_ex.restype = st
    lib.ks_matmul_bias.argtypes = [vp, fp, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_matmul_bias.restype = st
    lib.ks_chain_bias.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_chain_bias.restype = st
    lib.ks_set_chain_fusion.argtypes = [ctypes.c_int]
    lib.ks_set_chain_fusion.restype = st
    lib.ks_chain_fusion_eligible.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64, ctypes.c_int]
    lib.ks_matmul_act.argtypes = [vp, fp, fp, fp, ctypes.c_int, i64, ctypes.c_int, vp]
    lib.ks_matmul_act.restype = ctypes.c_int
    lib.ks_chain_act.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, fp, ctypes.c_int, i64, ctypes.c_int, vp]
    lib.ks_chain_act.restype = ctypes.c_int
    lib.ks_matmul_io.argtypes = [vp, fp, ctypes.c_int, fp, ctypes.c_int, i64, vp]
    lib.ks_matmul_io.restype = ctypes.c_int
    lib.ks_set_chain_mixed_layouts.argtypes = [ctypes.c_int]
    lib.ks_set_chain_mixed_layouts.restype = ctypes.c_int
    lib.ks_chain_layouts.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    lib.ks_chain_layouts.restype = ctypes.c_int
    lib.ks_chain_fusion_eligible.restype = ctypes.c_int
    lib.ks_chain_host.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, i64, ctypes.c_int, vp]
    lib.ks_chain_host.restype = st
    lib.ks_read_packed.argtypes = [vp, ctypes.c_int, fp, i64]
    lib.ks_read_packed.restype = st
    lib.ks_trace_enable.argtypes = [ctypes.c_int]
    lib.ks_trace_enable.restype = st
    lib.ks_trace_read.argtypes = [i64, ctypes.POINTER(i64), vp, vp, vp]
    lib.ks_trace_read.restype = st
    lib.ks_last_error.argtypes = []
    lib.ks_last_error.restype = st
    lib.ks_last_error_message.argtypes = []
    lib.ks_last_error_message.restype = ctypes.c_char_p
    lib.ks_status_string.argtypes = [ctypes.c_int]
    lib.ks_status_string.restype = ctypes.c_char_p
    lib.ks_kernel_launch_count.argtypes = []
    lib.ks_kernel_launch_count.restype = ctypes.c_uint64
    lib.ks_abi_version.argtypes = []
    lib.ks_abi_version.restype = ctypes.c_int
    lib.ks_chain_graph.argtypes = [ctypes.POINTER(vp), ctypes.c_int, fp, fp, fp, i64, ctypes.c_int]
    lib.ks_chain_graph.restype = vp
    lib.ks_graph_launch.argtypes = [vp, vp]
    lib.ks_graph_launch.restype = st
    lib.ks_graph_kernel_count.argtypes = [vp]
    lib.ks_graph_kernel_count.restype = ctypes.c_int
    lib.ks_graph_free.argtypes = [vp]
    lib.ks_graph_free.restype = None
    lib.ks_peak_ffma.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    lib.ks_peak_ffma.restype = st
    lib.ks_set_knobs.argtypes = [vp, i64]
    lib.ks_set_knobs.restype = st
    lib.ks_plan_knobs.argtypes = [vp, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)]
    lib.ks_plan_knobs.restype = st
    lib.ks_preset_count.argtypes = []
    lib.ks_preset_count.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise KSError(status, _lib.ks_last_error_message().decode())


def _layout(layout) -> int:
    if layout in (BSF, "bsf", "BSF"):
        return BSF
    if layout in (BSL, "bsl", "BSL"):
        return BSL
    raise ValueError(f"layout must be 'bsf' or 'bsl', got {layout!r}")


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def launch_count() -> int:
    return int(load_library().ks_kernel_launch_count())


def peak_ffma_tflops(stream=None) -> float:
    """Measured FP32 FFMA TFLOP/s of the current device (ks_peak_ffma)."""
    out = ctypes.c_double(0.0)
    _check(load_library().ks_peak_ffma(_stream_ptr(stream), ctypes.byref(out)))
    return float(out.value)


def trace_enable(on: bool = True):
    """Start (clears) / stop the library's per-launch event tracing."""
    _check(load_library().ks_trace_enable(1 if on else 0))


def trace_read(max_records: int = 1 << 20):
    """(ms, family_name, model_bytes) per traced launch, oldest first; clears."""
    lib = load_library()
    cnt = ctypes.c_int64(0)
    ms = np.zeros(max_records, np.float32)
    fam = np.zeros(max_records, np.int32)
    byt = np.zeros(max_records, np.float64)
    _check(lib.ks_trace_read(max_records, ctypes.byref(cnt), ctypes.c_void_p(ms.ctypes.data),
                             ctypes.c_void_p(fam.ctypes.data), ctypes.c_void_p(byt.ctypes.data)))
    n = min(int(cnt.value), max_records)
    return ms[:n], [KERNEL_NAMES[int(f)] for f in fam[:n]], byt[:n]


class Factor:
    """One packed KS factor (opaque handle of ks_pack_weights)."""

    def __init__(self, a: int, b: int, c: int, d: int, K):
        lib = load_library()
        self.pattern = (int(a), int(b), int(c), int(d))
        self.M = a * b * d
        self.N = a * c * d
        self.nnz = a * b * c * d
        self._keep = None
        if min(self.pattern) < 1:      # let the library report KS_ERR_PATTERN
            h = lib.ks_pack_weights(a, b, c, d, None)
            _check(lib.ks_last_error())
        if isinstance(K, np.ndarray):
            arr = np.ascontiguousarray(K, dtype=np.float32).reshape(-1)
            if arr.size != self.nnz:
                raise ValueError(f"K must have a*b*c*d = {self.nnz} values")
            ptr = arr.ctypes.data
            self._keep = arr
        self.dtype = DTYPE_F32
        if not isinstance(K, np.ndarray):  # torch tensor (host or device)
            if K.numel() != self.nnz or not K.is_contiguous():
                raise ValueError(f"K must be contiguous with a*b*c*d = {self.nnz} values")
            import torch
            dt = {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16, torch.float16: DTYPE_F16}.get(K.dtype)
            if dt is None:
                raise TypeError("K must be float32, bfloat16 or float16")
            self.dtype = dt
            ptr = K.data_ptr()
            self._keep = K
        h = lib.ks_pack_weights_ex(a, b, c, d, ctypes.c_void_p(ptr), self.dtype)
        if not h:
            _check(lib.ks_last_error())
        self._h = ctypes.c_void_p(h)

    @property
    def handle(self):
        return self._h

    def set_math(self, math: int):
        _check(_lib.ks_set_math(self._h, int(math)))
        return self

    def set_kernel(self, kernel: int):
        _check(_lib.ks_set_kernel(self._h, int(kernel)))
        return self

    def plan(self, B: int, layout="bsf") -> str:
        out = ctypes.c_int(0)
        _check(_lib.ks_plan(self._h, int(B), _layout(layout), ctypes.byref(out)))
        return KERNEL_NAMES[out.value]

    def set_knobs(self, knobs: int):
        """Force the launch-plan knobs (KNOB_* bits) of every call on this handle; -1 = plan."""
        _check(_lib.ks_set_knobs(self._h, int(knobs)))
        return self

    def plan_knobs(self, B: int, layout="bsf"):
        """(knobs, source) a call would use; source 0 rules, 1 preset table, 2 override."""
        k, src = ctypes.c_uint32(0), ctypes.c_int(0)
        _check(_lib.ks_plan_knobs(self._h, int(B), _layout(layout), ctypes.byref(k), ctypes.byref(src)))
        return int(k.value), int(src.value)

    def get_pattern(self):
        out = (ctypes.c_int64 * 4)()
        _check(_lib.ks_get_pattern(self._h, out))
        return tuple(out)

    def read_packed(self, variant: int) -> np.ndarray:
        n = self.nnz * self.pattern[3] if variant == 4 else self.nnz
        out = np.empty(n, dtype=np.float32 if self.dtype == DTYPE_F32 else np.uint16)
        _check(_lib.ks_read_packed(self._h, int(variant), ctypes.c_void_p(out.ctypes.data), n))
        return out

    def free(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.ks_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _dev_ptr(t, what):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _torch_dtype(dtype_id):
    import torch
    return {DTYPE_F32: torch.float32, DTYPE_BF16: torch.bfloat16, DTYPE_F16: torch.float16}[dtype_id]


def _check_io(dtype_id, n_in, n_out, X, Y, B, lay, bias=None):
    """Reject, before the C ABI sees them, arguments that would make a kernel
    read or write out of bounds: element type, shapes against (B, N) / (B, M)
    in the given layout, bias length, and device.  Raises ValueError/TypeError."""
    want = _torch_dtype(dtype_id)
    if B < 0:
        raise ValueError(f"B must be >= 0, got {B}")
    for t, what, n in ((X, "X", n_in), (Y, "Y", n_out)):
        if t.dtype != want:
            raise TypeError(f"{what} has dtype {t.dtype}, the factor computes in {want}")
        exp = (B, n) if lay == BSF else (n, B)
        if tuple(t.shape) != exp:
            raise ValueError(f"{what} must have shape {exp} ({'BSF' if lay == BSF else 'BSL'}), got {tuple(t.shape)}")
    if X.device != Y.device:
        raise ValueError(f"X is on {X.device}, Y on {Y.device}")
    if bias is not None:
        if bias.dtype != want:
            raise TypeError(f"bias has dtype {bias.dtype}, expected {want}")
        if bias.numel() != n_out:
            raise ValueError(f"bias must have M = {n_out} values, got {bias.numel()}")
        if bias.device != X.device:
            raise ValueError(f"bias is on {bias.device}, X on {X.device}")


ACTIVATIONS = {None: 0, "none": 0, "gelu": 1}


def _act(act) -> int:
    if act not in ACTIVATIONS:
        raise ValueError(f"activation must be one of {sorted(k for k in ACTIVATIONS if k)} or None, got {act!r}")
    return ACTIVATIONS[act]


def matmul(f: Factor, X, Y=None, layout="bsf", stream=None, B: int | None = None, bias=None, act=None):
    """Y = act(X K^T (+ bias)) through ks_matmul / ks_matmul_bias / ks_matmul_act.
    X: CUDA tensor of the factor's element type, (B, N) for BSF or (N, B) for
    BSL; bias: (M,) or None; act: None or "gelu" (fused into the epilogue)."""
    import torch
    lay = _layout(layout)
    if B is None:
        B = X.shape[0] if lay == BSF else X.shape[1]
    if Y is None:
        Y = torch.empty((B, f.M) if lay == BSF else (f.M, B), device=X.device, dtype=_torch_dtype(f.dtype))
    _check_io(f.dtype, f.N, f.M, X, Y, int(B), lay, bias)
    a = _act(act)
    if a:
        bp = _dev_ptr(bias, "bias") if bias is not None else None
        _check(_lib.ks_matmul_act(f.handle, _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), bp, a, int(B), lay,
                                  _stream_ptr(stream)))
    elif f.dtype != DTYPE_F32:
        bp = _dev_ptr(bias, "bias") if bias is not None else None
        _check(_lib.ks_matmul_any(f.handle, _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), bp, int(B), lay,
                                  _stream_ptr(stream)))
    elif bias is None:
        _check(_lib.ks_matmul(f.handle, _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), int(B), lay, _stream_ptr(stream)))
    else:
        _check(_lib.ks_matmul_bias(f.handle, _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), _dev_ptr(bias, "bias"), int(B),
                                   lay, _stream_ptr(stream)))
    return Y


def _handles(factors):
    arr = (ctypes.c_void_p * len(factors))(*[f.handle.value for f in factors])
    return arr


def chain(factors, X, Y=None, layout="bsf", stream=None, bias=None, act=None):
    """Y = act(X K_L^T ... K_1^T (+ bias)) through ks_chain_ex / ks_chain_bias /
    ks_chain_act; factors in paper order K_1..K_L."""
    import torch
    lay = _layout(layout)
    if not factors:
        raise ValueError("a chain needs at least one factor")
    B = X.shape[0] if lay == BSF else X.shape[1]
    M = factors[0].M
    if Y is None:
        Y = torch.empty((B, M) if lay == BSF else (M, B), device=X.device, dtype=_torch_dtype(factors[0].dtype))
    if any(f.dtype != factors[0].dtype for f in factors):
        raise TypeError("all factors of a chain must have the same element type")
    _check_io(factors[0].dtype, factors[-1].N, M, X, Y, int(B), lay, bias)
    a = _act(act)
    if a:
        bp = _dev_ptr(bias, "bias") if bias is not None else None
        _check(_lib.ks_chain_act(_handles(factors), len(factors), _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), bp, a,
                                 int(B), lay, _stream_ptr(stream)))
    elif factors[0].dtype != DTYPE_F32:
        bp = _dev_ptr(bias, "bias") if bias is not None else None
        _check(_lib.ks_chain_any(_handles(factors), len(factors), _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), bp,
                                 int(B), lay, _stream_ptr(stream)))
    elif bias is None:
        _check(_lib.ks_chain_ex(_handles(factors), len(factors), _dev_ptr(X, "X"), _dev_ptr(Y, "Y"),
                                int(B), lay, _stream_ptr(stream)))
    else:
        _check(_lib.ks_chain_bias(_handles(factors), len(factors), _dev_ptr(X, "X"), _dev_ptr(Y, "Y"),
                                  _dev_ptr(bias, "bias"), int(B), lay, _stream_ptr(stream)))
    return Y


def set_chain_fusion(enable: bool):
    """Process-wide chain fusion policy (ks_set_chain_fusion); default on."""
    _check(load_library().ks_set_chain_fusion(1 if enable else 0))


def chain_fusion_eligible(factors, B: int, layout="bsf") -> bool:
    return bool(load_library().ks_chain_fusion_eligible(_handles(factors), len(factors), int(B), _layout(layout)))


def matmul_io(f: Factor, X, x_layout, Y=None, y_layout="bsf", stream=None, B: int | None = None):
    """Y = X K^T with X in x_layout and Y in y_layout (ks_matmul_io; FP32 handles)."""
    import torch
    xl, yl = _layout(x_layout), _layout(y_layout)
    if f.dtype != DTYPE_F32:
        raise TypeError("matmul_io: FP32 handles only")
    if B is None:
        B = X.shape[0] if xl == BSF else X.shape[1]
    if Y is None:
        Y = torch.empty((B, f.M) if yl == BSF else (f.M, B), device=X.device, dtype=torch.float32)
    if B < 0:
        raise ValueError(f"B must be >= 0, got {B}")
    for t, what, n, lay in ((X, "X", f.N, xl), (Y, "Y", f.M, yl)):
        if t.dtype != torch.float32:
            raise TypeError(f"{what} has dtype {t.dtype}, the factor computes in torch.float32")
        exp = (B, n) if lay == BSF else (n, B)
        if tuple(t.shape) != exp:
            raise ValueError(f"{what} must have shape {exp} ({'BSF' if lay == BSF else 'BSL'}), got {tuple(t.shape)}")
    if X.device != Y.device:
        raise ValueError(f"X is on {X.device}, Y on {Y.device}")
    _check(_lib.ks_matmul_io(f.handle, _dev_ptr(X, "X"), xl, _dev_ptr(Y, "Y"), yl, int(B), _stream_ptr(stream)))
    return Y


def set_chain_mixed_layouts(enable: bool):
    """Process-wide mixed-layout intermediate policy (ks_set_chain_mixed_layouts); default on."""
    _check(load_library().ks_set_chain_mixed_layouts(1 if enable else 0))


def chain_layouts(factors, B: int, layout="bsf"):
    """(mixed, [layout of the output of K_1 (= Y's) .. K_L, X's layout]) that ks_chain_ex would use."""
    L = len(factors)
    out = (ctypes.c_int * (L + 1))()
    r = load_library().ks_chain_layouts(_handles(factors), L, int(B), _layout(layout), out)
    if r < 0:
        raise ValueError("invalid chain")
    return bool(r), ["bsf" if v == BSF else "bsl" for v in out]


def chain_host(factors, X_host, Y_host, layout="bsf", stream=None):
    """ks_chain_host: host X in, host Y out (copies enqueued on `stream`)."""
    lay = _layout(layout)
    B = X_host.shape[0] if lay == BSF else X_host.shape[1]
    for t, w in ((X_host, "X_host"), (Y_host, "Y_host")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{w} must be a contiguous host tensor")
    if factors[0].dtype != DTYPE_F32:
        raise TypeError("ks_chain_host takes F32 factors")
    _check_io(DTYPE_F32, factors[-1].N, factors[0].M, X_host, Y_host, int(B), lay)
    _check(_lib.ks_chain_host(_handles(factors), len(factors), ctypes.c_void_p(X_host.data_ptr()),
                              ctypes.c_void_p(Y_host.data_ptr()), int(B), lay, _stream_ptr(stream)))
    return Y_host


class ChainGraph:
    """ks_chain_graph: the launches of chain(factors, X, Y, layout, bias) captured
    once into a CUDA graph; launch() replays them with one cudaGraphLaunch.  X, Y
    and bias are bound at construction (their contents may change between
    launches); the factors must outlive the graph."""

    def __init__(self, factors, X, Y, layout="bsf", bias=None):
        lay = _layout(layout)
        lib = load_library()
        B = X.shape[0] if lay == BSF else X.shape[1]
        _check_io(factors[0].dtype, factors[-1].N, factors[0].M, X, Y, int(B), lay, bias)
        self._keep = (list(factors), X, Y, bias)
        bp = _dev_ptr(bias, "bias") if bias is not None else None
        h = lib.ks_chain_graph(_handles(factors), len(factors), _dev_ptr(X, "X"), _dev_ptr(Y, "Y"), bp, int(B), lay)
        if not h:
            raise KSError(lib.ks_last_error(), lib.ks_last_error_message().decode())
        self._g = ctypes.c_void_p(h)
        self.kernels = int(lib.ks_graph_kernel_count(self._g))

    def launch(self, stream=None):
        _check(_lib.ks_graph_launch(self._g, _stream_ptr(stream)))

    def free(self):
        if getattr(self, "_g", None) is not None and _lib is not None:
            _lib.ks_graph_free(self._g)
            self._g = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass
