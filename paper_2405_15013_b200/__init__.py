"""B200-native Kronecker-sparse matmul (arXiv 2405.15013 hot path).

The product is libks.so (C ABI in include/ks.h, CUDA for sm_100a in csrc/);
``ks`` is its thin Python binding.
"""
from .ks import (  # noqa: F401
    BSF, BSL, MATH_FP32, MATH_TF32, MATH_F32X3, DTYPE_F32, DTYPE_BF16, DTYPE_F16,
    KERNEL_AUTO, KERNEL_GENERIC, KERNEL_STREAM, KERNEL_FFMA, KERNEL_TF32, KERNEL_SPLITC,
    Factor, KSError, matmul, chain, chain_host, launch_count, load_library, LIB_PATH, EXPORTS,
    trace_enable, trace_read, set_chain_fusion, chain_fusion_eligible, ChainGraph, peak_ffma_tflops,
    matmul_io, set_chain_mixed_layouts, chain_layouts,
)
from .kslinear import KSLinear  # noqa: F401
