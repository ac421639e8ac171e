"""Host-side argument checks of the Python binding (ks._check_io), run on CPU
tensors: every mismatch that would make a kernel read or write out of bounds
is rejected before the C ABI is called."""
import pytest
import torch

from paper_2405_15013_b200 import ks


def _io(B, N, M, lay="bsf", dt=torch.float32):
    X = torch.zeros((B, N) if lay == "bsf" else (N, B), dtype=dt)
    Y = torch.zeros((B, M) if lay == "bsf" else (M, B), dtype=dt)
    return X, Y


def test_accepts_matching_shapes_both_layouts():
    for lay, L in (("bsf", ks.BSF), ("bsl", ks.BSL)):
        X, Y = _io(7, 16, 24, lay)
        ks._check_io(ks.DTYPE_F32, 16, 24, X, Y, 7, L, torch.zeros(24))
        Xh, Yh = _io(7, 16, 24, lay, torch.bfloat16)
        ks._check_io(ks.DTYPE_BF16, 16, 24, Xh, Yh, 7, L)


@pytest.mark.parametrize("case", ["dtype_x", "dtype_y", "feat", "out", "B_big", "B_neg", "bias_len",
                                  "bias_dtype", "bsl_transposed"])
def test_rejects_mismatches(case):
    X, Y = _io(8, 16, 24)
    bias = None
    B, lay, n_in, n_out, dt = 8, ks.BSF, 16, 24, ks.DTYPE_F32
    if case == "dtype_x":
        X = X.half()
    elif case == "dtype_y":
        Y = Y.bfloat16()
    elif case == "feat":
        n_in = 32
    elif case == "out":
        Y = torch.zeros(8, 12)
    elif case == "B_big":
        B = 9
    elif case == "B_neg":
        B = -1
    elif case == "bias_len":
        bias = torch.zeros(23)
    elif case == "bias_dtype":
        bias = torch.zeros(24, dtype=torch.float64)
    elif case == "bsl_transposed":
        lay = ks.BSL                     # BSF-shaped tensors passed as BSL
    with pytest.raises((ValueError, TypeError)):
        ks._check_io(dt, n_in, n_out, X, Y, B, lay, bias)
