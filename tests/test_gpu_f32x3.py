"""GPU parity of the F32X3 mode: FP32 accuracy on the tcgen05 tensor cores
through the 3xTF32 split (not in the paper).

x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi) (split in shared
memory), and the same for k at pack time; every MMA operand is then exact
TF32.  The kernel accumulates x_lo k_hi + x_hi k_lo + x_hi k_hi in FP32,
dropping x_lo k_lo (<= 2^-22 |x k|) and the rounding of the two low parts
(<= 2^-22 each): per product at most 3 * 2^-22 < 2^-20 relative, i.e.
u_in = 2^-21 in the O-6 envelope, over 3c accumulated terms (gamma_{4c} via
envelope_delta(2c, .), with slack).
The contract is the FP32 one: normwise error <= 1e-5 against the FP64 oracle.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import ksgen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


def run(ksb, f, X_bsf, layout, bias=None):
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
    bt = None if bias is None else dev(bias)
    if layout == "bsf":
        Y = ksb.matmul(f, dev(X_bsf), layout="bsf", bias=bt)
        torch.cuda.synchronize()
        return Y.cpu().numpy()
    Y = ksb.matmul(f, dev(ksgen.to_bsl(X_bsf)), layout="bsl", bias=bt)
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


CASES = [((1, 48, 48, 1), "bsf"), ((1, 64, 64, 1), "bsf"), ((2, 128, 128, 1), "bsf"), ((6, 64, 256, 1), "bsf"),
         ((64, 64, 64, 1), "bsf"), ((1, 16, 24, 1), "bsf"), ((2, 96, 96, 1), "bsf"),
         ((1, 768, 192, 2), "bsl"), ((1, 256, 64, 16), "bsl"), ((1, 48, 48, 64), "bsl"), ((3, 96, 96, 4), "bsl"),
         ((1, 128, 128, 3), "bsl"), ((2, 16, 24, 3), "bsl"), ((6, 64, 64, 1), "bsl"), ((1, 320, 40, 2), "bsl"),
         # BSF, d > 1: J = d contiguous (d <= 4), four-j gather (d % 4 == 0, d > 4)
         ((1, 64, 64, 4), "bsf"), ((2, 48, 48, 16), "bsf"), ((1, 128, 128, 8), "bsf"), ((3, 96, 96, 4), "bsf"),
         ((2, 16, 32, 12), "bsf"), ((1, 256, 64, 16), "bsf"), ((1, 128, 128, 3), "bsf"), ((2, 48, 48, 2), "bsf"),
         ((1, 768, 192, 2), "bsf")]


@pytest.mark.parametrize("p,layout", CASES)
def test_f32x3_matches_oracle(ksb, p, layout):
    M, N, _ = O.dims(p)
    B = 300
    K4 = ksgen.k4_uniform(*p, seed=1000 + p[1])
    X = ksgen.x_normal(B, N, seed=0)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_F32X3)
    assert f.plan(B, layout) == "tf32"          # the tcgen05 family
    Yt = run(ksb, f, X, layout)
    rows = np.arange(B) if M * N <= 1 << 22 else np.array([0, 1, 100, 127, 128, 255, 256, 299])
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    err = O.normwise_error(Yt[rows], Yref)
    assert err <= FP32_TOL, err
    assert np.all(np.abs(Yt[rows] - Yref) <= O.envelope_delta(2 * p[2], 2.0 ** -21) * env)
    # FP32-class, ~500x below plain TF32 (~1e-3); measured 0.4-2e-6 (the tensor
    # core's FP32 accumulation is not round-to-nearest, so a bit above FFMA's ~5e-7)
    assert err <= 3e-6, err


@pytest.mark.parametrize("p,layout", [((1, 64, 64, 1), "bsf"), ((2, 48, 32, 3), "bsl"), ((1, 32, 32, 8), "bsf")])
def test_f32x3_integer_bit_exact_with_bias(ksb, p, layout):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_int(*p, seed=2001)
    X = ksgen.x_int(260, N, seed=2000)
    bias = ksgen.x_int(1, M, seed=2003)[0]
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_F32X3)
    Y = run(ksb, f, X, layout, bias=bias)
    assert np.array_equal(Y.astype(np.float64), O.matmul(p, K4, X) + bias[None, :].astype(np.float64))


def test_f32x3_bsf_d6_runs_fp32_cuda_cores(ksb):
    p = (2, 48, 48, 6)
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=5)).set_math(ksb.MATH_F32X3)
    assert f.plan(256, "bsf") == "ffma"
    assert f.plan(256, "bsl") == "tf32"


def test_f32x3_low_halves_packed(ksb):
    p = (2, 16, 24, 3)
    a, b, c, d = p
    K4 = ksgen.k4_uniform(*p, seed=9)
    f = ksb.Factor(*p, K4)
    with pytest.raises(ksb.KSError):
        f.read_packed(3)                          # not allocated before F32X3 is selected
    f.set_math(ksb.MATH_F32X3)
    hi = f.read_packed(2)
    lo = f.read_packed(3)
    tiles = K4.transpose(0, 3, 1, 2).reshape(-1)     # [i][j][k][l]
    assert np.array_equal(hi, O.round_tf32_rna(tiles))
    assert np.array_equal(lo, O.round_tf32_rna((tiles.astype(np.float32) - hi).astype(np.float32)))
    t64 = tiles.astype(np.float64)
    assert np.all(np.abs(hi.astype(np.float64) + lo.astype(np.float64) - t64) <= 2.0 ** -22 * np.abs(t64))


def test_f32x3_many_tiles_per_cta():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_MAXGRID="7", KS_MULTITILE_MATH="f32x3")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "multitile_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
