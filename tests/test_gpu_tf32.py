"""GPU parity of the TF32 tensor-core kernel (tcgen05) against the oracle.

Contract: normwise error <= 5e-3 against the FP64 oracle on the FP32 inputs
(north star), every element inside the O-6 envelope with u_in = 2^-10; and a
much tighter check against the oracle evaluated on the TF32 operands the
tensor core actually multiplies (K rounded RNA at pack, X truncated by the
hardware): there only FP32 accumulation error remains.  Small-integer data
is exact in TF32, so those runs are bit-exact.
"""
import numpy as np
import pytest

import ksgen
from ksgen import configs
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TF32_TOL = 5e-3


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def run(ksb, f, X_bsf, layout):
    if layout == "bsf":
        Y = ksb.matmul(f, to_dev(X_bsf), layout="bsf")
        torch.cuda.synchronize()
        return Y.cpu().numpy()
    Y = ksb.matmul(f, to_dev(ksgen.to_bsl(X_bsf)), layout="bsl")
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


CASES = [((1, 48, 48, 1), "bsf"), ((1, 64, 64, 1), "bsf"), ((2, 128, 128, 1), "bsf"), ((1, 768, 192, 2), "bsl"),
         ((6, 64, 64, 1), "bsf"), ((6, 64, 256, 1), "bsf"), ((64, 64, 64, 1), "bsf"), ((1, 256, 64, 16), "bsl"),
         ((1, 48, 48, 64), "bsl"), ((3, 96, 96, 4), "bsl"), ((1, 128, 128, 3), "bsl"), ((2, 16, 24, 3), "bsl"),
         ((1, 16, 16, 1), "bsf"), ((1, 320, 40, 2), "bsl"), ((2, 96, 96, 1), "bsl"), ((6, 64, 64, 1), "bsl"),
         # BSF, d > 1: J = d contiguous 2-D box (d <= 8), J = 8 / 4 3-D gather (d > 8)
         ((1, 64, 64, 4), "bsf"), ((2, 48, 48, 16), "bsf"), ((1, 128, 128, 8), "bsf"), ((3, 96, 96, 4), "bsf"),
         ((1, 64, 256, 16), "bsf"), ((1, 256, 64, 16), "bsf"), ((2, 16, 32, 12), "bsf"),
         ((1, 768, 192, 2), "bsf"), ((1, 128, 128, 3), "bsf"), ((2, 48, 48, 6), "bsf"), ((1, 96, 96, 6), "bsf"),
         ((1, 128, 128, 12), "bsf"), ((1, 64, 64, 32), "bsf"), ((2, 96, 96, 16), "bsf"), ((1, 320, 48, 2), "bsf"),
         ((3, 48, 64, 2), "bsf"), ((1, 112, 32, 3), "bsf"), ((2, 64, 48, 8), "bsf")]


@pytest.mark.parametrize("p,layout", CASES)
def test_tf32_matches_oracle(ksb, p, layout):
    M, N, _ = O.dims(p)
    B = 300
    K4 = ksgen.k4_uniform(*p, seed=1000 + p[1])
    X = ksgen.x_normal(B, N, seed=0)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    assert f.plan(B, layout) == "tf32"
    Yt = run(ksb, f, X, layout)
    rows = np.arange(B) if M * N <= 1 << 22 else np.array([0, 1, 100, 127, 128, 255, 256, 299])
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    err = O.normwise_error(Yt[rows], Yref)
    assert err <= TF32_TOL, err
    assert np.all(np.abs(Yt[rows] - Yref) <= O.envelope_delta(p[2], 2.0 ** -10) * env)
    # against the oracle on the operands the tensor core sees
    Ytf = O.matmul(p, O.round_tf32_rna(K4), O.truncate_tf32(X), rows=rows, want_env=False)
    Yabs = O.matmul(p, np.abs(O.round_tf32_rna(K4)), np.abs(O.truncate_tf32(X)), rows=rows)
    assert np.all(np.abs(Yt[rows] - Ytf) <= O.envelope_delta(p[2], 0.0) * Yabs + 1e-30)


@pytest.mark.parametrize("p,layout", [((1, 64, 64, 1), "bsf"), ((2, 48, 32, 3), "bsl"), ((64, 64, 64, 1), "bsf"),
                                      ((1, 256, 64, 16), "bsl"), ((2, 48, 32, 3), "bsf"), ((1, 128, 64, 6), "bsf"),
                                      ((1, 64, 64, 16), "bsf"), ((1, 128, 128, 12), "bsf")])
def test_tf32_integer_bit_exact(ksb, p, layout):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_int(*p, seed=2001)
    X = ksgen.x_int(260, N, seed=2000)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    assert np.array_equal(run(ksb, f, X, layout).astype(np.float64), O.matmul(p, K4, X))


@pytest.mark.parametrize("B", [4, 8, 124, 132])
def test_tf32_ragged_batches(ksb, B):
    p = (2, 64, 96, 2)
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=3)
    X = ksgen.x_normal(B, N, seed=4)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Yt = run(ksb, f, X, "bsl")
    assert O.normwise_error(Yt, O.matmul(p, K4, X)) <= TF32_TOL


@pytest.mark.parametrize("layout", ["bsl", "bsf"])
@pytest.mark.parametrize("name", ["VIT_UP", "VIT_DOWN", "GPT2_DOWN", "GPT2_UP"])
def test_tf32_model_chains(ksb, name, layout):
    pats = getattr(configs, name)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = configs.chain_dims(pats)[0]
    B = 256
    X = ksgen.x_normal(B, N, seed=0)
    fs = [ksb.Factor(*p, k).set_math(ksb.MATH_TF32) for p, k in zip(pats, K4s)]
    assert all(f.plan(B, layout) == "tf32" for f in fs)
    Y = ksb.chain(fs, to_dev(ksgen.to_bsl(X) if layout == "bsl" else X), layout=layout)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy().T if layout == "bsl" else Y.cpu().numpy()
    err = O.normwise_error(Yh, O.chain(pats, K4s, X))
    assert err <= TF32_TOL, err


@pytest.mark.parametrize("p,layout", [((1, 128, 128, 64), "bsl"), ((4, 64, 64, 16), "bsl"), ((1, 96, 96, 1), "bsl"),
                                      ((1, 128, 128, 64), "bsf"), ((4, 64, 64, 16), "bsf"), ((1, 96, 96, 1), "bsf"),
                                      ((1, 128, 128, 3), "bsf"), ((1, 96, 96, 6), "bsf"), ((1, 48, 48, 2), "bsf"),
                                      ((3, 64, 64, 16), "bsf")])
def test_tf32_sweep_full_size_sampled_rows(ksb, p, layout):
    """configs[2] at B = 25088, TF32, both layouts, in bench's launch configuration."""
    B = configs.SWEEP_BATCH
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=1000)
    X = ksgen.x_normal(B, N, seed=0)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    assert f.plan(B, layout) == "tf32"
    Yg = run(ksb, f, X, layout)
    rows = np.array([0, 1, 127, 128, 12543, 25087] + list(np.random.default_rng(3).integers(0, B, 4)))
    Yref = O.matmul(p, K4, X, rows=rows)
    assert O.normwise_error(Yg[rows], Yref) <= TF32_TOL


@pytest.mark.parametrize("grid", [1, 2, 3])
def test_tf32_many_tiles_per_cta(grid):
    """Persistent kernels with a capped grid (KS_TF32_MAXGRID) so every CTA runs
    several tiles: exercises the mbarrier ring / TMEM double-buffer wrap-around
    (a missing proxy fence once showed up only here)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_MAXGRID=str(grid))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "multitile_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
