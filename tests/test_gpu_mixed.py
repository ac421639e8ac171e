"""Mixed-layout calls (ks_matmul_io) and mixed-layout chain intermediates
against the oracle.

A BSL array is the transpose of the BSF one (PAPER.md:86 / 631-641), so a
BSF-in / BSL-out product is Y^T of the same Y = X K^T: the oracle computes Y
from the BSF X and the test transposes what the kernel wrote.  TF32 calls use
the contract of tests/test_gpu_tf32.py (normwise <= 5e-3 against the FP64
oracle, every element inside the O-6 envelope with u_in = 2^-10, and the much
tighter envelope against the oracle on the TF32 operands); FP32 calls run the
generic kernel (normwise <= 1e-5); small-integer data is exact in TF32 and FP32
so those runs are bit-exact.  The library's trace records show which family ran.
"""
import numpy as np
import pytest

import ksgen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TF32_TOL = 5e-3
FAMILY_TF32, FAMILY_GENERIC = "tf32", "generic"


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def run_io(ksb, f, X_bsf, xl, yl):
    """Y (BSF numpy, B x M) of ks_matmul_io with X given in xl and Y written in yl,
    and the kernel families the call launched."""
    Xd = to_dev(X_bsf if xl == "bsf" else ksgen.to_bsl(X_bsf))
    ksb.trace_read()                       # drain
    ksb.trace_enable(True)
    Y = ksb.matmul_io(f, Xd, xl, y_layout=yl)
    torch.cuda.synchronize()
    _, fam, _ = ksb.trace_read()
    ksb.trace_enable(False)
    Y = Y.cpu().numpy()
    return (Y if yl == "bsf" else Y.T), list(fam)


# (pattern, direction): d = 1 (ks_tf32_kernel with the other epilogue), BSF in with
# J = d contiguous boxes and J = 4 / 8 gathers, BSL in with J = d, 8, 4; wide b
# (several output chunks), ragged batch tiles (B = 300).
CASES = [((6, 64, 64, 1), "fl"), ((64, 64, 64, 1), "fl"), ((6, 64, 256, 1), "fl"), ((1, 128, 128, 1), "lf"),
         ((64, 64, 64, 1), "lf"), ((2, 96, 96, 1), "lf"), ((1, 48, 48, 1), "lf"),
         ((1, 768, 192, 2), "fl"), ((1, 128, 128, 3), "fl"), ((1, 256, 64, 16), "fl"), ((1, 64, 256, 16), "fl"),
         ((2, 48, 48, 6), "fl"), ((1, 128, 128, 12), "fl"), ((1, 64, 64, 32), "fl"), ((3, 96, 96, 4), "fl"),
         ((1, 768, 192, 2), "lf"), ((1, 128, 128, 3), "lf"), ((1, 64, 256, 16), "lf"), ((1, 256, 64, 16), "lf"),
         ((2, 48, 48, 6), "lf"), ((1, 128, 128, 12), "lf"), ((2, 64, 48, 8), "lf"), ((3, 96, 96, 4), "lf"),
         ((1, 48, 48, 64), "lf"), ((2, 16, 32, 12), "lf"), ((1, 320, 48, 2), "lf"), ((1, 112, 32, 3), "lf")]
DIRS = {"fl": ("bsf", "bsl"), "lf": ("bsl", "bsf")}


@pytest.mark.parametrize("p,dirn", CASES)
def test_tf32_mixed_matches_oracle(ksb, p, dirn):
    xl, yl = DIRS[dirn]
    M, N, _ = O.dims(p)
    B = 300
    K4 = ksgen.k4_uniform(*p, seed=2000 + p[1])
    X = ksgen.x_normal(B, N, seed=3)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Yt, fam = run_io(ksb, f, X, xl, yl)
    assert fam == [FAMILY_TF32], fam
    rows = np.arange(B) if M * N <= 1 << 22 else np.array([0, 1, 100, 127, 128, 255, 256, 299])
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    err = O.normwise_error(Yt[rows], Yref)
    assert err <= TF32_TOL, err
    assert np.all(np.abs(Yt[rows] - Yref) <= O.envelope_delta(p[2], 2.0 ** -10) * env)
    Ytf = O.matmul(p, O.round_tf32_rna(K4), O.truncate_tf32(X), rows=rows)
    Yabs = O.matmul(p, np.abs(O.round_tf32_rna(K4)), np.abs(O.truncate_tf32(X)), rows=rows)
    assert np.all(np.abs(Yt[rows] - Ytf) <= O.envelope_delta(p[2], 0.0) * Yabs + 1e-30)


@pytest.mark.parametrize("p,dirn", [((6, 64, 64, 1), "fl"), ((1, 256, 64, 16), "fl"), ((1, 64, 256, 16), "lf"),
                                    ((2, 48, 48, 6), "lf"), ((1, 768, 192, 2), "lf"), ((64, 64, 64, 1), "lf")])
def test_tf32_mixed_integer_bit_exact(ksb, p, dirn):
    xl, yl = DIRS[dirn]
    M, N, _ = O.dims(p)
    B = 260
    K4 = ksgen.k4_int(*p, seed=7)
    X = ksgen.x_int(B, N, seed=8)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Yt, fam = run_io(ksb, f, X, xl, yl)
    assert fam == [FAMILY_TF32]
    rows = np.array([0, 1, 127, 128, 200, 259])
    assert np.array_equal(Yt[rows], O.matmul(p, K4, X, rows=rows).astype(np.float32))


@pytest.mark.parametrize("p,dirn,B", [((2, 4, 4, 2), "fl", 8), ((2, 4, 4, 2), "lf", 8), ((3, 5, 7, 2), "fl", 33),
                                      ((1, 64, 64, 4), "lf", 301), ((6, 64, 64, 1), "fl", 100)])
def test_fp32_mixed_generic_matches_oracle(ksb, p, dirn, B):
    xl, yl = DIRS[dirn]
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=5)
    X = ksgen.x_normal(B, N, seed=6)
    f = ksb.Factor(*p, K4)
    Yt, fam = run_io(ksb, f, X, xl, yl)
    assert fam == [FAMILY_GENERIC]
    assert O.normwise_error(Yt, O.matmul(p, K4, X)) <= 1e-5


def test_tf32_bsl_in_ragged_batch_falls_back(ksb):
    """BSL in needs B % 4 == 0 for the TMA view; B = 302 runs the generic kernel."""
    p = (1, 64, 64, 4)
    K4 = ksgen.k4_uniform(*p, seed=9)
    X = ksgen.x_normal(302, 256, seed=1)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Yt, fam = run_io(ksb, f, X, "bsl", "bsf")
    assert fam == [FAMILY_GENERIC]
    assert O.normwise_error(Yt, O.matmul(p, K4, X)) <= 1e-5


MODEL_CHAINS = {       # mixed plans: an intermediate next to a factor with d > 8 goes BSL
    "gpt2_down": [(1, 64, 256, 16), (64, 64, 64, 1)],
    "gpt2_up": [(64, 64, 64, 1), (1, 256, 64, 16)],
    "three": [(1, 64, 64, 12), (12, 64, 64, 1), (1, 48, 64, 16)],
    "wide_j": [(1, 64, 128, 16), (4, 64, 64, 8)],
}


@pytest.mark.parametrize("name", sorted(MODEL_CHAINS))
def test_chain_mixed_intermediates_match_oracle(ksb, name):
    pats = MODEL_CHAINS[name]
    K4s = [ksgen.k4_uniform(*q, seed=300 + l) for l, q in enumerate(pats)]
    fs = [ksb.Factor(*q, k).set_math(ksb.MATH_TF32) for q, k in zip(pats, K4s)]
    B = 260
    N = O.dims(pats[-1])[1]
    X = ksgen.x_normal(B, N, seed=4)
    mixed, lay = ksb.chain_layouts(fs, B)
    assert mixed and lay[0] == lay[-1] == "bsf" and lay[1] == "bsl", lay
    if name == "three":
        assert lay == ["bsf", "bsl", "bsl", "bsf"]
    Xd = to_dev(X)
    ksb.set_chain_fusion(False)
    try:
        Ym = ksb.chain(fs, Xd).cpu().numpy()
        ksb.set_chain_mixed_layouts(False)
        assert ksb.chain_layouts(fs, B)[0] is False
        Yu = ksb.chain(fs, Xd).cpu().numpy()
    finally:
        ksb.set_chain_mixed_layouts(True)
        ksb.set_chain_fusion(True)
    rows = np.array([0, 1, 127, 128, 200, 259])
    Yref = O.chain(pats, K4s, X, rows=rows)
    for Y in (Ym, Yu):
        assert O.normwise_error(Y[rows], Yref) <= TF32_TOL
    # the same arithmetic in another layout: the two plans agree far inside the contract
    assert O.normwise_error(Ym, Yu) <= 1e-4
    if len(pats) == 2:       # the chain ran the planned calls: bit-identical to them made by hand
        T = ksb.matmul_io(fs[1], Xd, "bsf", y_layout="bsl")
        Yh = ksb.matmul_io(fs[0], T, "bsl", y_layout="bsf")
        assert np.array_equal(Ym, Yh.cpu().numpy())


def test_chain_layouts_uniform_cases(ksb):
    pats = [(2, 64, 64, 1), (2, 64, 64, 1)]
    fs = [ksb.Factor(*q, ksgen.k4_uniform(*q, seed=1)).set_math(ksb.MATH_TF32) for q in pats]
    assert ksb.chain_layouts(fs, 256) == (False, ["bsf"] * 3)          # all d = 1
    for pats in ([(1, 768, 192, 2), (6, 64, 64, 1)], [(1, 128, 128, 3), (6, 64, 256, 1)]):   # ViT-S: d <= 8
        fs = [ksb.Factor(*q, ksgen.k4_uniform(*q, seed=1)).set_math(ksb.MATH_TF32) for q in pats]
        assert ksb.chain_layouts(fs, 256) == (False, ["bsf"] * 3)
    pats = MODEL_CHAINS["gpt2_up"]
    fs = [ksb.Factor(*q, ksgen.k4_uniform(*q, seed=1)) for q in pats]  # FP32 math: no mixed plan
    assert ksb.chain_layouts(fs, 256)[0] is False
    fs = [f.set_math(ksb.MATH_TF32) for f in fs]
    assert ksb.chain_layouts(fs, 256, "bsl") == (False, ["bsl"] * 3)   # caller chose BSL
    assert ksb.chain_layouts(fs, 258)[0] is False                      # BSL in needs B % 4 == 0


def test_chain_graph_replays_mixed_plan_bit_identical(ksb):
    """ks_chain_graph captures the mixed-layout plan (BSL intermediate) and its
    replay equals the direct chain bit for bit."""
    pats = MODEL_CHAINS["gpt2_up"]
    K4s = [ksgen.k4_uniform(*q, seed=400 + l) for l, q in enumerate(pats)]
    fs = [ksb.Factor(*q, k).set_math(ksb.MATH_TF32) for q, k in zip(pats, K4s)]
    B = 512
    X = to_dev(ksgen.x_normal(B, O.dims(pats[-1])[1], seed=9))
    assert ksb.chain_layouts(fs, B)[0]
    Y = ksb.chain(fs, X)
    Yg = torch.empty_like(Y)
    g = ksb.ChainGraph(fs, X, Yg)
    g.launch()
    torch.cuda.synchronize()
    assert torch.equal(Yg, Y)
    g.free()


@pytest.mark.parametrize("grid", [1, 3])
def test_tf32_mixed_many_tiles_per_cta(grid):
    """Mixed-layout J-kernels (MN-major A for BSL in, TMA-store epilogue) with a capped
    persistent grid (KS_TF32_MAXGRID): every CTA runs several tiles, so the operand
    ring, the accumulator double buffer and the store buffers all wrap."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_MAXGRID=str(grid), KS_MULTITILE_MATH="tf32mixed")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "multitile_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("p,dirn,B", [((1, 64, 256, 16), "lf", 65536), ((1, 256, 64, 16), "fl", 65536),
                                      ((1, 128, 128, 16), "lf", 25088), ((64, 64, 64, 1), "lf", 65536)])
def test_tf32_mixed_full_size_sampled_rows(ksb, p, dirn, B):
    """configs[4]-size mixed-layout calls in the launch configuration the chains use
    (MN-major BSL-in J-kernel, J = 4 BSF-in/BSL-out, the d = 1 TMA-store epilogue):
    sampled rows against the oracle, inside the per-element envelope."""
    xl, yl = DIRS[dirn]
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=4000 + p[1])
    X = ksgen.x_normal(B, N, seed=11)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Yt, fam = run_io(ksb, f, X, xl, yl)
    assert fam == [FAMILY_TF32], fam
    rows = np.array([0, 1, 127, 128, B // 2 + 3, B - 129, B - 1])
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    assert O.normwise_error(Yt[rows], Yref) <= TF32_TOL
    assert np.all(np.abs(Yt[rows] - Yref) <= O.envelope_delta(p[2], 2.0 ** -10) * env)
