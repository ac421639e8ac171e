"""Fused multi-factor chain kernel (NEXT-1): same result as the per-factor
launches, bit for bit (identical FMA order), and the oracle contract."""
import numpy as np
import pytest

import ksgen
from ksgen import configs
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    yield ksb
    ksb.set_chain_fusion(True)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def both(ksb, fs, X):
    ksb.set_chain_fusion(True)
    n0 = ksb.launch_count()
    Yf = ksb.chain(fs, to_dev(X))
    torch.cuda.synchronize()
    fused_launches = ksb.launch_count() - n0
    ksb.set_chain_fusion(False)
    Yu = ksb.chain(fs, to_dev(X))
    torch.cuda.synchronize()
    ksb.set_chain_fusion(True)
    return Yf.cpu().numpy(), Yu.cpu().numpy(), fused_launches


CHAINS = {
    "dyadic3": configs.dyadic_patterns(3),
    "dyadic7": configs.dyadic_patterns(7),
    "dyadic12": configs.dyadic_patterns(12),
    "kaleidoscope6": configs.dyadic_patterns(6) + list(reversed(configs.dyadic_patterns(6))),
    "radix4_butterfly": [(1, 4, 4, 16), (4, 4, 4, 4), (16, 4, 4, 1)],
    "square_mixed": [(2, 2, 2, 4), (8, 2, 2, 1), (4, 2, 2, 2), (1, 2, 2, 8)],
}


@pytest.mark.parametrize("name", sorted(CHAINS))
@pytest.mark.parametrize("B", [1, 7, 300])
def test_fused_equals_per_factor_bitwise(ksb, name, B):
    pats = CHAINS[name]
    N = configs.chain_dims(pats)[0]
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    assert ksb.chain_fusion_eligible(fs, B, "bsf")
    X = ksgen.x_normal(B, N, seed=0)
    Yf, Yu, nl = both(ksb, fs, X)
    assert nl == 1
    assert np.array_equal(Yf, Yu)
    assert O.normwise_error(Yf, O.chain(pats, K4s, X)) <= 1e-5


@pytest.mark.parametrize("L", [2, 5, 12])
def test_fused_hadamard_exact(ksb, L):
    pats, K4s = O.hadamard_factors(L)
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_int(33, 2 ** L, seed=2002)
    Yf, _, _ = both(ksb, fs, X)
    assert np.array_equal(Yf.astype(np.float64), O.chain(pats, K4s, X))


def test_fused_fft_full_size_sampled_rows(ksb):
    """configs[1] (B = 8192) through the fused kernel, sampled rows vs the oracle."""
    L, B = configs.FFT_L, configs.FFT_BATCH
    pats = configs.dyadic_patterns(L)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(B, 2 ** L, seed=0)
    Yf, Yu, nl = both(ksb, fs, X)
    assert nl == 1 and np.array_equal(Yf, Yu)
    rows = np.array([0, 5, 4095, 8191])
    assert O.normwise_error(Yf[rows], O.chain(pats, K4s, X, rows=rows)) <= 1e-5


@pytest.mark.parametrize("L,B", [(12, 1036), (12, 1500), (12, 8191), (11, 2072), (11, 2999), (9, 2100)])
def test_fused_register_blocked_rows(ksb, L, B):
    """Enough rows per SM for row groups of 7 / 14 (the register-blocked radix-8
    passes, chunks of 7 rows): bit-identical to the per-factor launches, with a
    ragged last group (rows past B are computed on zero fill and not stored)."""
    pats = configs.dyadic_patterns(L)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(B, 2 ** L, seed=L)
    Yf, Yu, nl = both(ksb, fs, X)
    assert nl == 1 and np.array_equal(Yf, Yu)
    rows = np.array([0, 6, 7, B // 2, B - 1])
    assert O.normwise_error(Yf[rows], O.chain(pats, K4s, X, rows=rows)) <= 1e-5


def test_fused_register_blocked_bias_gelu(ksb):
    """Bias + GELU epilogue after the register-blocked passes (N = 4096, R = 7)."""
    L, B = 12, 1500
    pats = configs.dyadic_patterns(L)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(B, 2 ** L, seed=3)
    bias = ksgen.x_normal(1, 2 ** L, seed=4)[0]
    ksb.set_chain_fusion(True)
    Yf = ksb.chain(fs, to_dev(X), bias=to_dev(bias), act="gelu").cpu().numpy()
    ksb.set_chain_fusion(False)
    Yu = ksb.chain(fs, to_dev(X), bias=to_dev(bias), act="gelu").cpu().numpy()
    ksb.set_chain_fusion(True)
    assert np.array_equal(Yf, Yu)


def test_fusion_eligibility(ksb):
    pats = configs.dyadic_patterns(4)
    fs = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1)) for p in pats]
    assert ksb.chain_fusion_eligible(fs, 64, "bsf")
    assert not ksb.chain_fusion_eligible(fs, 64, "bsl")          # BSF only
    fs[0].set_kernel(ksb.KERNEL_GENERIC)                         # forced kernel -> per factor
    assert not ksb.chain_fusion_eligible(fs, 64, "bsf")
    fs[0].set_kernel(ksb.KERNEL_AUTO)
    ksb.set_chain_fusion(False)
    assert not ksb.chain_fusion_eligible(fs, 64, "bsf")
    ksb.set_chain_fusion(True)
    g = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1)) for p in configs.VIT_UP]
    assert not ksb.chain_fusion_eligible(g, 64, "bsf")           # not square small-block


def test_fused_chain_host_and_trace(ksb):
    pats = configs.dyadic_patterns(10)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(100, 1024, seed=0)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty((100, 1024)).pin_memory()
    ksb.trace_enable(True)
    ksb.chain_host(fs, Xh, Yh)
    torch.cuda.synchronize()
    ms, fam, byts = ksb.trace_read()
    ksb.trace_enable(False)
    assert fam == ["fused_chain"]
    assert byts[0] == 4 * (100 * 1024 * 2 + sum(np.prod(p) for p in pats))
    Yf, Yu, _ = both(ksb, fs, X)
    assert np.array_equal(Yh.numpy(), Yu)


# ------------------------------------------------------- CUDA-graph chains ----
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_chain_graph_replays_bit_identical(ksb, fused, layout):
    """ks_chain_graph: the captured launches replay to exactly
    the direct chain's result, repeatedly, after the input changes, on another
    stream; the replay's kernel count is credited to the launch counter."""
    pats = configs.dyadic_patterns(8) if layout == "bsf" else configs.VIT_DOWN
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    N = configs.chain_dims(pats)[0]
    B = 300
    X = torch.from_numpy(ksgen.x_normal(B, N, seed=0)).cuda()
    if layout == "bsl":
        X = X.t().contiguous()
    ksb.set_chain_fusion(fused)
    try:
        Yd = ksb.chain(fs, X, layout=layout)
        Yg = torch.empty_like(Yd)
        g = ksb.ChainGraph(fs, X, Yg, layout=layout)
        assert g.kernels == (1 if (fused and ksb.chain_fusion_eligible(fs, B, layout)) else len(fs))
        n0 = ksb.launch_count()
        for _ in range(3):
            g.launch()
        torch.cuda.synchronize()
        assert ksb.launch_count() - n0 == 3 * g.kernels
        assert torch.equal(Yg, Yd)
        X.mul_(-0.5)                                  # new contents, same buffer
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g.launch(s)
        s.synchronize()
        Yd2 = ksb.chain(fs, X, layout=layout)
        torch.cuda.synchronize()
        assert torch.equal(Yg, Yd2)
        g.free()
    finally:
        ksb.set_chain_fusion(True)
