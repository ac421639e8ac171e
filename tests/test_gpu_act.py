"""Epilogue activation (NEXT-2, "+ GELU" of the FFN row):
Y = gelu(X K^T + bias) fused into the epilogue of every kernel family, and of
the last factor of a chain (per-factor, mixed-layout and fused), against the
FP64 oracle: oracle.gelu(oracle.matmul(...) + bias).

GELU's derivative is bounded (|gelu'| <= 1.13), so the linear part's error
carries over almost unchanged and FP32 erff adds a few ulp: the contracts of
the plain calls hold (FP32 normwise <= 1e-5, TF32 <= 5e-3, half <= 3u against
the oracle on the half inputs)."""
import numpy as np
import pytest

import ksgen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


def _ref(p, K4, X, bias):
    return O.gelu(O.matmul(p, K4, X) + bias.astype(np.float64))


# (pattern, layout, B, setup) -- setup picks the kernel family
FP32_CASES = [
    ((3, 5, 7, 2), "bsf", 33, "generic"), ((3, 5, 7, 2), "bsl", 33, "generic"),
    ((8, 2, 2, 16), "bsf", 100, "auto"), ((8, 4, 4, 8), "bsl", 128, "auto"),          # stream
    ((2, 64, 64, 2), "bsf", 24, "auto"),                                                # split-c (B <= 64)
    ((2, 64, 64, 4), "bsf", 300, "regstaged"), ((2, 80, 64, 1), "bsl", 300, "auto"),    # register-staged
    ((6, 64, 64, 1), "bsf", 300, "auto"), ((4, 128, 128, 2), "bsl", 300, "auto"),       # warp-specialised
    ((2, 64, 64, 8), "bsf", 300, "wsg"), ((2, 64, 64, 8), "bsf", 300, "wsl"), ((1, 96, 64, 3), "bsf", 300, "auto"),
]


def _setup(ksb, f, setup):
    from paper_2405_15013_b200 import ks
    if setup == "generic":
        f.set_kernel(ksb.KERNEL_GENERIC)
    elif setup == "regstaged":
        f.set_knobs(0)
    elif setup == "wsg":
        f.set_knobs(ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32)
    elif setup == "wsl":
        f.set_knobs(ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32 | ks.KNOB_FFMA_WSL)


@pytest.mark.parametrize("p,layout,B,setup", FP32_CASES)
def test_fp32_families_gelu(ksb, p, layout, B, setup):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=31)
    X = ksgen.x_normal(B, N, seed=32)
    bias = np.random.default_rng(33).standard_normal(M).astype(np.float32)
    f = ksb.Factor(*p, K4)
    _setup(ksb, f, setup)
    Xd = torch.from_numpy(X if layout == "bsf" else ksgen.to_bsl(X)).cuda()
    Y = ksb.matmul(f, Xd, layout=layout, bias=torch.from_numpy(bias).cuda(), act="gelu")
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    assert O.normwise_error(Yh, _ref(p, K4, X, bias)) <= 1e-5


TF32_CASES = [((2, 128, 64, 1), "bsf", {}), ((1, 64, 64, 4), "bsl", {}), ((1, 48, 48, 2), "bsl", {"mn": True}),
              ((2, 64, 64, 4), "bsf", {}), ((1, 128, 128, 3), "bsf", {"densify": True}), ((1, 64, 64, 16), "bsf", {}),
              ((2, 96, 64, 1), "bsl", {"v2": True})]


@pytest.mark.parametrize("p,layout,opt", TF32_CASES)
def test_tf32_families_gelu(ksb, p, layout, opt):
    from paper_2405_15013_b200 import ks
    M, N, _ = O.dims(p)
    B = 300 if layout == "bsf" else 296
    K4 = ksgen.k4_uniform(*p, seed=34)
    X = ksgen.x_normal(B, N, seed=35)
    bias = np.random.default_rng(36).standard_normal(M).astype(np.float32)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    if opt:
        knobs, _ = f.plan_knobs(B, layout)
        if opt.get("mn"):
            knobs |= ks.KNOB_TF32_MN
        if opt.get("densify"):
            knobs |= ks.KNOB_DENSIFY
        if opt.get("v2"):
            knobs |= ks.KNOB_TF32_V2
        f.set_knobs(knobs)
    assert f.plan(B, layout) == "tf32"
    Xd = torch.from_numpy(X if layout == "bsf" else ksgen.to_bsl(X)).cuda()
    Y = ksb.matmul(f, Xd, layout=layout, bias=torch.from_numpy(bias).cuda(), act="gelu")
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    assert O.normwise_error(Yh, _ref(p, K4, X, bias)) <= 5e-3


@pytest.mark.parametrize("dt", ["bf16", "f16"])
@pytest.mark.parametrize("p,layout", [((2, 64, 64, 1), "bsf"), ((2, 64, 64, 4), "bsf"), ((1, 64, 64, 2), "bsl")])
def test_half_gelu(ksb, dt, p, layout):
    tdt = torch.bfloat16 if dt == "bf16" else torch.float16
    u = 2.0 ** -8 if dt == "bf16" else 2.0 ** -11
    M, N, _ = O.dims(p)
    B = 256
    K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=37)).to(tdt)
    X = torch.from_numpy(ksgen.x_normal(B, N, seed=38)).to(tdt)
    bias = torch.from_numpy(np.random.default_rng(39).standard_normal(M).astype(np.float32)).to(tdt)
    f = ksb.Factor(*p, K4.cuda())
    Xd = (X if layout == "bsf" else X.t().contiguous()).cuda()
    Y = ksb.matmul(f, Xd, layout=layout, bias=bias.cuda(), act="gelu")
    torch.cuda.synchronize()
    Yh = (Y if layout == "bsf" else Y.t()).float().cpu().numpy()
    ref = _ref(p, K4.float().numpy(), X.float().numpy(), bias.float().numpy())
    assert O.normwise_error(Yh, ref) <= 3 * u


CHAINS = {"fft_fused": [(1, 2, 2, 32), (2, 2, 2, 16), (4, 2, 2, 8), (8, 2, 2, 4), (16, 2, 2, 2), (32, 2, 2, 1)],
          "vit_up": [(1, 768, 192, 2), (6, 64, 64, 1)], "gpt2_up_tf32": [(64, 64, 64, 1), (1, 256, 64, 16)]}


@pytest.mark.parametrize("name", sorted(CHAINS))
def test_chain_gelu_after_last_factor(ksb, name):
    pats = CHAINS[name]
    K4s = [ksgen.k4_uniform(*q, seed=40 + l) for l, q in enumerate(pats)]
    fs = [ksb.Factor(*q, k) for q, k in zip(pats, K4s)]
    tf32 = name.endswith("tf32")
    if tf32:
        fs = [f.set_math(ksb.MATH_TF32) for f in fs]
        assert ksb.chain_layouts(fs, 256)[0]                      # mixed-layout plan
    if name == "fft_fused":
        assert ksb.chain_fusion_eligible(fs, 256)
    M = O.dims(pats[0])[0]
    N = O.dims(pats[-1])[1]
    X = ksgen.x_normal(256, N, seed=41)
    bias = np.random.default_rng(42).standard_normal(M).astype(np.float32)
    Y = ksb.chain(fs, torch.from_numpy(X).cuda(), bias=torch.from_numpy(bias).cuda(), act="gelu")
    torch.cuda.synchronize()
    ref = O.gelu(O.chain(pats, K4s, X) + bias.astype(np.float64))
    assert O.normwise_error(Y.cpu().numpy(), ref) <= (5e-3 if tf32 else 1e-5)


def test_kslinear_gelu_and_bad_activation(ksb):
    pats = [(1, 768, 192, 2), (6, 64, 64, 1)]
    g = torch.Generator().manual_seed(5)
    lin = ksb.KSLinear(pats, bias=True, activation="gelu", generator=g)
    plain = ksb.KSLinear(pats, weights=[f.read_packed(0).reshape(p) for f, p in zip(lin.factors, pats)],
                         bias=lin.bias.detach().clone())
    x = torch.randn(3, 7, 384, device="cuda")
    y = lin(x)
    y0 = plain(x)
    torch.cuda.synchronize()
    ref = O.gelu(y0.double().cpu().numpy())
    assert O.normwise_error(y.cpu().numpy(), ref) <= 1e-5
    with pytest.raises(ValueError):
        ksb.KSLinear(pats, activation="relu6")
    f = lin.factors[0]
    with pytest.raises(ValueError):
        ksb.matmul(f, torch.zeros(4, f.N, device="cuda"), act="swish")
