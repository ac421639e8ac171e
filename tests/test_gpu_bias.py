"""NEXT-2: bias fused into the last factor's epilogue, and the KSLinear module."""
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


FAMILIES = [((2, 3, 2, 3), "generic", "fp32"), ((4, 2, 2, 8), "stream", "fp32"), ((2, 64, 48, 4), "ffma", "fp32"),
            ((1, 64, 48, 2), "ffma", "fp32"), ((3, 48, 64, 1), "ffma", "fp32"), ((1, 96, 64, 3), "ffma", "fp32"),
            ((1, 64, 64, 1), "tf32", "tf32"), ((2, 48, 48, 8), "tf32", "tf32"), ((1, 128, 128, 3), "tf32", "tf32"),
            ((1, 64, 48, 16), "tf32", "tf32"), ((1, 128, 128, 12), "tf32", "tf32")]


@pytest.mark.parametrize("p,family,math", FAMILIES)
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_matmul_bias(ksb, p, family, math, layout):
    M, N, _ = O.dims(p)
    B = 260
    K4 = ksgen.k4_uniform(*p, seed=5)
    X = ksgen.x_normal(B, N, seed=6)
    bias = ksgen.x_normal(1, M, seed=7)[0]
    f = ksb.Factor(*p, K4)
    if math == "tf32":
        f.set_math(ksb.MATH_TF32)
    plan = f.plan(B, layout)
    assert plan == family, plan
    Xd = to_dev(X if layout == "bsf" else ksgen.to_bsl(X))
    Y = ksb.matmul(f, Xd, layout=layout, bias=to_dev(bias))
    Y0 = ksb.matmul(f, Xd, layout=layout)
    torch.cuda.synchronize()
    Yb, Yn = Y.cpu().numpy(), Y0.cpu().numpy()
    if layout == "bsl":
        Yb, Yn = Yb.T, Yn.T
    # bias is one FP32 add after the reduction
    assert np.array_equal(Yb, (Yn + bias[None, :]).astype(np.float32))
    tol = 1e-5 if math == "fp32" else 5e-3
    assert O.normwise_error(Yb, O.matmul(p, K4, X) + bias[None, :]) <= tol


@pytest.mark.parametrize("fused", [True, False])
def test_chain_bias_fused_and_per_factor(ksb, fused):
    pats = configs.dyadic_patterns(9)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(77, 512, seed=0)
    bias = ksgen.x_normal(1, 512, seed=9)[0]
    ksb.set_chain_fusion(fused)
    Y = ksb.chain(fs, to_dev(X), bias=to_dev(bias))
    torch.cuda.synchronize()
    ksb.set_chain_fusion(True)
    assert O.normwise_error(Y.cpu().numpy(), O.chain(pats, K4s, X) + bias[None, :]) <= 1e-5


@pytest.mark.parametrize("name,layout", [("VIT_UP", "bsf"), ("VIT_DOWN", "bsl"), ("GPT2_DOWN", "bsf")])
def test_kslinear_module(ksb, name, layout):
    pats = getattr(configs, name)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    lin = ksb.KSLinear(pats, weights=K4s, bias=True, layout=layout)
    N, M = lin.in_features, lin.out_features
    assert (N, M) == (configs.chain_dims(pats)[0], configs.chain_dims(pats)[-1])
    X = ksgen.x_normal(2 * 37, N, seed=3)
    bias = lin.bias.detach().cpu().numpy()
    ref = O.chain(pats, K4s, X) + bias[None, :]
    if layout == "bsf":
        y = lin(to_dev(X).reshape(2, 37, N))
        assert tuple(y.shape) == (2, 37, M)
        got = y.reshape(-1, M).cpu().numpy()
    else:
        got = lin(to_dev(ksgen.to_bsl(X))).cpu().numpy().T
    assert O.normwise_error(got, ref) <= 1e-5


def test_kslinear_rejects_unchainable(ksb):
    with pytest.raises(ValueError):
        ksb.KSLinear([(1, 4, 4, 1), (1, 3, 3, 1)])
