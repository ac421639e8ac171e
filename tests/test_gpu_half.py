"""NEXT-3: half-precision handles (BF16 / FP16 operands on tcgen05 kind::f16,
FP32 accumulation, output rounded to nearest-even) against the FP64 oracle.

Products of two half values are exact in FP32 and the oracle is evaluated on
the exact half inputs, so the only errors are FP32 accumulation (envelope
gamma_{2c}) and the final rounding of Y to the half format (relative u_out =
2^-8 for BF16, 2^-11 for FP16): |Y^ - Y| <= u_out |Y| + (1 + u_out) gamma |X||K|.
"""
import numpy as np
import pytest

import ksgen
from ksgen import configs
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U_OUT = {"bf16": 2.0 ** -8, "f16": 2.0 ** -11}     # unit roundoff: 8- and 11-bit significands


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


def tdt(name):
    return torch.bfloat16 if name == "bf16" else torch.float16


def half_inputs(p, B, name, seed=0):
    M, N, _ = O.dims(p)
    K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=1000 + seed)).to(tdt(name))
    X = torch.from_numpy(ksgen.x_normal(B, N, seed=seed)).to(tdt(name))
    return K4, X, K4.float().numpy(), X.float().numpy()


def check(Yg, p, K4f, Xf, name, L=1):
    Yref, env = O.matmul(p, K4f, Xf, want_env=True)
    u = U_OUT[name]
    bound = u * np.abs(Yref) + (1 + u) * O.envelope_delta(p[2], 0.0) * env
    assert np.all(np.abs(Yg - Yref) <= bound + 1e-30)
    assert O.normwise_error(Yg, Yref) <= 2 * u


CASES = [((1, 64, 64, 1), "bsf"), ((6, 64, 256, 1), "bsf"), ((2, 128, 128, 1), "bsf"), ((1, 48, 48, 4), "bsl"),
         ((1, 768, 192, 2), "bsl"), ((3, 96, 96, 3), "bsl"), ((2, 16, 32, 2), "bsl"),
         # BSF d > 1: J-column gather, J = d (2-D box) or J = 8 (3-D box)
         ((2, 128, 64, 2), "bsf"), ((1, 48, 48, 3), "bsf"), ((3, 64, 64, 4), "bsf"), ((1, 96, 96, 6), "bsf"),
         ((1, 64, 64, 8), "bsf"), ((1, 32, 48, 16), "bsf"), ((2, 16, 16, 24), "bsf"),
         # d % 4 == 0, d % 8 != 0: J = 4 out of an 8-wide box, per-row 8-byte stores
         ((1, 48, 64, 12), "bsf"), ((2, 64, 64, 12), "bsf"), ((1, 32, 32, 20), "bsf"),
         # c % 32 == 0, J <= 4: 32 l per stage (SWIZZLE_64B operand rows)
         ((2, 64, 96, 3), "bsf"), ((1, 96, 64, 2), "bsf"), ((2, 128, 128, 4), "bsf"), ((1, 32, 64, 4), "bsf")]


@pytest.mark.parametrize("name", ["bf16", "f16"])
@pytest.mark.parametrize("p,layout", CASES)
def test_half_tensor_core(ksb, name, p, layout):
    B = 264
    K4, X, K4f, Xf = half_inputs(p, B, name)
    f = ksb.Factor(*p, K4)
    assert f.plan(B, layout) == "tf32"           # the tcgen05 family (kind::f16 here)
    Xd = (X if layout == "bsf" else X.t().contiguous()).cuda()
    Y = ksb.matmul(f, Xd, layout=layout)
    torch.cuda.synchronize()
    assert Y.dtype == tdt(name)
    Yg = Y.float().cpu().numpy()
    check(Yg if layout == "bsf" else Yg.T, p, K4f, Xf, name)


@pytest.mark.parametrize("name", ["bf16", "f16"])
@pytest.mark.parametrize("p,layout", [((2, 4, 4, 2), "bsf"), ((1, 64, 64, 5), "bsf"), ((1, 48, 64, 10), "bsf"),
                                      ((2, 3, 5, 7), "bsl")])
def test_half_generic(ksb, name, p, layout):
    B = 33
    K4, X, K4f, Xf = half_inputs(p, B, name)
    f = ksb.Factor(*p, K4)
    assert f.plan(B, layout) == "generic"
    Xd = (X if layout == "bsf" else X.t().contiguous()).cuda()
    Yg = ksb.matmul(f, Xd, layout=layout).float().cpu().numpy()
    check(Yg if layout == "bsf" else Yg.T, p, K4f, Xf, name)


@pytest.mark.parametrize("name", ["bf16", "f16"])
@pytest.mark.parametrize("p,layout", [((2, 64, 64, 1), "bsf"), ((1, 32, 32, 8), "bsf"), ((2, 48, 48, 3), "bsf"),
                                      ((1, 64, 32, 12), "bsf"),
                                      ((2, 32, 32, 4), "bsl")])
def test_half_integer_exact_and_bias(ksb, name, p, layout):
    M, N, _ = O.dims(p)
    B = 200
    K4 = torch.from_numpy(ksgen.k4_int(*p, seed=2001)).to(tdt(name))
    X = torch.from_numpy(ksgen.x_int(B, N, seed=2000)).to(tdt(name))
    bias = torch.from_numpy(ksgen.x_int(1, M, seed=2003)[0]).to(tdt(name))
    f = ksb.Factor(*p, K4)
    assert f.plan(B, layout) == "tf32"
    Xd = (X if layout == "bsf" else X.t().contiguous()).cuda()
    Y = ksb.matmul(f, Xd, bias=bias.cuda(), layout=layout).float().cpu().numpy()
    Y = Y if layout == "bsf" else Y.T
    ref = O.matmul(p, K4.float().numpy(), X.float().numpy()) + bias.float().numpy()[None, :]
    assert np.abs(ref).max() <= 256        # integers <= 2^8: exact in BF16 and FP16, so bit-exact
    assert np.array_equal(Y.astype(np.float64), ref)


@pytest.mark.parametrize("name", ["bf16", "f16"])
def test_half_chain(ksb, name):
    pats = configs.GPT2_DOWN
    B = 128
    Ks = [torch.from_numpy(ksgen.k4_uniform(*p, seed=1000 + l)).to(tdt(name)) for l, p in enumerate(pats, 1)]
    X = torch.from_numpy(ksgen.x_normal(B, configs.chain_dims(pats)[0], seed=0)).to(tdt(name))
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, Ks)]
    Y = ksb.chain(fs, X.cuda()).float().cpu().numpy()
    ref = O.chain(pats, [k.float().numpy() for k in Ks], X.float().numpy())
    assert O.normwise_error(Y, ref) <= 4 * U_OUT[name]       # one extra rounding per hop


def test_half_packing_is_a_permutation(ksb):
    p = (2, 16, 32, 3)
    K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=3)).to(torch.bfloat16)
    f = ksb.Factor(*p, K4)
    raw = K4.view(torch.int16).numpy().astype(np.uint16)
    assert np.array_equal(f.read_packed(0), raw.reshape(-1))
    a, b, c, d = p
    assert np.array_equal(f.read_packed(2), raw.reshape(a, b, c, d).transpose(0, 3, 1, 2).reshape(-1))
