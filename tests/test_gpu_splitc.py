"""Small-batch split-c warp-shuffle kernel against
the oracle: lanes split the reduction over l and a fixed butterfly of
__shfl_xor_sync combines them.  Deterministic, within the FP32 contract, and
bit-exact on small-integer data (exact arithmetic)."""
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


def run(ksb, f, X, layout, bias=None):
    Xd = torch.from_numpy(X if layout == "bsf" else ksgen.to_bsl(X)).cuda()
    bd = torch.from_numpy(bias).cuda() if bias is not None else None
    Y = ksb.matmul(f, Xd, layout=layout, bias=bd)
    torch.cuda.synchronize()
    return Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T


PATS = [(1, 128, 128, 1), (2, 48, 48, 8), (6, 64, 64, 1), (1, 64, 256, 16), (3, 16, 24, 5), (1, 768, 192, 2),
        (2, 8, 200, 3), (4, 32, 33, 2)]


@pytest.mark.parametrize("p", PATS)
@pytest.mark.parametrize("B", [1, 3, 8, 33, 64])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_splitc_matches_oracle(ksb, p, B, layout):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=5)
    X = ksgen.x_normal(B, N, seed=6)
    f = ksb.Factor(*p, K4).set_kernel(ksb.KERNEL_SPLITC)
    Y = run(ksb, f, X, layout)
    Yref, env = O.matmul(p, K4, X, want_env=True)
    assert O.normwise_error(Y, Yref) <= 1e-5
    assert np.all(np.abs(Y - Yref) <= O.envelope_delta(p[2], 0.0) * env)
    assert np.array_equal(run(ksb, f, X, layout), Y)            # deterministic


@pytest.mark.parametrize("p", [(1, 128, 128, 1), (2, 48, 48, 8), (3, 16, 24, 5)])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_splitc_integer_bit_exact_and_bias(ksb, p, layout):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_int(*p, seed=2001)
    X = ksgen.x_int(37, N, seed=2000)
    f = ksb.Factor(*p, K4).set_kernel(ksb.KERNEL_SPLITC)
    assert np.array_equal(run(ksb, f, X, layout).astype(np.float64), O.matmul(p, K4, X))
    bias = ksgen.x_normal(1, M, seed=7)[0]
    Yb = run(ksb, f, X, layout, bias)
    assert np.array_equal(Yb, (run(ksb, f, X, layout) + bias[None, :]).astype(np.float32))


def test_splitc_plan_boundary(ksb):
    f = ksb.Factor(1, 64, 64, 1, ksgen.k4_uniform(1, 64, 64, 1, seed=1))
    assert f.plan(64, "bsf") == "splitc"
    assert f.plan(65, "bsf") != "splitc"
    assert f.plan(64, "bsl") == "splitc"
    h = ksb.Factor(64, 64, 64, 1, ksgen.k4_uniform(64, 64, 64, 1, seed=1))  # BSL, B >= 32, > 8 M MACs
    assert h.plan(16, "bsl") == "splitc" and h.plan(40, "bsl") != "splitc" and h.plan(64, "bsf") == "splitc"
    g = ksb.Factor(1, 60, 64, 1, ksgen.k4_uniform(1, 60, 64, 1, seed=1))     # b % 8 != 0
    assert g.plan(8, "bsf") != "splitc"
