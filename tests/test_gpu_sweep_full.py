"""configs[2] (the 88-pattern sweep) at its full batch B = 25088, every pattern,
FP32 and TF32, BSF and BSL, in the auto plan the bench times: sampled rows
against the FP64 oracle computed one by one (round 1
checked 7 FP32 and 10 TF32 of the 88 at full size).

X is one seeded host matrix (ksgen, no method arithmetic) whose first N columns
feed pattern (a, b, c, d); the oracle sees exactly those rows.  FP32: normwise
<= 1e-5 and every element inside the O-6 envelope (u_in = 0); TF32: normwise
<= 5e-3, the envelope with u_in = 2^-10, and the tight envelope against the
oracle on the TF32 operands (R10).
"""
import functools

import numpy as np
import pytest

import ksgen
from ksgen import configs
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

B = configs.SWEEP_BATCH
PATS = ksgen.grid.sweep_patterns()
NMAX = max(a * c * d for a, b, c, d in PATS)
ROWS = np.array([0, 1, 127, 128, 12543, 25086, 25087] + list(np.random.default_rng(5).integers(0, B, 3)))


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    return ksb


@pytest.fixture(scope="module")
def xfull():
    X = ksgen.x_normal(B, NMAX, seed=0)
    return X, torch.from_numpy(X).to("cuda:0")


@functools.lru_cache(maxsize=None)
def _k4(p):
    return ksgen.k4_uniform(*p, seed=1000)


def _oracle(p, Xrows, tf32):
    K4 = _k4(p)
    Yref, env = O.matmul(p, K4, Xrows, want_env=True)
    if not tf32:
        return Yref, env, None, None
    Ytf = O.matmul(p, O.round_tf32_rna(K4), O.truncate_tf32(Xrows))
    Yabs = O.matmul(p, np.abs(O.round_tf32_rna(K4)), np.abs(O.truncate_tf32(Xrows)))
    return Yref, env, Ytf, Yabs


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
@pytest.mark.parametrize("p", PATS, ids=[",".join(map(str, p)) for p in PATS])
def test_sweep_pattern_full_batch(ksb, xfull, p, layout, math):
    a, b, c, d = p
    M, N = a * b * d, a * c * d
    X, Xdev = xfull
    f = ksb.Factor(*p, _k4(p))
    if math == "tf32":
        f.set_math(ksb.MATH_TF32)
        assert f.plan(B, layout) == "tf32"
    Xd = Xdev[:, :N].contiguous() if layout == "bsf" else Xdev[:, :N].t().contiguous()
    Y = ksb.matmul(f, Xd, layout=layout)
    torch.cuda.synchronize()
    Yg = (Y[ROWS] if layout == "bsf" else Y[:, ROWS].t()).cpu().numpy()
    del Xd, Y
    Yref, env, Ytf, Yabs = _oracle(p, X[ROWS, :N], math == "tf32")
    if math == "fp32":
        assert O.normwise_error(Yg, Yref) <= 1e-5
        assert np.all(np.abs(Yg - Yref) <= O.envelope_delta(c, 0.0) * env + 1e-30)
    else:
        assert O.normwise_error(Yg, Yref) <= 5e-3
        assert np.all(np.abs(Yg - Yref) <= O.envelope_delta(c, 2.0 ** -10) * env)
        assert np.all(np.abs(Yg - Ytf) <= O.envelope_delta(c, 0.0) * Yabs + 1e-30)
    f.free()
