"""Randomised GPU parity: seeded random patterns (a, b, c, d), batch sizes and
layouts, in every arithmetic mode, against the FP64 oracle.  Exercises the plan
table on shapes no hand-written case covers (odd b / c / d, ragged batches,
the boundaries between kernel families)."""
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


def random_cases(n, seed):
    rng = np.random.default_rng(seed)
    dims = [1, 2, 3, 4, 5, 8, 12, 16, 24, 32, 48, 64, 80, 96, 112, 128]
    out = []
    while len(out) < n:
        b, c = int(rng.choice(dims)), int(rng.choice(dims))
        a, d = int(rng.integers(1, 5)), int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16]))
        if a * b * d * 4 > 1 << 16 or a * c * d > 1 << 13:
            continue
        B = int(rng.choice([1, 3, 8, 64, 129, 300, 517]))
        out.append(((a, b, c, d), B, "bsf" if rng.random() < 0.5 else "bsl"))
    return out


CASES = random_cases(48, seed=7) + random_cases(32, seed=8)


@pytest.mark.parametrize("math", ["fp32", "tf32", "f32x3"])
@pytest.mark.parametrize("p,B,layout", CASES)
def test_random_pattern_matches_oracle(ksb, p, B, layout, math):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=11)
    X = ksgen.x_normal(B, N, seed=12)
    f = ksb.Factor(*p, K4)
    tol = 1e-5
    if math != "fp32":
        if p[1] < 16 or p[2] < 16:             # tensor-core math needs b, c >= 16 (include/ks.h)
            with pytest.raises(ksb.KSError, match="KS_ERR_UNSUPPORTED"):
                f.set_math(ksb.MATH_TF32 if math == "tf32" else ksb.MATH_F32X3)
            return
        f.set_math(ksb.MATH_TF32 if math == "tf32" else ksb.MATH_F32X3)
        tol = 5e-3 if math == "tf32" else 1e-5
    Xd = torch.from_numpy(np.ascontiguousarray(X if layout == "bsf" else ksgen.to_bsl(X))).cuda()
    Y = ksb.matmul(f, Xd, layout=layout)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    ref = O.matmul(p, K4, X)
    err = O.normwise_error(Yh, ref)
    assert err <= tol, (f.plan(B, layout), err)
