"""TF32 BSF densified super-blocks (2 <= d <= 8): the packed (bd x cd) blocks
bit-exactly against the oracle's masked dense K (Def. 1)
rounded to TF32, and the forced densified path against the oracle."""
import os
import subprocess
import sys

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


@pytest.mark.parametrize("p", [(2, 16, 24, 3), (1, 48, 48, 2), (3, 32, 16, 4), (1, 16, 16, 8), (2, 24, 40, 5)])
def test_dense_blocks_bit_exact(ksb, p):
    a, b, c, d = p
    K4 = ksgen.k4_uniform(*p, seed=11)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    got = f.read_packed(4).reshape(a, b * d, c * d)
    D = O.dense(p, K4)                                   # M x N, FP64, zeros off the support
    for i in range(a):
        blk = D[i * b * d:(i + 1) * b * d, i * c * d:(i + 1) * c * d].astype(np.float32)
        assert np.array_equal(got[i].view(np.uint32), O.round_tf32_rna(blk).view(np.uint32))


@pytest.mark.parametrize("mode", ["2", "1"])
def test_densified_path_matches_oracle(mode):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_DENSIFY=mode)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "dense_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
