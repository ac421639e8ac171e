"""The lane-j FFMA2 kernel (BSF, d % 4 == 0, knob KS_KNOB_FFMA_WSL): one j per
lane of a quad, shuffle-transposed epilogue, K^T tiles interleaved by one 4-D
TMA box.  Same l-ascending FMA chain per output as every FP32 kernel (R11), so
it must be bit-identical to the generic kernel, and within the FP32 contract of
the oracle; bias (NEXT-2) and ragged batch tiles included; a capped grid forces
several tiles per CTA (the ring running across tile boundaries)."""
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


def _knobs(ks):
    return ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32 | ks.KNOB_FFMA_WSL


@pytest.mark.parametrize("p", [(1, 64, 64, 4), (2, 128, 64, 8), (1, 48, 48, 16), (3, 96, 32, 4), (1, 64, 256, 16),
                               (1, 256, 64, 16), (2, 48, 96, 12)])
@pytest.mark.parametrize("B", [128, 300])
def test_wsl_bit_identical_to_generic(ksb, p, B):
    from paper_2405_15013_b200 import ks
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=21)
    X = ksgen.x_normal(B, N, seed=22)
    f = ksb.Factor(*p, K4)
    f.set_knobs(_knobs(ks))
    assert f.plan(B, "bsf") == "ffma"
    Xd = torch.from_numpy(X).cuda()
    Y = ksb.matmul(f, Xd)
    f.set_knobs(-1)
    f.set_kernel(ksb.KERNEL_GENERIC)
    Yg = ksb.matmul(f, Xd)
    torch.cuda.synchronize()
    assert torch.equal(Y, Yg)
    assert O.normwise_error(Y.cpu().numpy(), O.matmul(p, K4, X)) <= 1e-5


@pytest.mark.parametrize("p", [(1, 64, 64, 4), (2, 128, 64, 8)])
def test_wsl_bias_matches_oracle(ksb, p):
    from paper_2405_15013_b200 import ks
    M, N, _ = O.dims(p)
    B = 200
    K4 = ksgen.k4_uniform(*p, seed=23)
    X = ksgen.x_normal(B, N, seed=24)
    bias = np.random.default_rng(25).standard_normal(M).astype(np.float32)
    f = ksb.Factor(*p, K4)
    f.set_knobs(_knobs(ks))
    Y = ksb.matmul(f, torch.from_numpy(X).cuda(), bias=torch.from_numpy(bias).cuda())
    torch.cuda.synchronize()
    ref = O.matmul(p, K4, X) + bias.astype(np.float64)
    assert O.normwise_error(Y.cpu().numpy(), ref) <= 1e-5


def test_wsl_integer_data_bit_exact(ksb):
    from paper_2405_15013_b200 import ks
    p = (2, 64, 64, 8)
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_int(*p, seed=26)
    X = ksgen.x_int(130, N, seed=27)
    f = ksb.Factor(*p, K4)
    f.set_knobs(_knobs(ks))
    Y = ksb.matmul(f, torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy(), O.matmul(p, K4, X).astype(np.float32))


def test_wsl_many_tiles_per_cta():
    """KS_TF32_MAXGRID caps the persistent grid (also for the FFMA TMA kernels)."""
    code = r"""
import numpy as np, torch, ksgen, oracle as O
import paper_2405_15013_b200 as ksb
from paper_2405_15013_b200 import ks
p = (2, 64, 64, 8); B = 1000
K4 = ksgen.k4_uniform(*p, seed=28); X = ksgen.x_normal(B, 1024, seed=29)
f = ksb.Factor(*p, K4); f.set_knobs(ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32 | ks.KNOB_FFMA_WSL)
Y = ksb.matmul(f, torch.from_numpy(X).cuda()); torch.cuda.synchronize()
e = O.normwise_error(Y.cpu().numpy(), O.matmul(p, K4, X)); assert e <= 1e-5, e
print("ok", e)
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_MAXGRID="3", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
