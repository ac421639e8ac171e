"""Former performance cliffs to the one-thread-per-output generic kernel
(VERDICT r1 weak #6): BSL batches with B % 4 != 0 and X / Y views that are only
4-byte aligned now run the register-tiled FFMA kernel's scalar instantiation,
bit-identical to the generic kernel (same l-ascending FMA chain, R11)
and checked against the oracle."""
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


@pytest.mark.parametrize("p", [(1, 128, 128, 12), (2, 48, 48, 8), (3, 96, 64, 5), (6, 64, 64, 1)])
@pytest.mark.parametrize("B", [129, 257, 1003])
def test_bsl_ragged_batch_runs_ffma(ksb, p, B):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=3)
    X = ksgen.x_normal(B, N, seed=4)
    f = ksb.Factor(*p, K4)
    assert f.plan(B, "bsl") == "ffma"
    Xd = torch.from_numpy(ksgen.to_bsl(X)).cuda()
    Y = ksb.matmul(f, Xd, layout="bsl")
    f.set_kernel(ksb.KERNEL_GENERIC)
    Yg = ksb.matmul(f, Xd, layout="bsl")
    torch.cuda.synchronize()
    assert torch.equal(Y, Yg)                                  # same FMA order: bit-identical
    assert O.normwise_error(Y.cpu().numpy().T, O.matmul(p, K4, X)) <= 1e-5


@pytest.mark.parametrize("layout", ["bsf", "bsl"])
@pytest.mark.parametrize("p", [(1, 128, 128, 1), (2, 64, 48, 4), (1, 96, 64, 3)])
def test_four_byte_aligned_views(ksb, p, layout):
    M, N, _ = O.dims(p)
    B = 260
    K4 = ksgen.k4_uniform(*p, seed=5)
    X = ksgen.x_normal(B, N, seed=6)
    Xl = X if layout == "bsf" else ksgen.to_bsl(X)
    big = torch.empty(Xl.size + 1, device="cuda")
    big[1:] = torch.from_numpy(Xl.ravel()).cuda()
    Xv = big[1:].view(Xl.shape)                                # 4-byte aligned, not 16
    ybig = torch.empty(M * B + 3, device="cuda")
    Yv = ybig[3:].view((B, M) if layout == "bsf" else (M, B))
    f = ksb.Factor(*p, K4)
    assert f.plan(B, layout) == "ffma"
    ksb.matmul(f, Xv, Yv, layout=layout)
    f.set_kernel(ksb.KERNEL_GENERIC)
    Yg = ksb.matmul(f, Xv, layout=layout)
    torch.cuda.synchronize()
    assert torch.equal(Yv, Yg)
    Yh = Yv.cpu().numpy() if layout == "bsf" else Yv.cpu().numpy().T
    assert O.normwise_error(Yh, O.matmul(p, K4, X)) <= 1e-5


@pytest.mark.parametrize("layout", ["bsf", "bsl"])
@pytest.mark.parametrize("p", [(1, 80, 64, 1), (2, 112, 48, 3), (1, 40, 64, 4), (3, 16, 32, 2), (1, 8, 16, 6),
                               (4, 80, 80, 2), (1, 144, 96, 1)])
def test_b_multiple_of_8_runs_ffma(ksb, p, layout):
    """b % 8 == 0 outside 24Z u 32Z (b = 80, 112, 40, 16, 8, 144) runs the FFMA
    kernel's 16- / 8-wide warp tiles, bit-identical to the generic kernel."""
    M, N, _ = O.dims(p)
    B = 300
    K4 = ksgen.k4_uniform(*p, seed=7)
    X = ksgen.x_normal(B, N, seed=8)
    f = ksb.Factor(*p, K4)
    assert f.plan(B, layout) == "ffma"
    Xd = torch.from_numpy(X if layout == "bsf" else ksgen.to_bsl(X)).cuda()
    Y = ksb.matmul(f, Xd, layout=layout)
    f.set_kernel(ksb.KERNEL_GENERIC)
    Yg = ksb.matmul(f, Xd, layout=layout)
    torch.cuda.synchronize()
    assert torch.equal(Y, Yg)
    Yh = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    assert O.normwise_error(Yh, O.matmul(p, K4, X)) <= 1e-5
