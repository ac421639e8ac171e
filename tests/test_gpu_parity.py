"""GPU parity: the CUDA path through the C ABI vs the FP64 CPU oracle.

Contract (north star): normwise error max|Y^-Y|/max|Y| <= 1e-5
for FP32 (5e-3 for TF32), every element inside the O-6 envelope, and
bit-exact results on small-integer data, one-hot probes and packed index maps.
"""
import itertools

import numpy as np
import pytest

import ksgen
from ksgen import configs
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def ksb():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()          # raises if libks.so is missing: no fallback
    return ksb


def dev():
    return torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def run(ksb, f, X_bsf, layout):
    """Run ks_matmul in `layout` on BSF host data; return BSF host result."""
    if layout == "bsf":
        Y = ksb.matmul(f, to_dev(X_bsf), layout="bsf")
        torch.cuda.synchronize()
        return Y.cpu().numpy()
    Y = ksb.matmul(f, to_dev(ksgen.to_bsl(X_bsf)), layout="bsl")
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


def check_fp32(Yg, Yref, env, c):
    err = O.normwise_error(Yg, Yref)
    assert err <= FP32_TOL, err
    bound = O.envelope_delta(c, 0.0) * env
    assert np.all(np.abs(Yg.astype(np.float64) - Yref) <= bound + 1e-300), "outside envelope"
    return err


TINY = list(itertools.product(range(1, 5), repeat=4))


@pytest.mark.parametrize("kernel", ["auto", "generic"])
def test_exhaustive_tiny_patterns(ksb, kernel):
    """All 256 patterns with a,b,c,d in {1..4} x B in {1,7,8,33} x both layouts."""
    for p in TINY:
        a, b, c, d = p
        M, N, _ = O.dims(p)
        K4 = ksgen.k4_uniform(*p, seed=1000 + a + 4 * b)
        X = ksgen.x_normal(33, N, seed=0)
        Yref, env = O.matmul(p, K4, X, want_env=True)
        f = ksb.Factor(*p, K4)
        if kernel == "generic":
            f.set_kernel(ksb.KERNEL_GENERIC)
        for B in (1, 7, 8, 33):
            for layout in ("bsf", "bsl"):
                Yg = run(ksb, f, X[:B], layout)
                check_fp32(Yg, Yref[:B], env[:B], c)


@pytest.mark.parametrize("p", [(2, 4, 4, 2), (2, 4, 4, 4), (4, 4, 4, 2), (1, 2, 2, 1), (3, 3, 5, 7),
                               (2048, 2, 2, 1), (1, 2, 2, 2048), (5, 1, 1, 3), (1, 1, 9, 1), (1, 9, 1, 4)])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_integer_data_bit_exact(ksb, p, layout):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_int(*p, seed=2001)
    for B in (1, 5, 64):
        X = ksgen.x_int(B, N, seed=2000)
        Yref = O.matmul(p, K4, X)
        f = ksb.Factor(*p, K4)
        for kern in (ksb.KERNEL_AUTO, ksb.KERNEL_GENERIC):
            f.set_kernel(kern)
            assert np.array_equal(run(ksb, f, X, layout).astype(np.float64), Yref)


@pytest.mark.parametrize("p", [(2, 3, 2, 3), (2, 4, 4, 2), (3, 2, 2, 5), (1, 4, 4, 8)])
def test_one_hot_probe_reads_support(ksb, p):
    """X = I_N reveals K^T exactly: device support and value mapping."""
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_labels(*p)
    D = O.dense(p, K4)
    f = ksb.Factor(*p, K4)
    for layout in ("bsf", "bsl"):
        assert np.array_equal(run(ksb, f, np.eye(N, dtype=np.float32), layout), D.T)


@pytest.mark.parametrize("p", [(2, 3, 2, 3), (1, 48, 48, 4), (3, 16, 32, 2)])
def test_packed_layouts_bit_exact(ksb, p):
    a, b, c, d = p
    K4 = ksgen.k4_uniform(*p, seed=7)
    f = ksb.Factor(*p, K4)
    assert np.array_equal(f.read_packed(0), K4.reshape(-1))
    Kb = O.bmm_weights(p, K4)                                  # (ad, b, c)
    assert np.array_equal(f.read_packed(1), Kb.transpose(0, 2, 1).astype(np.float32).reshape(-1))
    assert np.array_equal(f.read_packed(2).view(np.uint32),
                          O.round_tf32_rna(Kb.astype(np.float32)).view(np.uint32).reshape(-1))


def test_fft_chain_full_size_sampled_rows(ksb):
    """configs[1] in bench.py's launch configuration (B=8192, BSF, ks_chain):
    sampled rows vs the oracle computed row by row."""
    L, B = configs.FFT_L, configs.FFT_BATCH
    pats = configs.dyadic_patterns(L)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    X = ksgen.x_normal(B, 2 ** L, seed=0)
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    Y = ksb.chain(fs, to_dev(X))
    torch.cuda.synchronize()
    rows = np.array([0, 1, 2, 3, 4095, 4096, 8190, 8191] + list(np.random.default_rng(1).integers(0, B, 8)))
    Yref, env = O.chain(pats, K4s, X, rows=rows, want_env=True)
    Yg = Y.cpu().numpy()[rows]
    err = O.normwise_error(Yg, Yref)
    assert err <= FP32_TOL, err
    delta = O.envelope_delta(2, 0.0)
    assert np.all(np.abs(Yg - Yref) <= ((1 + delta) ** L - 1) * env)


@pytest.mark.parametrize("layout", ["bsf", "bsl"])
@pytest.mark.parametrize("L", [1, 3, 8, 12])
def test_hadamard_chain_bit_exact(ksb, L, layout):
    pats, K4s = O.hadamard_factors(L)
    N = 2 ** L
    X = ksgen.x_int(37, N, seed=2002)
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    Xd = to_dev(X if layout == "bsf" else ksgen.to_bsl(X))
    Y = ksb.chain(fs, Xd, layout=layout)
    torch.cuda.synchronize()
    Yg = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    assert np.array_equal(Yg.astype(np.float64), O.chain(pats, K4s, X))


def test_dft_chain_real_imag_split_matches_numpy_fft(ksb):
    """Fig. 1 worked example on the GPU: complex factors split into real
    handles, two real ks_matmul launches per factor on the stacked batch."""
    L, B = 12, 16
    N = 2 ** L
    pats, K4c = O.dft_factors(L)
    Zr = ksgen.x_normal(B, N, seed=20)
    Zi = ksgen.x_normal(B, N, seed=21)
    ref = np.fft.fft((Zr.astype(np.float64) + 1j * Zi)[:, O.bitrev(L)], axis=1)
    Z = to_dev(np.concatenate([Zr, Zi]))
    for p, K in zip(reversed(pats), reversed(K4c)):
        Kr, Ki = O.split_complex_factor(K)
        U = ksb.matmul(ksb.Factor(*p, Kr), Z)
        V = ksb.matmul(ksb.Factor(*p, Ki), Z)
        Z = torch.cat([U[:B] - V[B:], V[:B] + U[B:]])
    torch.cuda.synchronize()
    Zh = Z.cpu().numpy().astype(np.float64)
    got = Zh[:B] + 1j * Zh[B:]
    # complex moduli: real AND imaginary parts are compared (normwise_error
    # promotes to complex128); each half is also checked on its own
    assert O.normwise_error(got, ref) < 1e-5
    assert O.normwise_error(Zh[:B], ref.real) < 1e-5 * np.abs(ref).max() / np.abs(ref.real).max()
    assert O.normwise_error(Zh[B:], ref.imag) < 1e-5 * np.abs(ref).max() / np.abs(ref.imag).max()


@pytest.mark.parametrize("name", ["VIT_UP", "VIT_DOWN", "GPT2_DOWN", "GPT2_UP"])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_model_chains_small_batch(ksb, name, layout):
    pats = getattr(configs, name)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = configs.chain_dims(pats)[0]
    B = 67
    X = ksgen.x_normal(B, N, seed=0)
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    Xd = to_dev(X if layout == "bsf" else ksgen.to_bsl(X))
    Y = ksb.chain(fs, Xd, layout=layout)
    torch.cuda.synchronize()
    Yg = Y.cpu().numpy() if layout == "bsf" else Y.cpu().numpy().T
    assert O.normwise_error(Yg, O.chain(pats, K4s, X)) <= FP32_TOL


def test_chain_host_equals_device(ksb):
    pats = configs.dyadic_patterns(10)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    X = ksgen.x_normal(300, 1024, seed=0)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty((300, 1024), dtype=torch.float32).pin_memory()
    ksb.chain_host(fs, Xh, Yh)
    torch.cuda.synchronize()
    Yd = ksb.chain(fs, to_dev(X))
    torch.cuda.synchronize()
    assert np.array_equal(Yh.numpy(), Yd.cpu().numpy())


@pytest.mark.parametrize("layout", ["bsf", "bsl"])
@pytest.mark.parametrize("pinned", [True, False])
def test_chain_host_pipelined_chunks(ksb, layout, pinned):
    """ks_chain_host cuts big batches into ~16 MB chunks pipelined over three
    internal streams (H2D / chain / D2H): several chunks with a ragged last one,
    both layouts (BSL chunks are 2-D column-block copies), pinned and pageable
    host memory, a non-default caller stream -> bit-identical to the device chain."""
    pats = [(6, 64, 64, 1), (1, 128, 128, 3)]            # configs[3] DOWN shapes, FFMA (FP32)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    N, M = configs.chain_dims(pats)[0], fs[0].M
    B = 9002                                              # 3 KB per row -> 4 chunks of 5462 / ... ragged
    X = ksgen.x_normal(B, N, seed=0)
    Xl = X if layout == "bsf" else ksgen.to_bsl(X)
    Xh = torch.from_numpy(np.ascontiguousarray(Xl))
    Yh = torch.empty((B, M) if layout == "bsf" else (M, B), dtype=torch.float32)
    if pinned:
        Xh, Yh = Xh.pin_memory(), Yh.pin_memory()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ksb.chain_host(fs, Xh, Yh, layout=layout, stream=s)
    s.synchronize()
    Yd = ksb.chain(fs, to_dev(Xl), layout=layout)
    torch.cuda.synchronize()
    assert np.array_equal(Yh.numpy(), Yd.cpu().numpy())
    rows = np.array([0, 1, 5461, 5462, B - 1])
    Yr = Yh.numpy() if layout == "bsf" else Yh.numpy().T
    assert O.normwise_error(Yr[rows], O.chain(pats, K4s, X, rows=rows)) <= 1e-5


def test_deterministic_and_misaligned(ksb):
    p = (4, 2, 2, 16)
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=3)
    f = ksb.Factor(*p, K4)
    X = ksgen.x_normal(129, N, seed=4)
    Y1 = run(ksb, f, X, "bsf")
    Y2 = run(ksb, f, X, "bsf")
    assert np.array_equal(Y1, Y2)
    # 4-byte but not 16-byte aligned views take the narrower vector path
    buf = torch.zeros(129 * N + 1, device=dev())
    buf[1:].copy_(to_dev(X).reshape(-1))
    Xv = buf[1:].view(129, N)
    out = torch.zeros(129 * M + 1, device=dev())
    Yv = out[1:].view(129, M)
    ksb.matmul(f, Xv, Yv)
    torch.cuda.synchronize()
    assert np.array_equal(Yv.cpu().numpy(), Y1)


def test_edge_cases_and_errors(ksb):
    p = (2, 2, 2, 2)
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
    X = torch.zeros((0, 8), device=dev())
    Y = torch.zeros((0, 8), device=dev())
    ksb.matmul(f, X, Y)                                    # B = 0: no-op
    X = torch.zeros((4, 8), device=dev())
    with pytest.raises(ksb.KSError):                       # overlap
        ksb.matmul(f, X, X)
    g = ksb.Factor(1, 3, 3, 1, np.ones(9, np.float32))
    with pytest.raises(ksb.KSError) as e:                  # not chainable
        ksb.chain([f, g], torch.zeros((4, 3), device=dev()))
    assert e.value.status == 3
    with pytest.raises(ksb.KSError) as e:                  # TF32 needs b,c >= 16
        f.set_math(ksb.MATH_TF32)
    assert e.value.status == 4
    f.set_kernel(ksb.KERNEL_STREAM)
    h = ksb.Factor(1, 3, 3, 1, np.ones(9, np.float32)).set_kernel(ksb.KERNEL_STREAM)
    with pytest.raises(ksb.KSError) as e:                  # forced family cannot run b=3
        ksb.matmul(h, torch.zeros((4, 3), device=dev()))
    assert e.value.status == 4
    with pytest.raises(ksb.KSError):
        ksb.Factor(0, 1, 1, 1, np.ones(1, np.float32))


def test_plan_table(ksb):
    f = ksb.Factor(2, 2, 2, 8, np.ones(64, np.float32))
    assert f.plan(8192, "bsf") == "stream"
    g = ksb.Factor(1, 3, 5, 2, np.ones(30, np.float32))
    assert g.plan(8, "bsl") == "generic"


# ---------------------------------------------------------- FFMA kernel ----
GEMMLIKE = [(1, 48, 48, 1), (1, 64, 64, 2), (2, 96, 96, 4), (1, 128, 128, 3), (3, 64, 64, 16),
            (1, 48, 48, 64), (6, 64, 64, 1), (1, 768, 192, 2), (6, 64, 256, 1), (64, 64, 64, 1),
            (1, 64, 256, 16), (1, 256, 64, 16), (2, 32, 16, 4), (1, 24, 8, 5), (2, 192, 48, 2),
            (2, 96, 64, 3), (1, 64, 48, 3), (3, 32, 32, 2), (1, 48, 48, 3), (4, 96, 96, 1), (1, 96, 160, 1), (1, 64, 64, 6), (2, 96, 32, 6)]


@pytest.mark.parametrize("p", GEMMLIKE)
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_ffma_matches_oracle_and_generic(ksb, p, layout):
    """Register-tiled kernel: same FMA order as the generic kernel (bit-equal)
    and within the FP32 contract of the oracle; ragged batch tails."""
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=1000 + p[1])
    X = ksgen.x_normal(300, N, seed=0)
    f = ksb.Factor(*p, K4)
    assert f.plan(300, layout) == "ffma"
    f.set_kernel(ksb.KERNEL_FFMA)
    Yf = run(ksb, f, X, layout)
    f.set_kernel(ksb.KERNEL_GENERIC)
    Yg = run(ksb, f, X, layout)
    assert np.array_equal(Yf, Yg)
    rows = np.arange(300) if M * N <= 1 << 22 else np.array([0, 1, 63, 64, 127, 128, 255, 256, 299])
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    check_fp32(Yf[rows], Yref, env, p[2])
    if layout == "bsf":
        f.set_kernel(ksb.KERNEL_FFMA)
        for B in (1, 7):
            assert np.array_equal(run(ksb, f, X[:B], layout), Yg[:B])


@pytest.mark.parametrize("grid", [1, 3, 7])
def test_ffma_ws_many_tiles_per_cta(grid):
    """Warp-specialised FFMA kernel with a capped persistent grid (KS_TF32_MAXGRID):
    every CTA runs several tiles, so the TMA ring and its last-reader refills wrap."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KS_TF32_MAXGRID=str(grid), KS_MULTITILE_MATH="fp32")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "multitile_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("p", [(1, 128, 128, 64), (16, 48, 48, 4), (1, 96, 96, 1), (4, 64, 64, 16), (1, 128, 128, 1), (1, 64, 64, 2), (1, 128, 128, 6)])
@pytest.mark.parametrize("layout", ["bsf", "bsl"])
def test_sweep_full_size_sampled_rows(ksb, p, layout):
    """configs[2] at B = 25088 in bench's launch configuration (auto plan):
    sampled rows against the oracle, computed one by one."""
    B = configs.SWEEP_BATCH
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=1000)
    X = ksgen.x_normal(B, N, seed=0)
    f = ksb.Factor(*p, K4)
    Yg = run(ksb, f, X, layout)
    rows = np.array([0, 1, 2, 127, 128, 12543, 25086, 25087] + list(np.random.default_rng(2).integers(0, B, 4)))
    Yref, env = O.matmul(p, K4, X, rows=rows, want_env=True)
    check_fp32(Yg[rows], Yref, env, p[2])


@pytest.mark.parametrize("name", ["VIT_UP", "VIT_DOWN", "GPT2_DOWN", "GPT2_UP"])
def test_model_chain_full_size_sampled_rows(ksb, name):
    pats = getattr(configs, name)
    B = configs.VIT_BATCH if name.startswith("VIT") else configs.GPT2_BATCH
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = configs.chain_dims(pats)[0]
    X = ksgen.x_normal(B, N, seed=0)
    fs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    Y = ksb.chain(fs, to_dev(X))
    torch.cuda.synchronize()
    rows = np.array([0, 1, 127, 128, B // 2, B - 2, B - 1])
    Yref = O.chain(pats, K4s, X, rows=rows)
    assert O.normwise_error(Y.cpu().numpy()[rows], Yref) <= FP32_TOL


@pytest.mark.parametrize("math", ["tf32", "f32x3"])
@pytest.mark.parametrize("name", ["VIT_UP", "VIT_DOWN", "GPT2_DOWN", "GPT2_UP"])
def test_model_chain_full_size_tensor_core_sampled_rows(ksb, name, math):
    """configs[3]/[4] at the bench's sizes and launch configuration (BSF, per-factor
    launches) in TF32 (normwise 5e-3) and 3xTF32 (FP32 contract 1e-5), sampled rows
    against the FP64 oracle, and the CUDA-graph replay bit-identical to it."""
    pats = getattr(configs, name)
    B = configs.VIT_BATCH if name.startswith("VIT") else configs.GPT2_BATCH
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = configs.chain_dims(pats)[0]
    X = ksgen.x_normal(B, N, seed=0)
    fs = [ksb.Factor(*p, k).set_math(ksb.MATH_TF32 if math == "tf32" else ksb.MATH_F32X3)
          for p, k in zip(pats, K4s)]
    assert all(f.plan(B, "bsf") == "tf32" for f in fs)
    Xd = to_dev(X)
    Y = ksb.chain(fs, Xd)
    Yg = torch.empty_like(Y)
    g = ksb.ChainGraph(fs, Xd, Yg)
    g.launch()
    torch.cuda.synchronize()
    assert torch.equal(Yg, Y)
    g.free()
    rows = np.array([0, 1, 127, 128, B // 2, B - 1])
    Yref = O.chain(pats, K4s, X, rows=rows)
    assert O.normwise_error(Y.cpu().numpy()[rows], Yref) <= (5e-3 if math == "tf32" else FP32_TOL)
