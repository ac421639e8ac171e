"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test ties an oracle function to something other than itself: a brute
force Kronecker product, a numpy/scipy routine, a worked example printed in
the paper or SPEC (tests/golden/, each with its citation), or an exact
integer identity between independently written routes.  The selection is
meant to catch a dropped term, a wrong sign/index or a transposed operand.
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.linalg

import ksgen
from ksgen import configs, grid
import oracle as O

from conftest import GOLDEN

SMALL = [p for p in itertools.product(range(1, 5), repeat=4)]


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- support --
def _kron_mask(a, b, c, d):
    return np.kron(np.kron(np.eye(a), np.ones((b, c))), np.eye(d)) != 0


@pytest.mark.parametrize("p", SMALL[::3] + [(1, 5, 3, 2), (3, 2, 5, 3), (2, 6, 1, 5)])
def test_support_mask_equals_kronecker(p):
    """Def. 1: S = I_a (x) 1_{bxc} (x) I_d, brute force."""
    m = O.support_mask(p)
    assert np.array_equal(m, _kron_mask(*p))
    M, N, nnz = O.dims(p)
    assert m.shape == (M, N)
    assert int(m.sum()) == nnz                      # abcd nonzeros
    assert O.density(p) * M * N == pytest.approx(nnz)  # density 1/(ad)


def test_support_golden():
    g = _golden("spec_examples.json")["support_1222"]
    assert np.array_equal(O.support_mask(g["pattern"]).astype(int), np.array(g["mask"]))


@pytest.mark.parametrize("p", SMALL[::2])
def test_dense_support_and_values(p):
    """O-1 puts exactly abcd values on the Kronecker support, each label once."""
    a, b, c, d = p
    K4 = ksgen.k4_labels(a, b, c, d)
    D = O.dense(p, K4)
    assert np.array_equal(D != 0, _kron_mask(*p))
    assert sorted(D[D != 0].astype(int).tolist()) == list(range(1, a * b * c * d + 1))


def test_to_dense_golden():
    g = _golden("spec_examples.json")["to_dense_1222"]
    p = tuple(g["pattern"])
    K4 = ksgen.k4_labels(*p)
    D = O.dense(p, K4)
    for r, s, idx in g["entries"]:
        assert D[r, s] == K4[tuple(idx)]


# ------------------------------------------------------------ tile sets ----
def test_fig4_tile_sets_golden():
    g = _golden("fig4_tiles.json")
    for t in g["tiles"]:
        row, col = O.tile_sets(g["pattern"], t["i"], t["j"])
        assert row == t["row"] and col == t["col"]


@pytest.mark.parametrize("p", SMALL)
def test_tile_sets_partition_and_support(p):
    """row_{i,j} partition [0,M), col_{i,j} partition [0,N), and
    the support of K is exactly the union of row_{i,j} x col_{i,j}."""
    a, b, c, d = p
    M, N, _ = O.dims(p)
    rows, cols = [], []
    mask = np.zeros((M, N), dtype=bool)
    for i in range(a):
        for j in range(d):
            r, s = O.tile_sets(p, i, j)
            assert r == sorted(r) and s == sorted(s)
            rows += r
            cols += s
            mask[np.ix_(r, s)] = True
    assert sorted(rows) == list(range(M))
    assert sorted(cols) == list(range(N))
    assert np.array_equal(mask, _kron_mask(*p))


# -------------------------------------------------------- matmul (O-2) -----
def test_matmul_golden_1221():
    g = _golden("spec_examples.json")["matmul_1221"]
    Y = O.matmul(g["pattern"], np.array(g["K4"], np.float32), np.array(g["X"], np.float32))
    assert np.array_equal(Y, np.array(g["Y"], np.float64))


@pytest.mark.parametrize("p", [(2, 3, 2, 3), (1, 4, 2, 3), (3, 2, 5, 2), (2, 4, 4, 2), (1, 7, 5, 1)])
def test_matmul_equals_numpy_on_dense(p):
    """The C triple loop equals numpy's X @ D^T (library matmul) and the
    brute-force definition with the Kronecker mask applied to a dense draw."""
    a, b, c, d = p
    M, N, _ = O.dims(p)
    X = ksgen.x_normal(9, N, seed=3)
    K4 = ksgen.k4_uniform(*p, seed=4)
    Y = O.matmul(p, K4, X)
    D = O.dense(p, K4)
    np.testing.assert_allclose(Y, X.astype(np.float64) @ D.T, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("p", [(2, 3, 2, 3), (3, 2, 5, 2), (1, 1, 1, 1), (4, 1, 3, 2)])
def test_matmul_layouts_rows_and_threads(p):
    M, N, _ = O.dims(p)
    X = ksgen.x_normal(11, N, seed=5)
    K4 = ksgen.k4_uniform(*p, seed=6)
    Yf = O.matmul(p, K4, X, O.BSF, threads=1)
    Yl = O.matmul(p, K4, ksgen.to_bsl(X), O.BSL, threads=3)
    assert np.array_equal(Yf, Yl)                    # layout only changes addressing
    rows = [10, 0, 7]
    assert np.array_equal(O.matmul(p, K4, X, O.BSF, rows=rows), Yf[rows])
    assert np.array_equal(O.matmul(p, K4, ksgen.to_bsl(X), O.BSL, rows=rows), Yf[rows])


def test_matmul_special_cases_library():
    """(1,M,N,1) dense GEMM; (a,b,c,1) block-diagonal; (a,1,1,d) diagonal scale;
    (a,1,1,d) with unit values is the identity."""
    X = ksgen.x_normal(5, 12, seed=7)
    # dense
    K = ksgen.k4_uniform(1, 6, 12, 1, seed=8)
    np.testing.assert_allclose(O.matmul((1, 6, 12, 1), K, X), X.astype(np.float64) @ K[0, :, :, 0].T.astype(np.float64), rtol=1e-13)
    # block diagonal
    K = ksgen.k4_uniform(3, 2, 4, 1, seed=9)
    BD = scipy.linalg.block_diag(*[K[i, :, :, 0].astype(np.float64) for i in range(3)])
    np.testing.assert_allclose(O.matmul((3, 2, 4, 1), K, X), X.astype(np.float64) @ BD.T, rtol=1e-13)
    # diagonal
    K = ksgen.k4_uniform(3, 1, 1, 4, seed=10)
    np.testing.assert_allclose(O.matmul((3, 1, 1, 4), K, X), X.astype(np.float64) * K.reshape(-1).astype(np.float64), rtol=1e-15)
    assert np.array_equal(O.matmul((3, 1, 1, 4), np.ones((3, 1, 1, 4), np.float32), X), X.astype(np.float64))


def test_one_hot_probe_reads_columns():
    """A one-hot X row e_s returns column s of D."""
    p = (2, 3, 2, 3)
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_labels(*p)
    D = O.dense(p, K4)
    Y = O.matmul(p, K4, np.eye(N, dtype=np.float32))
    assert np.array_equal(Y, D.T)


# -------------------------------------------- O-5: Alg.1 == einsum == Alg.2 --
@pytest.mark.parametrize("p", SMALL[::5] + [(2, 3, 2, 3), (1, 3, 1, 2), (3, 4, 2, 5), (2, 4, 4, 2)])
def test_alg1_einsum_alg2_bit_exact_on_integers(p):
    """Alg. 1 (App. A bmm listing), the einsum contraction, Alg. 2's tile loop and
    the dense triple loop agree bit-exactly on small-integer data."""
    a, b, c, d = p
    M, N, _ = O.dims(p)
    X = ksgen.x_int(7, N, seed=2000 + a)
    K4 = ksgen.k4_int(*p, seed=2100 + b)
    ref = O.matmul(p, K4, X)
    assert np.array_equal(O.alg1_bmm(p, K4, X), ref)
    assert np.array_equal(O.einsum_matmul(p, K4, X), ref)
    assert np.array_equal(O.alg2_tiles(p, K4, X), ref)


# ---------------------------------------------------- perfect shuffles -----
def test_perfect_shuffle_golden():
    g = _golden("spec_examples.json")["shuffles"]
    assert O.perfect_shuffle(2, 2).tolist() == g["p2q2"]
    assert O.perfect_shuffle(3, 2).tolist() == g["p3q2"]
    K = O.kron_shuffle_matrix(2, 2, 2)
    assert (K @ np.arange(8)).tolist() == g["kron_a2_p2q2"]


def test_perfect_shuffle_is_reshape_read_columnwise():
    """App. B Def.: reshape a length-pq vector into p x q row-major, read column-wise."""
    for p_, q_ in [(2, 3), (3, 2), (4, 5), (1, 4), (4, 1)]:
        v = np.arange(p_ * q_)
        assert np.array_equal(O.shuffle_matrix(p_, q_) @ v, v.reshape(p_, q_).T.reshape(-1))


@pytest.mark.parametrize("p", [p for p in SMALL if p[0] <= 3])
def test_block_diagonalisation(p):
    """App. B with the §8c-2 reading: P S Q^T = I_{ad} (x) 1_{bxc}
    for P = I_a (x) P_{b,d}, Q = I_a (x) P_{c,d}; and its blocks are App. A's K~."""
    a, b, c, d = p
    P = O.kron_shuffle_matrix(a, b, d)
    Q = O.kron_shuffle_matrix(a, c, d)
    S = _kron_mask(*p).astype(np.int64)
    assert np.array_equal(P @ S @ Q.T, np.kron(np.eye(a * d, dtype=np.int64), np.ones((b, c), np.int64)))
    K4 = ksgen.k4_labels(*p)
    Kt = P @ O.dense(p, K4) @ Q.T
    Kb = O.bmm_weights(p, K4)
    for t in range(a * d):
        assert np.array_equal(Kt[t * b:(t + 1) * b, t * c:(t + 1) * c], Kb[t])


def test_printed_transpose_convention_fails_when_b_ne_d():
    """Documents reading §8c-2: the literal P^T S Q^T of P:1017 is not block
    diagonal for (1,3,1,2)."""
    a, b, c, d = 1, 3, 1, 2
    P = O.kron_shuffle_matrix(a, b, d)
    Q = O.kron_shuffle_matrix(a, c, d)
    S = _kron_mask(a, b, c, d).astype(np.int64)
    target = np.kron(np.eye(a * d, dtype=np.int64), np.ones((b, c), np.int64))
    assert not np.array_equal(P.T @ S @ Q.T, target)


# -------------------------------------------------------- chains (O-3) -----
@pytest.mark.parametrize("pats", [configs.VIT_UP, configs.VIT_DOWN, [(2, 3, 2, 3), (3, 4, 2, 1)]])
def test_chain_matches_dense_product(pats):
    """Applied K_L first equals X (K_1...K_L)^T formed densely."""
    assert configs.chainable(pats)
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = configs.chain_dims(pats)[0]
    X = ksgen.x_normal(4, N, seed=11)
    Y = O.chain(pats, K4s, X)
    W = O.chain_dense_product(pats, K4s)
    np.testing.assert_allclose(Y, X.astype(np.float64) @ W.T, rtol=1e-11, atol=1e-11)
    Yl = O.chain(pats, K4s, ksgen.to_bsl(X), O.BSL)
    np.testing.assert_allclose(Yl, Y, rtol=0, atol=0)


def test_chain_rejects_unchainable():
    with pytest.raises(ValueError):
        O.chain([(1, 2, 2, 1), (1, 3, 3, 1)], [np.ones((1, 2, 2, 1)), np.ones((1, 3, 3, 1))], np.ones((1, 3)))


@pytest.mark.parametrize("L", range(1, 9))
def test_hadamard_chain_exact(L):
    """Dyadic factors with [[1,1],[1,-1]] blocks multiply to Sylvester H_{2^L}
    (S:427-438), checked against scipy.linalg.hadamard; H H = 2^L I."""
    pats, K4s = O.hadamard_factors(L)
    N = 2 ** L
    W = O.chain_dense_product(pats, K4s)
    H = scipy.linalg.hadamard(N)
    assert np.array_equal(W, H)
    X = ksgen.x_int(3, N, seed=2200)
    assert np.array_equal(O.chain(pats, K4s, X), X.astype(np.float64) @ H.T)
    assert np.array_equal(H @ H, N * np.eye(N))


@pytest.mark.parametrize("L", [1, 2, 3, 5, 8])
def test_fft_factorisation(L):
    """Fig. 1: K_1...K_L = F_N R_N with F the DFT and R_N the
    bit reversal (§8c-4).  Checked against numpy.fft."""
    pats, K4s = O.dft_factors(L)
    assert pats == configs.dyadic_patterns(L)
    N = 2 ** L
    W = np.eye(N, dtype=np.complex128)
    for p, K in zip(pats, K4s):
        W = W @ O.dense_complex(p, K)
    F = np.fft.fft(np.eye(N), axis=0)              # F[u, v] = exp(-2 pi i u v / N)
    R = np.eye(N)[:, O.bitrev(L)]                  # column permutation
    np.testing.assert_allclose(W, F @ R, atol=1e-12)
    Xc = ksgen.x_normal(3, N, seed=12) + 1j * ksgen.x_normal(3, N, seed=13)
    np.testing.assert_allclose(Xc @ W.T, np.fft.fft(Xc[:, O.bitrev(L)], axis=1), atol=1e-11)


def test_fft_real_imag_split_through_real_oracle():
    """Complex chain evaluated with the real oracle on (Re, Im) parts per factor
    (the GPU test's procedure, SURVEY §8c GPU-vs-oracle (5)) equals numpy.fft."""
    L = 6
    N = 2 ** L
    pats, K4s = O.dft_factors(L)
    Zr = ksgen.x_normal(4, N, seed=14).astype(np.float64)
    Zi = ksgen.x_normal(4, N, seed=15).astype(np.float64)
    ref = np.fft.fft((Zr + 1j * Zi)[:, O.bitrev(L)], axis=1)
    for p, K in zip(reversed(pats), reversed(K4s)):
        Kr, Ki = O.split_complex_factor(K)
        Dr, Di = O.dense(p, Kr), O.dense(p, Ki)
        Zr, Zi = (O.matmul_dense(Dr, Zr) - O.matmul_dense(Di, Zi),
                  O.matmul_dense(Di, Zr) + O.matmul_dense(Dr, Zi))
    np.testing.assert_allclose(Zr + 1j * Zi, ref, atol=1e-4)   # twiddles rounded to fp32


# -------------------------------------------------- traffic / grid / misc --
def test_traffic_golden_and_invariants():
    g = _golden("spec_examples.json")["traffic_1441"]
    p, B = tuple(g["pattern"]), g["B"]
    assert O.io_elements_baseline(p, B) == g["baseline_io"]
    assert O.io_elements_fused(p, B) == g["fused_io"]
    assert O.model_flops(p, B) // 2 == g["useful_macs"]
    assert 2 * O.io_elements_fused(p, B) / (O.model_flops(p, B) // 2) == g["wasted_ratio"]
    for p in SMALL[::7]:
        assert O.io_elements_baseline(p, 5) == 3 * O.io_elements_fused(p, 5)
        assert 2 * O.io_elements_fused(p, 5) / (O.model_flops(p, 5) // 2) == pytest.approx(2 * O.h_ratio(p))


def test_h_and_density_golden():
    g = _golden("spec_examples.json")
    for p, v in g["h_values"]["cases"]:
        assert O.h_ratio(p) == pytest.approx(v, rel=1e-12)
    for p, v in g["density"]["cases"]:
        assert O.density(p) == pytest.approx(v, rel=1e-12)


def test_grid_statistics_golden():
    g = _golden("grid_stats.json")
    pats = set(grid.paper_grid())
    assert len(pats) >= g["min_count"]
    nondense = [p for p in pats if p[0] * p[3] > 1]
    sp = np.array([100.0 * (1 - O.density(p)) for p in nondense])
    assert abs(np.median(sp) - g["median_sparsity_pct"]) <= g["rounding_pct"]
    assert abs(np.percentile(sp, 25) - g["q25_sparsity_pct"]) <= g["rounding_pct"]
    mn = np.array([O.dims(p)[0] * O.dims(p)[1] for p in pats], dtype=np.float64)
    assert abs(np.percentile(mn, 25) / g["mn_q1"] - 1) < g["mn_rel_tol"]
    assert abs(np.percentile(mn, 75) / g["mn_q3"] - 1) < g["mn_rel_tol"]
    assert len(grid.sweep_patterns()) == g["sweep_count"]


def test_envelope_bounds_fp32_gemm():
    """An FP32 computation (numpy sgemm) stays within the O-6 envelope."""
    p = (2, 48, 48, 4)
    M, N, _ = O.dims(p)
    X = ksgen.x_normal(64, N, seed=16)
    K4 = ksgen.k4_uniform(*p, seed=17)
    Y, E = O.matmul(p, K4, X, want_env=True)
    D32 = O.dense(p, K4).astype(np.float32)
    Y32 = (X @ D32.T).astype(np.float64)
    bound = O.envelope_delta(N, 0.0) * E        # dense sgemm sums N terms
    assert np.all(np.abs(Y32 - Y) <= bound)
    assert np.all(E >= np.abs(Y))
    assert O.normwise_error(Y32, Y) < 1e-5


def test_inputs_are_seeded_and_distributed():
    a = ksgen.x_normal(3, 5, seed=1)
    assert np.array_equal(a, ksgen.x_normal(3, 5, seed=1))
    k = ksgen.k4_uniform(2, 3, 16, 2, seed=5)
    assert k.dtype == np.float32 and np.all(np.abs(k) <= 0.25)
    r = ksgen.x_rows_normal([4, 1], 7, seed=9)
    assert np.array_equal(r[1], ksgen.x_rows_normal([1], 7, seed=9)[0])
    for pats in (configs.VIT_UP, configs.VIT_DOWN, configs.GPT2_UP, configs.GPT2_DOWN,
                 configs.dyadic_patterns(configs.FFT_L)):
        assert configs.chainable(pats)


def test_round_tf32_rna():
    """TF32 keeps 10 mantissa bits: representable values are fixed points, the
    rounding error is <= 2^-11 relative, ties go away from zero."""
    x = np.array([1.0, -3.5, 1 + 2 ** -10, 2.0 ** -20], np.float32)
    assert np.array_equal(O.round_tf32_rna(x), x)
    assert O.round_tf32_rna(np.float32(1 + 2 ** -11)) == np.float32(1 + 2 ** -10)     # tie away
    assert O.round_tf32_rna(np.float32(-(1 + 2 ** -11))) == np.float32(-(1 + 2 ** -10))
    assert O.round_tf32_rna(np.float32(1 + 2 ** -12)) == np.float32(1.0)
    r = ksgen.x_normal(1, 100000, seed=3)[0]
    t = O.round_tf32_rna(r)
    assert np.all(np.abs(t.astype(np.float64) - r) <= 2.0 ** -11 * np.abs(r))
    assert np.all((t.view(np.uint32) & np.uint32(0x1FFF)) == 0)


def test_truncate_tf32():
    """Truncation toward zero to 10 mantissa bits: |t| <= |x|, error < 2^-10 relative."""
    x = np.array([1.0, -3.5, 1 + 2 ** -10], np.float32)
    assert np.array_equal(O.truncate_tf32(x), x)
    assert O.truncate_tf32(np.float32(1 + 2 ** -11 + 2 ** -12)) == np.float32(1.0)
    assert O.truncate_tf32(np.float32(-(1 + 2 ** -11))) == np.float32(-1.0)
    r = ksgen.x_normal(1, 100000, seed=4)[0]
    t = O.truncate_tf32(r)
    assert np.all(np.abs(t) <= np.abs(r))
    assert np.all(np.abs(t.astype(np.float64) - r) < 2.0 ** -10 * np.abs(r))


# ------------------------------------------- the contract metric (R9, c-10) --
def test_normwise_error_hand_values_real():
    """max|Y_hat - Y| / max|Y| worked by hand."""
    ref = np.array([[3.0, -4.0], [0.0, 2.0]])
    got = np.array([[3.0, -3.0], [0.5, 2.0]])
    assert O.normwise_error(got, ref) == 0.25            # max diff 1.0 / max |ref| 4.0
    assert O.normwise_error(ref, ref) == 0.0
    assert O.normwise_error(np.zeros(3), np.zeros(3)) == 0.0
    assert O.normwise_error(np.array([0.0, 1e-30]), np.zeros(2)) == float("inf")
    assert O.normwise_error(np.array([np.nan, 0.0]), np.array([1.0, 0.0])) == float("inf")
    # max, not mean: one bad element among many good ones decides
    ref = np.ones(1000)
    got = ref.copy()
    got[517] = 1.5
    assert O.normwise_error(got, ref) == 0.5
    # float32 inputs are widened, not compared in float32
    assert O.normwise_error(np.float32([1 + 2 ** -23]), np.float64([1.0])) == 2.0 ** -23
    with pytest.raises(ValueError):
        O.normwise_error(np.zeros((2, 3)), np.zeros((3, 2)))


def test_normwise_error_hand_values_complex():
    """Complex moduli (the Fig. 1 DFT check): ref=[3+4j, 0],
    got=[3+4j, 1j] -> |1j| / |3+4j| = 1/5."""
    assert O.normwise_error(np.array([3 + 4j, 1j]), np.array([3 + 4j, 0])) == pytest.approx(0.2, abs=0)
    # an error only in the imaginary part is seen
    assert O.normwise_error(np.array([1 + 100j, 2 - 50j]), np.array([1 + 1j, 2 + 5j])) == \
        pytest.approx(99 / np.hypot(2, 5), rel=1e-15)
    # real got vs complex ref: the missing imaginary part counts
    assert O.normwise_error(np.array([1.0, 0.0]), np.array([1 + 1j, 0])) == pytest.approx(1 / np.sqrt(2))


def test_normwise_error_catches_corrupted_imaginary_half():
    """The GPU DFT test's recombination: a corrupted imaginary half of the
    stacked [Re; Im] batch must fail the 1e-5 contract."""
    L, B = 6, 4
    N = 2 ** L
    Zr = ksgen.x_normal(B, N, seed=30).astype(np.float64)
    Zi = ksgen.x_normal(B, N, seed=31).astype(np.float64)
    ref = np.fft.fft((Zr + 1j * Zi)[:, O.bitrev(L)], axis=1)
    good = ref.real + 1j * ref.imag
    assert O.normwise_error(good, ref) == 0.0
    bad_im = ref.real + 1j * (ref.imag + 1e-3 * np.abs(ref).max() * (np.arange(N) == 7))
    assert O.normwise_error(bad_im, ref) > 1e-5
    bad_sign = ref.real - 1j * ref.imag                  # conjugated output (a sign slip)
    assert O.normwise_error(bad_sign, ref) > 1e-2


def test_envelope_delta_hand_values():
    """delta = 2 u_in + u_in^2 + gamma_{2c}, gamma_n = n u / (1 - n u)."""
    assert O.envelope_delta(2, 0.1, u=0.01) == pytest.approx(0.2 + 0.01 + 0.04 / 0.96, rel=1e-15)
    assert O.envelope_delta(1, 0.0, u=0.25) == pytest.approx(0.5 / 0.5, rel=1e-15)
    u = 2.0 ** -24
    assert O.envelope_delta(64, 0.0) == pytest.approx(128 * u / (1 - 128 * u), rel=1e-15)
    assert O.envelope_delta(64, 2.0 ** -10) == pytest.approx(2 ** -9 + 2 ** -20 + 128 * u / (1 - 128 * u),
                                                             rel=1e-15)


def test_envelope_delta_covers_worst_observed_fp32_and_tf32_dots():
    """The bound holds for real FP32 sequential-FMA dot products (Higham's
    gamma_c is the textbook bound; the envelope uses 2c) and for TF32-truncated
    operands with u_in = 2^-10, on adversarially scaled data; and it is not
    vacuous: it is within 2^9 of the worst observed error."""
    rng = np.random.default_rng(7)
    worst_ratio = 0.0
    for c in (2, 16, 48, 128):
        x = rng.standard_normal((4000, c)).astype(np.float32)
        k = rng.uniform(-1, 1, (c,)).astype(np.float32)
        x[:, 0] *= 1e4                                  # large first term, cancellations later
        exact = x.astype(np.float64) @ k.astype(np.float64)
        env = np.abs(x).astype(np.float64) @ np.abs(k).astype(np.float64)
        acc = np.zeros(4000, np.float32)
        for l in range(c):                              # one rounding per add, ascending l
            acc = (acc + x[:, l] * k[l]).astype(np.float32)
        err = np.abs(acc.astype(np.float64) - exact)
        assert np.all(err <= O.envelope_delta(c, 0.0) * env)
        worst_ratio = max(worst_ratio, float(np.max(err / (O.envelope_delta(c, 0.0) * env))))
        xt = O.truncate_tf32(x).astype(np.float64)
        kt = O.round_tf32_rna(k).astype(np.float64)
        err_t = np.abs(xt @ kt - exact)
        assert np.all(err_t <= O.envelope_delta(c, 2.0 ** -10) * env)
    assert worst_ratio > 2.0 ** -9


def test_model_bytes_and_pattern_check_hand_values():
    """Byte model: 4 (B N + abcd + B M) bytes; FFT factor of
    configs[1]: (2^{l-1},2,2,2^{12-l}), B = 8192 -> 4 (2 * 8192 * 4096 + 8192)
    = 268,468,224 bytes (the per-launch figure in DESIGN §5.1 / BENCH_r01)."""
    assert O.model_bytes((1, 2, 2, 2048), 8192) == 268_468_224
    assert O.model_bytes((2048, 2, 2, 1), 8192) == 268_468_224
    # (2,4,4,2), B = 8 (configs[0]): N = M = 16, nnz = 64 -> 4 (128 + 64 + 128)
    assert O.model_bytes((2, 4, 4, 2), 8) == 1280
    assert O.model_bytes((1, 3, 5, 1), 2, elem_bytes=2) == 2 * (10 + 15 + 6)
    for bad in ((0, 1, 1, 1), (1, -2, 1, 1), (1, 1, 1, 0)):
        with pytest.raises(ValueError):
            O.check_pattern(bad)
    assert O.check_pattern((2, 3, 4, 5)) == (2, 3, 4, 5)


def test_gelu_hand_values_and_identity():
    """oracle.gelu against y * Phi(y) with Phi from the standard library's
    NormalDist (not math.erf), hand values, and gelu(y) - gelu(-y) = y."""
    from statistics import NormalDist
    phi = NormalDist().cdf
    ys = np.array([-6.0, -3.0, -1.0, -0.5, 0.0, 0.25, 1.0, 2.0, 5.0])
    g = O.gelu(ys)
    for y, v in zip(ys, g):
        assert abs(v - y * phi(y)) <= 1e-15 * max(1.0, abs(y))
    assert O.gelu(np.array([0.0]))[0] == 0.0
    assert abs(O.gelu(np.array([1.0]))[0] - 0.8413447460685429) < 1e-15
    assert abs(O.gelu(np.array([-1.0]))[0] + 0.15865525393145705) < 1e-15
    assert np.allclose(O.gelu(ys) - O.gelu(-ys), ys, rtol=0, atol=1e-15)
