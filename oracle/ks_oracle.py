"""CPU oracle for Kronecker-sparse (KS) matmul -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.

Citations are PAPER.md line numbers (``P:n``) with the section / algorithm /
equation they fall in; ``S:n`` is SPEC.md; ``§8c-k`` are the readings listed
in SURVEY.md §8(c) and DESIGN.md "Readings of the paper".

Pins (tests/test_oracle_pins.py) tie each function to something other than
itself: brute-force Kronecker products, numpy/scipy routines (FFT, Hadamard,
matmul), hand-worked examples printed in the paper/spec (tests/golden/), and
exact integer identities.  Every arithmetic function below is pinned,
including the contract metric normwise_error (hand-computed real and complex
values) and envelope_delta (hand values + real FP32/TF32 dot products); none
is "parity unpinned".  (Round 1 claimed this while normwise_error dropped
imaginary parts; fixed in round 2.)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ks_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libks_oracle.so")
_lib = None
_lib_lock = threading.Lock()

BSF = 0  # batch-size-first: X is B x N row-major (§2.2)
BSL = 1  # batch-size-last:  X is N x B row-major (§2.2; §8c-17)


# --------------------------------------------------------------------------
# the C part (naive FP64 triple loop)
# --------------------------------------------------------------------------
def build_lib(force: bool = False) -> str:
    """Compile oracle/ks_oracle.c with gcc (-O2, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lib_lock:
        if _lib is None:
            build_lib()
            lib = ctypes.CDLL(_LIB_PATH)
            i64, dp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
            lib.ks_oracle_dense.argtypes = [i64, i64, i64, i64, dp, dp]
            lib.ks_oracle_dense.restype = ctypes.c_int
            lib.ks_oracle_matmul_dense.argtypes = [
                i64, i64, dp, dp, i64, ctypes.c_int, ctypes.POINTER(i64), i64,
                dp, dp, ctypes.c_int]
            lib.ks_oracle_matmul_dense.restype = ctypes.c_int
            lib.ks_oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads() -> int:
    """Threads the oracle uses by default: the cores this process may run on."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# pattern algebra (Def. 1; Eq. heuristic)
# --------------------------------------------------------------------------
def check_pattern(p) -> tuple[int, int, int, int]:
    a, b, c, d = (int(v) for v in p)
    if min(a, b, c, d) < 1:
        raise ValueError(f"KS pattern entries must be >= 1, got {p}")
    return a, b, c, d


def dims(p) -> tuple[int, int, int]:
    """(M, N, nnz) = (abd, acd, abcd)  -- P:142 (Def. 1)."""
    a, b, c, d = check_pattern(p)
    return a * b * d, a * c * d, a * b * c * d


def density(p) -> float:
    """1/(ad)  -- P:163."""
    a, b, c, d = check_pattern(p)
    return 1.0 / (a * d)


def h_ratio(p) -> float:
    """h(b,c) = (b+c)/(bc)  -- Eq. (heuristic)."""
    a, b, c, d = check_pattern(p)
    return (b + c) / (b * c)


def support_mask(p) -> np.ndarray:
    """Boolean M x N support, from Def. 1 / Fig. 2 in index form:
    (r, s) is in the support iff r and s lie in the same diagonal super-block
    i (r // bd == s // cd) and carry the same inner offset j (r % d == s % d).
    Pinned against np.kron(np.kron(I_a, 1_{bxc}), I_d)."""
    a, b, c, d = check_pattern(p)
    M, N, _ = dims(p)
    r = np.arange(M)[:, None]
    s = np.arange(N)[None, :]
    return ((r // (b * d)) == (s // (c * d))) & ((r % d) == (s % d))


def tile_sets(p, i: int, j: int) -> tuple[list[int], list[int]]:
    """row_{i,j} and col_{i,j} of Alg. 2 lines 3-4:
    row = {i M/a + j + k d : 0 <= k < b},  col = {i N/a + j + l d : 0 <= l < c}."""
    a, b, c, d = check_pattern(p)
    M, N, _ = dims(p)
    if not (0 <= i < a and 0 <= j < d):
        raise IndexError((i, j))
    row = [i * (M // a) + j + k * d for k in range(b)]
    col = [i * (N // a) + j + l * d for l in range(c)]
    return row, col


# --------------------------------------------------------------------------
# O-1 / O-2 / O-3: dense oracle, matmul, chain
# --------------------------------------------------------------------------
def dense(p, K4) -> np.ndarray:
    """O-1: masked dense K (FP64, M x N) -- Def. 1 + canonical values (C code)."""
    a, b, c, d = check_pattern(p)
    K4 = np.ascontiguousarray(np.asarray(K4, dtype=np.float64).reshape(a, b, c, d))
    M, N, _ = dims(p)
    D = np.empty((M, N), dtype=np.float64)
    rc = _load().ks_oracle_dense(a, b, c, d, _dp(K4), _dp(D))
    if rc != 0:
        raise ValueError("ks_oracle_dense failed")
    return D


def matmul_dense(D: np.ndarray, X, layout: int = BSF, rows=None, threads=None,
                 want_env: bool = False):
    """O-2 on an already materialised dense K: Y = X D^T by the naive
    triple loop in C (FP64, s ascending).  Returns Y (nrows x M, BSF order) and,
    if requested, the envelope sum |X||D|."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    M, N = D.shape
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
    if layout == BSF:
        if X.ndim != 2 or X.shape[1] != N:
            raise ValueError(f"X must be B x {N} (BSF), got {X.shape}")
        B = X.shape[0]
    elif layout == BSL:
        if X.ndim != 2 or X.shape[0] != N:
            raise ValueError(f"X must be {N} x B (BSL), got {X.shape}")
        B = X.shape[1]
    else:
        raise ValueError("layout must be BSF (0) or BSL (1)")
    if rows is None:
        rows_arr, nrows, rows_ptr = None, B, None
    else:
        rows_arr = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        nrows = rows_arr.size
        rows_ptr = rows_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    Y = np.empty((nrows, M), dtype=np.float64)
    env = np.empty((nrows, M), dtype=np.float64) if want_env else None
    if nrows == 0:
        return (Y, env) if want_env else Y
    rc = _load().ks_oracle_matmul_dense(
        M, N, _dp(D), _dp(X), B, int(layout), rows_ptr, nrows, _dp(Y),
        _dp(env) if want_env else None, int(threads or default_threads()))
    if rc != 0:
        raise ValueError("ks_oracle_matmul_dense failed (row index out of range?)")
    return (Y, env) if want_env else Y


def matmul(p, K4, X, layout: int = BSF, rows=None, threads=None, want_env=False):
    """Y = X K^T for one KS factor, FP64, rows subset optional.
    Output is BSF-ordered (nrows x M) whatever the input layout."""
    return matmul_dense(dense(p, K4), X, layout, rows, threads, want_env)


def chain(patterns, K4s, X, layout: int = BSF, rows=None, threads=None,
          want_env: bool = False):
    """O-3: Y = X K_L^T ... K_1^T (P:53-54 with Y = X K^T of P:86; §8c-5):
    K_L is applied first; patterns/K4s are in product order K_1..K_L.
    FP64 throughout; the envelope is the same chain applied to |X| and |K|."""
    if len(patterns) != len(K4s) or not patterns:
        raise ValueError("need one K4 per pattern, L >= 1")
    for q, p in zip(patterns[:-1], patterns[1:]):
        if dims(q)[1] != dims(p)[0]:
            raise ValueError(f"not chainable: {q} then {p} (P:955)")
    Z = matmul(patterns[-1], K4s[-1], X, layout, rows, threads)
    E = None
    if want_env:
        Xa = np.abs(np.asarray(X, dtype=np.float64))
        E = matmul(patterns[-1], np.abs(np.asarray(K4s[-1], np.float64)), Xa, layout, rows, threads)
    for p, K4 in zip(reversed(patterns[:-1]), reversed(K4s[:-1])):
        Z = matmul(p, K4, Z, BSF, None, threads)
        if want_env:
            E = matmul(p, np.abs(np.asarray(K4, np.float64)), E, BSF, None, threads)
    return (Z, E) if want_env else Z


def chain_dense_product(patterns, K4s) -> np.ndarray:
    """W = K_1 ... K_L as a dense FP64 matrix (second route of O-3)."""
    W = dense(patterns[0], K4s[0])
    for p, K4 in zip(patterns[1:], K4s[1:]):
        W = W @ dense(p, K4)
    return W


# --------------------------------------------------------------------------
# O-5 independent cross-checks: Alg. 1 (App. A/B), einsum, Alg. 2
# --------------------------------------------------------------------------
def perfect_shuffle(p: int, q: int) -> np.ndarray:
    """Index vector of the (p,q) perfect shuffle P_{p,q} (App. B Def.):
    the rows of P_{p,q} are the identity rows R_0, ..., R_{q-1} with
    R_i = {i + q j : 0 <= j < p}; entry t of the vector is the identity row
    placed at row t, so (P_{p,q} v)[t] = v[perm[t]]."""
    return np.array([i + q * j for i in range(q) for j in range(p)], dtype=np.int64)


def shuffle_matrix(p: int, q: int) -> np.ndarray:
    perm = perfect_shuffle(p, q)
    P = np.zeros((p * q, p * q), dtype=np.int64)
    P[np.arange(p * q), perm] = 1
    return P


def kron_shuffle_matrix(a: int, p: int, q: int) -> np.ndarray:
    """I_a (x) P_{p,q} (Eq. permutations)."""
    return np.kron(np.eye(a, dtype=np.int64), shuffle_matrix(p, q))


def bmm_weights(p, K4) -> np.ndarray:
    """K~ as the (ad, b, c) tensor of App. A: block i*d + j is
    K[row_{i,j}, col_{i,j}] (§8c-2 reading: App. A reshape code is normative)."""
    a, b, c, d = check_pattern(p)
    K4 = np.asarray(K4, dtype=np.float64).reshape(a, b, c, d)
    return np.ascontiguousarray(K4.transpose(0, 3, 1, 2).reshape(a * d, b, c))


def alg1_bmm(p, K4, X_bsf) -> np.ndarray:
    """Alg. 1 executed as the App. A ``kronecker_bmm`` listing,
    restated in numpy: permute X (view (B,a,c,d) -> swap last two -> (B,ad,c)),
    batched GEMM with K~, permute back ((B,ad,b) -> (B,a,d,b) -> swap -> (B,abd)).
    Returns the Y_bsf the listing computes (§8c-3)."""
    a, b, c, d = check_pattern(p)
    X = np.asarray(X_bsf, dtype=np.float64)
    B = X.shape[0]
    Xp = X.reshape(B, a, c, d).transpose(0, 1, 3, 2).reshape(B, a * d, c)
    Kb = bmm_weights(p, K4)                                  # (ad, b, c)
    Yp = np.einsum("nqc,qbc->nqb", Xp, Kb, optimize=False)   # ad GEMMs (B x c)(c x b)
    return Yp.reshape(B, a, d, b).transpose(0, 1, 3, 2).reshape(B, a * b * d)


def einsum_matmul(p, K4, X_bsf) -> np.ndarray:
    """The 4-D contraction of App. A: Y[:,a,b,d] = sum_c X[:,a,c,d] K[a,b,c,d]."""
    a, b, c, d = check_pattern(p)
    X = np.asarray(X_bsf, dtype=np.float64)
    B = X.shape[0]
    K = np.asarray(K4, dtype=np.float64).reshape(a, b, c, d)
    Y = np.einsum("nicj,ikcj->nikj", X.reshape(B, a, c, d), K, optimize=False)
    return Y.reshape(B, a * b * d)


def alg2_tiles(p, K4, X_bsf) -> np.ndarray:
    """Alg. 2: for every (i,j), Y[:,row] += X[:,col] K^T[col,row]."""
    a, b, c, d = check_pattern(p)
    X = np.asarray(X_bsf, dtype=np.float64)
    D = dense(p, K4)
    M, N, _ = dims(p)
    Y = np.zeros((X.shape[0], M))
    for i in range(a):
        for j in range(d):
            row, col = tile_sets(p, i, j)
            Y[:, row] += X[:, col] @ D[np.ix_(row, col)].T
    return Y


# --------------------------------------------------------------------------
# FFT / Hadamard worked examples (Fig. 1; §8c-4)
# --------------------------------------------------------------------------
def bitrev(L: int) -> np.ndarray:
    """Bit-reversal permutation of 0..2^L-1."""
    n = np.arange(2 ** L)
    r = np.zeros_like(n)
    for bit in range(L):
        r |= ((n >> bit) & 1) << (L - 1 - bit)
    return r


def dft_factors(L: int):
    """Complex K4 values of the radix-2 decimation-in-time factors (§8c-4):
    K_l = I_{2^{l-1}} (x) [[I_d, W_d], [I_d, -W_d]],  d = 2^{L-l},
    W_d = diag(w^j), w = exp(-2 pi i / (2d)).  In canonical form
    K4[i,0,0,j] = 1, K4[i,0,1,j] = w^j, K4[i,1,0,j] = 1, K4[i,1,1,j] = -w^j.
    Then K_1 ... K_L = F_N R_N (DFT times bit reversal; Fig. 1 "up to a
    column permutation"), pinned against numpy.fft."""
    pats, vals = [], []
    for l in range(1, L + 1):
        a, d = 2 ** (l - 1), 2 ** (L - l)
        w = np.exp(-2j * np.pi * np.arange(d) / (2 * d))
        K = np.empty((a, 2, 2, d), dtype=np.complex128)
        K[:, 0, 0, :] = 1.0
        K[:, 0, 1, :] = w
        K[:, 1, 0, :] = 1.0
        K[:, 1, 1, :] = -w
        pats.append((a, 2, 2, d))
        vals.append(K)
    return pats, vals


def hadamard_factors(L: int):
    """Real dyadic factors with every 2x2 block [[1,1],[1,-1]]:
    their product is the Sylvester Hadamard matrix H_2^{(x)L}."""
    pats, vals = [], []
    for l in range(1, L + 1):
        a, d = 2 ** (l - 1), 2 ** (L - l)
        K = np.empty((a, 2, 2, d), dtype=np.float32)
        K[:, 0, 0, :] = 1.0
        K[:, 0, 1, :] = 1.0
        K[:, 1, 0, :] = 1.0
        K[:, 1, 1, :] = -1.0
        pats.append((a, 2, 2, d))
        vals.append(K)
    return pats, vals


def dense_complex(p, K4c) -> np.ndarray:
    """O-4: complex instantiation of O-1 (numpy, same index rule as O-1)."""
    a, b, c, d = check_pattern(p)
    M, N, _ = dims(p)
    D = np.zeros((M, N), dtype=np.complex128)
    K = np.asarray(K4c).reshape(a, b, c, d)
    for i in range(a):
        for k in range(b):
            for l in range(c):
                for j in range(d):
                    D[i * b * d + k * d + j, i * c * d + l * d + j] = K[i, k, l, j]
    return D


def split_complex_factor(K4c):
    """(Re K4, Im K4) as float32 arrays for the real/imag split of §8c GPU-vs-oracle (5)."""
    K4c = np.asarray(K4c)
    return K4c.real.astype(np.float32), K4c.imag.astype(np.float32)


# --------------------------------------------------------------------------
# byte / flop model (§4.3) and accuracy contract
# --------------------------------------------------------------------------
def io_elements_fused(p, B: int) -> int:
    """Elements the fused kernel moves on X and Y: B(N+M)."""
    M, N, _ = dims(p)
    return B * (N + M)


def io_elements_baseline(p, B: int) -> int:
    """permute-GEMM-permute: 2BN + (BN+BM) + 2BM = 3B(N+M)."""
    M, N, _ = dims(p)
    return 3 * B * (N + M)


def model_bytes(p, B: int, elem_bytes: int = 4) -> int:
    """Byte model of the metric: read X, read nnz(K), write Y."""
    M, N, nnz = dims(p)
    return elem_bytes * (B * N + nnz + B * M)


def model_flops(p, B: int) -> int:
    """Useful flops 2 B abcd."""
    return 2 * B * dims(p)[2]


def gelu(Y) -> np.ndarray:
    """GELU, the FFN activation of the paper's ViT-S/16 layer table (Table 7
    "2 x Linear + GELU + LN"; NEXT-2's optional epilogue): the exact form
    gelu(y) = y * Phi(y) = 0.5 * y * (1 + erf(y / sqrt 2)), FP64 (math.erf per
    element; the paper does not define it, R18)."""
    import math
    y = np.asarray(Y, dtype=np.float64)
    erf = np.vectorize(math.erf, otypes=[np.float64])
    return 0.5 * y * (1.0 + erf(y / math.sqrt(2.0)))


def normwise_error(Y_hat, Y_ref) -> float:
    """max |Y_hat - Y| / max |Y| over the tensor (§8c-10 reading of the
    north-star 'max relative error').  |.| is the modulus, so complex inputs
    (the Fig. 1 DFT check) compare real AND imaginary parts: both
    sides are promoted to complex128 when either is complex, else float64.
    The shapes must match exactly (no broadcasting)."""
    Y_hat = np.asarray(Y_hat)
    Y_ref = np.asarray(Y_ref)
    if Y_hat.shape != Y_ref.shape:
        raise ValueError(f"shape mismatch: {Y_hat.shape} vs {Y_ref.shape}")
    wide = np.complex128 if (np.iscomplexobj(Y_hat) or np.iscomplexobj(Y_ref)) else np.float64
    Y_hat = Y_hat.astype(wide)
    Y_ref = Y_ref.astype(wide)
    if Y_ref.size == 0:
        return 0.0
    den = float(np.max(np.abs(Y_ref)))
    num = float(np.max(np.abs(Y_hat - Y_ref)))
    if not (np.isfinite(num) and np.isfinite(den)):
        return float("inf")
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return num / den


def round_tf32_rna(x) -> np.ndarray:
    """Round float32 values to TF32 (10 explicit mantissa bits), to nearest with
    ties away from zero (the RNA rounding SURVEY §8c-11 fixes for packed K).
    Sign-magnitude encoding: adding half an ulp (bit 12) to the magnitude bits
    and truncating the low 13 bits rounds |x| half-up.  Finite inputs only."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def truncate_tf32(x) -> np.ndarray:
    """TF32 value of float32 bits read by a tensor core that ignores the 13
    low mantissa bits (round toward zero).  Finite inputs only."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (b & np.uint32(0xFFFFE000)).view(np.float32)


def envelope_delta(c: int, u_in: float, u: float = 2.0 ** -24) -> float:
    """Per-hop relative factor delta = 2 u_in + u_in^2 + gamma_{2c}
    (SURVEY §8c O-6): standard order-independent summation bound with slack."""
    n = 2 * c
    gamma = n * u / (1.0 - n * u)
    return 2 * u_in + u_in * u_in + gamma
