"""Seeded input generators (App. E.1 "Matrix Entries").

* X entries:   i.i.d. N(0, 1)
* K nonzeros:  i.i.d. U[-1/sqrt(c), 1/sqrt(c)]

K is always produced in the canonical (a, b, c, d) order with d fastest
(the einsum packing of PAPER.md:860-861), which is the boundary format of
``ks_pack_weights``.  Nothing here knows how K acts on X.

Seeds: X -> 0, factor l -> 1000 + l, integer variants -> 2000+.
All generation is on the host with numpy's PCG64 so the GPU and the oracle
see identical bytes.
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def x_normal(B: int, N: int, seed: int = 0) -> np.ndarray:
    """B x N float32 batch-size-first matrix, entries i.i.d. N(0,1)."""
    return _rng(seed).standard_normal((B, N), dtype=np.float32)


def x_rows_normal(rows, N: int, seed: int = 0) -> np.ndarray:
    """Counter-based rows: row n is drawn from its own stream (seed, n).

    Lets a caller materialise any subset of rows of a huge virtual batch
    (the oracle checks sampled rows of full-size outputs) with the same
    bytes the full generator would give.
    """
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((rows.size, N), dtype=np.float32)
    for t, n in enumerate(rows):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(n)])))
        out[t] = g.standard_normal(N, dtype=np.float32)
    return out


def k4_uniform(a: int, b: int, c: int, d: int, seed: int) -> np.ndarray:
    """Canonical (a,b,c,d) float32 nonzeros, i.i.d. U[-1/sqrt(c), 1/sqrt(c)]."""
    lim = 1.0 / np.sqrt(float(c))
    v = _rng(seed).uniform(-lim, lim, size=(a, b, c, d))
    return v.astype(np.float32)


def x_int(B: int, N: int, seed: int = 2000, lo: int = -2, hi: int = 2) -> np.ndarray:
    """Small-integer X (exact in FP32 and TF32)."""
    return _rng(seed).integers(lo, hi + 1, size=(B, N)).astype(np.float32)


def k4_int(a: int, b: int, c: int, d: int, seed: int = 2001, lo: int = -1, hi: int = 1) -> np.ndarray:
    """Small-integer canonical K values (exact in FP32 and TF32)."""
    return _rng(seed).integers(lo, hi + 1, size=(a, b, c, d)).astype(np.float32)


def k4_labels(a: int, b: int, c: int, d: int) -> np.ndarray:
    """Distinct integer labels 1..abcd (exact in FP32 while abcd < 2**24).

    Used with one-hot X rows to read the device's support/value mapping
    bit-exactly.
    """
    n = a * b * c * d
    if n >= (1 << 24):
        raise ValueError("labels would not be exact in fp32")
    return np.arange(1, n + 1, dtype=np.float32).reshape(a, b, c, d)


def to_bsl(X_bsf: np.ndarray) -> np.ndarray:
    """Batch-size-last copy (N x B row-major) of a batch-size-first matrix."""
    return np.ascontiguousarray(X_bsf.T)


def from_bsl(X_bsl: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(X_bsl.T)
