"""Workload shapes of BASELINE.json ``configs`` (pattern tuples + batch sizes).

Chains are listed in the paper's product order K_1, ..., K_L (handles[0] =
K_1); they are *applied* K_L first because Y = X K_L^T ... K_1^T
(SURVEY.md §8c-5).  Only shapes live here.
"""
from __future__ import annotations

from .grid import GRID_BATCH, sweep_patterns  # noqa: F401

# configs[0]: "(2,4,4,2), N=M=32, B=8" -- (2,4,4,2) gives N=M=16;
# the two N=M=32 neighbours are run too.
TINY_PATTERNS = [(2, 4, 4, 2), (2, 4, 4, 4), (4, 4, 4, 2)]
TINY_BATCH = 8

# configs[1]: FFT-style butterfly chain, N = 4096, 12 factors (Fig. 1).
FFT_L = 12
FFT_BATCH = 8192


def dyadic_patterns(L: int) -> list[tuple[int, int, int, int]]:
    """(2^{l-1}, 2, 2, 2^{L-l}) for l = 1..L (Table 3)."""
    return [(2 ** (l - 1), 2, 2, 2 ** (L - l)) for l in range(1, L + 1)]


# configs[2]: sweep, B = 25088.
SWEEP_BATCH = GRID_BATCH

# configs[3]: ViT-S/16 MLP KSLinear, batch 128 x 196 tokens.
VIT_BATCH = 25_088
VIT_UP = [(1, 768, 192, 2), (6, 64, 64, 1)]          # 384 -> 1536
VIT_DOWN = [(1, 128, 128, 3), (6, 64, 256, 1)]       # 1536 -> 384 (chainable order, §8c-6)

# configs[4]: GPT-2 medium MLP, seq 1024 x batch 64.
GPT2_BATCH = 65_536
GPT2_DOWN = [(1, 64, 256, 16), (64, 64, 64, 1)]      # 4096 -> 1024 (paper's patterns)
GPT2_UP = [(64, 64, 64, 1), (1, 256, 64, 16)]        # 1024 -> 4096 (transposed, §8c-7)


def chain_dims(patterns) -> list[int]:
    """[N_L, M_L(=N_{L-1}), ..., M_1]: feature sizes along the application order."""
    a, b, c, d = patterns[-1]
    dims = [a * c * d]
    for (a, b, c, d) in reversed(patterns):
        dims.append(a * b * d)
    return dims


def chainable(patterns) -> bool:
    """a_l c_l d_l == a_{l+1} b_{l+1} d_{l+1}."""
    for p, q in zip(patterns[:-1], patterns[1:]):
        if p[0] * p[2] * p[3] != q[0] * q[1] * q[3]:
            return False
    return True
