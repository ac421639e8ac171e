"""The paper's benchmark pattern grid (App. E.1, Fig.
"code-generate-patterns"), restated.

Two families are enumerated with batch size 25088 and an index-size cap of
2**31 - 1 on B*N, B*M and abcd:
  1. a = 1, (b, c) from the 48..1024 list with b = c, b = 4c or c = 4b,
     d from the 14-value list;
  2. a > 1 from the 14-value list, d in {4, 16, 64}, same (b, c) rule minus six
     excluded (b, c) pairs.
Only shapes come out of here.
"""
from __future__ import annotations

import itertools

GRID_BATCH = 25_088
SIZE_LIMIT = 2_147_483_647

A_VALUES = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128)
BC_VALUES = (48, 64, 96, 128, 192, 256, 384, 512, 768, 1024)
D_VALUES_A1 = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128)
D_VALUES_AGT1 = (4, 16, 64)
EXCLUDED_BC = ((1024, 256), (256, 1024), (128, 512), (512, 128), (64, 256), (256, 64))


def _shape_ok(b: int, c: int) -> bool:
    return b == c or b == 4 * c or c == 4 * b


def _fits(a: int, b: int, c: int, d: int) -> bool:
    B = GRID_BATCH
    return (B * a * c * d <= SIZE_LIMIT and B * a * b * d <= SIZE_LIMIT
            and a * b * c * d <= SIZE_LIMIT)


def paper_grid() -> list[tuple[int, int, int, int]]:
    """All patterns the generator emits, in emission order (duplicates kept)."""
    out = []
    for b, c, d in itertools.product(BC_VALUES, BC_VALUES, D_VALUES_A1):
        if _shape_ok(b, c) and _fits(1, b, c, d):
            out.append((1, b, c, d))
    for a, b, c, d in itertools.product(A_VALUES, BC_VALUES, BC_VALUES, D_VALUES_AGT1):
        if a != 1 and (b, c) not in EXCLUDED_BC and _shape_ok(b, c) and _fits(a, b, c, d):
            out.append((a, b, c, d))
    return out


def sweep_patterns() -> list[tuple[int, int, int, int]]:
    """BASELINE.json configs[2]: grid subset with b = c in {48,64,96,128} and a*d <= 64.

    Sorted, de-duplicated (SURVEY.md §8d workload 3: 88 patterns).
    """
    keep = set()
    for (a, b, c, d) in paper_grid():
        if b == c and b in (48, 64, 96, 128) and a * d <= 64:
            keep.add((a, b, c, d))
    return sorted(keep, key=lambda p: (p[1], p[0], p[3]))
