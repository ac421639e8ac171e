"""Batch partitioning across GPUs: rows of X are independent
(Y[n,:] depends only on X[n,:]), so the configuration's global
batch B is split into contiguous shards, B_g = ceil(B/G) rows per rank (the
last ranks one row fewer), and each rank runs the unchanged single-GPU path on
its shard -- there is no collective on the compute path.  torch.distributed
(NCCL on GPUs, gloo on CPU for tests) carries only the timing barrier / max
reduction, the byte totals, and sampled result rows gathered to rank 0 for
verification.  bench.py's multi-GPU leg is built from these functions, and
tests/test_dist_gloo.py drives the same functions at world size 2.
"""
from __future__ import annotations

import os

import numpy as np


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _dist_on():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def shard_bounds(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of a batch of B rows for `rank` of `world`:
    the first B % world ranks get one extra row (B_g = ceil(B / world));
    shards cover [0, B) exactly."""
    if world < 1 or not (0 <= rank < world) or B < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(B, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def sample_rows(lo: int, hi: int, k: int = 4) -> np.ndarray:
    """k global row indices of the shard [lo, hi) to verify: first, second,
    middle and last row (repeated when the shard is shorter; all -1 when it is
    empty).  Fixed length so every rank contributes the same tensor shape."""
    if hi <= lo:
        return np.full(k, -1, dtype=np.int64)
    cand = [lo, lo + 1, (lo + hi) // 2, hi - 1] + [hi - 1] * max(0, k - 4)
    rows = [min(max(r, lo), hi - 1) for r in cand[:k]]
    return np.asarray(rows, dtype=np.int64)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity if not distributed."""
    import torch
    import torch.distributed as dist
    if not _dist_on():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """Sum of a per-rank scalar (bytes moved) over all ranks; identity if not distributed."""
    import torch
    import torch.distributed as dist
    if not _dist_on():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_samples(rows: np.ndarray, values):
    """All-gather every rank's sampled rows (k global indices) and their
    result values (k x M tensor, BSF order) -> (rows_all (G*k,), vals_all
    (G*k x M) numpy float64) on every rank.  Verification only."""
    import torch
    import torch.distributed as dist
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=values.device)
    if not _dist_on():
        return r.cpu().numpy(), values.double().cpu().numpy()
    world = dist.get_world_size()
    rs = [torch.empty_like(r) for _ in range(world)]
    vs = [torch.empty_like(values) for _ in range(world)]
    dist.all_gather(rs, r)
    dist.all_gather(vs, values.contiguous())
    return torch.cat(rs).cpu().numpy(), torch.cat(vs).double().cpu().numpy()


def check_samples(rows_all: np.ndarray, vals_all: np.ndarray, ref_fn, err_fn) -> dict:
    """Compare gathered sample rows with a reference computed for those global
    rows: ref_fn(rows) -> (len(rows) x M) array; err_fn(got, ref) -> float.
    Empty-shard placeholders (-1) are skipped; duplicates are checked once."""
    keep = {}
    for i, r in enumerate(rows_all.tolist()):
        if r >= 0 and r not in keep:
            keep[r] = i
    rows = np.array(sorted(keep), dtype=np.int64)
    got = vals_all[[keep[r] for r in rows]]
    err = float(err_fn(got, ref_fn(rows))) if rows.size else 0.0
    return {"rows_checked": int(rows.size), "max_normwise_err": err}


def gather_rows(local, B: int, layout: str = "bsf"):
    """Reassemble a batch from per-rank contiguous shards (verification only).

    local: this rank's (rows x M) tensor for BSF, (M x rows) for BSL.
    Returns the full (B x M) / (M x B) tensor on every rank."""
    import torch
    import torch.distributed as dist
    if not _dist_on():
        return local
    world = dist.get_world_size()
    bsf = layout == "bsf"
    M = local.shape[1] if bsf else local.shape[0]
    sizes = [shard_bounds(B, world, r) for r in range(world)]
    maxrows = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxrows, M) if bsf else (M, maxrows), dtype=local.dtype, device=local.device)
    if bsf:
        pad[: local.shape[0]] = local
    else:
        pad[:, : local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    if bsf:
        return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)
    return torch.cat([p[:, : hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=1)
