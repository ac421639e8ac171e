"""Batch partitioning across GPUs: rows of X are independent, so
each rank owns a contiguous batch shard and runs the unchanged single-GPU
path on it -- there is no collective on the compute path.  torch.distributed
(NCCL on GPUs, gloo on CPU for tests) is used only for the timing barrier /
max reduction and to gather result shards for verification.
"""
from __future__ import annotations

import os


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_bounds(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of a batch of B rows for `rank` of `world`:
    the first B % world ranks get one extra row; shards cover [0, B) exactly."""
    if world < 1 or not (0 <= rank < world) or B < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(B, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity if not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, B: int, layout: str = "bsf"):
    """Reassemble a batch from per-rank contiguous shards (verification only).

    local: this rank's (rows x M) tensor for BSF, (M x rows) for BSL.
    Returns the full (B x M) / (M x B) tensor on every rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
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
