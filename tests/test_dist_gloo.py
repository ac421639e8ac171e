"""Multi-process (world size 2, gloo, CPU) tests of the batch-partitioned path.

The GPU compute step is replaced by the CPU oracle here (there is no GPU in
this container); what is under test is the host-side logic the N>1 bench and
verification use: shard bounds, max-over-ranks timing, and gathering shards
back into the full batch in both layouts.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ksgen
import oracle as O
from paper_2405_15013_b200.dist import gather_rows, max_over_ranks, shard_bounds


def test_shard_bounds_cover_batch():
    for B in (0, 1, 7, 8, 8192, 25087):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(5, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = (2, 3, 2, 4)
        M, N, _ = O.dims(p)
        B = 11
        K4 = ksgen.k4_uniform(*p, seed=1001)
        X = ksgen.x_normal(B, N, seed=0)
        lo, hi = shard_bounds(B, world, rank)
        # per-rank "compute": the shard only
        Yl = torch.from_numpy(O.matmul(p, K4, X[lo:hi]).astype(np.float32))
        Yf = gather_rows(Yl, B, "bsf")
        Ybsl = gather_rows(Yl.t().contiguous(), B, "bsl")
        t = max_over_ranks(1.0 + rank)
        if rank == 0:
            full = O.matmul(p, K4, X).astype(np.float32)
            out.put((np.array_equal(Yf.numpy(), full), np.array_equal(Ybsl.numpy(), full.T), t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_gather_and_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    bsf_ok, bsl_ok, tmax = res
    assert bsf_ok and bsl_ok
    assert tmax == 2.0
