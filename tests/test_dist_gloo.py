"""Multi-process (world size 2, gloo, CPU) tests of the batch-partitioned path.

There is no GPU in this container, so the per-rank compute is a CPU stand-in;
what is under test is the host-side code the N>1 bench runs: bench.py's
shard_input / verify_sharded and dist.py's shard bounds, sample gather,
max / sum over ranks, and gathering shards back in both layouts.
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
from paper_2405_15013_b200 import dist as kdist
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


# ---------------------------------------------------------------------------
# bench.py's own multi-GPU bookkeeping (shard_input -> per-rank compute ->
# verify_sharded / max_over_ranks / sum_over_ranks), driven at world size 2.
# The per-rank "kernel" is a torch CPU matmul with a dense K assembled here
# (not the oracle); the oracle only checks, exactly as in bench.py.
# ---------------------------------------------------------------------------
def _dense_local(p, K4):
    a, b, c, d = p
    D = np.zeros((a * b * d, a * c * d))
    for i in range(a):
        for k in range(b):
            for l in range(c):
                for j in range(d):
                    D[i * b * d + k * d + j, i * c * d + l * d + j] = K4[i, k, l, j]
    return torch.from_numpy(D)


def _bench_worker(rank, world, port, out, corrupt, layout, B):
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pats = [(2, 3, 4, 2), (1, 8, 6, 2)]               # chain: (1,8,6,2) applied first, N = 12 -> 16 -> 12
        K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
        N = 12
        lo, hi, Xb, Xl = bench.shard_input(B, N, rank, world, layout)
        assert Xb.shape == (hi - lo, N)
        Z = torch.from_numpy(Xb.astype(np.float64))
        for p, k in zip(reversed(pats), reversed(K4s)):
            Z = Z @ _dense_local(p, k).T
        Yl = Z.float()
        if corrupt and rank == 1:
            Yl = Yl + 1.0
        if layout == "bsl":
            Yl = Yl.t().contiguous()
        rec = bench.verify_sharded(Yl, lo, hi, layout, bench.oracle_ref(pats, K4s, N), 1e-5, O.normwise_error,
                                   check=rank == 0)
        tmax = kdist.max_over_ranks(2.0 + rank)
        tsum = kdist.sum_over_ranks(hi - lo)
        if rank == 0:
            out.put((rec, tmax, tsum))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
@pytest.mark.parametrize("layout,B", [("bsf", 11), ("bsl", 9), ("bsf", 1)])
def test_bench_sharded_verify_world2(corrupt, layout, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q, corrupt, layout, B)) for r in range(2)]
    for pr in procs:
        pr.start()
    rec, tmax, tsum = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert tmax == 3.0 and tsum == B                      # max time, all ranks' rows
    assert rec["ranks"] == 2
    assert rec["rows_checked"] == min(B, 8) or rec["rows_checked"] >= min(B, 3)
    if corrupt and B > 1:
        assert not rec["ok"] and rec["max_normwise_err"] > 1e-3
    else:
        assert rec["ok"], rec
