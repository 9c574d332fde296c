"""The N>1 path's host logic on CPU with torch.distributed (gloo, world_size 2):
every rank takes its partition(T, N) share of the GPU tile jobs, produces its
packed shard (values from the CPU oracle standing in for the device kernel,
one dot8 per owned cell), rank 0 gathers the shards through owned_runs and
must reproduce the single-worker packed result bit for bit; the
max-over-ranks timing reduction is exercised the way bench.py uses it."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1605_01584_b200.distributed import owned_runs, partition, shard_span

from conftest import random_values


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_values(u, n, runs, base, span):
    vals = np.full(span, np.nan)
    for lo, hi in runs:
        for idx in range(lo, hi):
            # packed index -> (y, x) by row walk
            y = _row_of(n, idx)
            x = idx - ((y * (2 * n + 1 - y)) >> 1) + y
            vals[idx - base] = oracle.dot8(u[y], u[x])
    return vals


def _row_of(n, idx):
    lo, hi = 0, n - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if (mid * (2 * n + 1 - mid)) >> 1 <= idx:
            lo = mid
        else:
            hi = mid - 1
    return lo


def _worker(rank, world, port, n, l, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = random_values(np.random.default_rng(5), n, l, special_rows=True)
        u, _ = oracle.normalize(x, threads=1)
        mg = -(-n // 128)
        T = mg * (mg + 1) // 2
        tb, te = partition(T, world)[rank]
        lo, hi = shard_span(n, tb, te)
        runs = owned_runs(n, tb, te)
        vals = _shard_values(u, n, runs, lo, max(0, hi - lo))
        gathered = [None] * world
        dist.all_gather_object(gathered, (tb, te, lo, vals))
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            packed = np.full(n * (n + 1) // 2, np.nan)
            for tb_r, te_r, base, v in gathered:
                for a, b in owned_runs(n, tb_r, te_r):
                    packed[a:b] = v[a - base:b - base]
            ref, _ = oracle.allpairs(x, t=4, threads=1)
            result_q.put((bool(np.array_equal(packed, ref)), float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,l", [(300, 9), (257, 5)])
def test_two_rank_sharded_allpairs_reassembles_bitwise(n, l):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, l, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    equal, tmax = q.get(timeout=10)
    assert equal
    assert tmax == float(world)


def _exchange_worker(rank, world, port, n, l, result_q):
    """Exchange mode: each rank fills only its row_slices block (the CPU
    oracle's normalisation standing in for K1 on that block), exchange_rows
    all-gathers the blocks; every rank must then hold the oracle's full U,
    zero pad rows and the full zero-variance flags."""
    from paper_1605_01584_b200.distributed import exchange_rows, row_slices

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = random_values(np.random.default_rng(7), n, l, special_rows=True)
        u_ref, zv_ref = oracle.normalize(x, threads=1)
        slices, S = row_slices(n, world)
        r0, r1 = slices[rank]
        ldu = -(-l // 32) * 32
        u = torch.full((world * S, ldu), float("nan"), dtype=torch.float64)
        flags = torch.full((world * S,), 7, dtype=torch.uint8)
        blk = slice(rank * S, (rank + 1) * S)
        u[blk] = 0.0
        flags[blk] = 0
        if r1 > r0:
            ub, zb = oracle.normalize(x[r0:r1], threads=1)
            u[r0:r1, :l] = torch.from_numpy(ub)
            flags[r0:r1] = torch.from_numpy(zb.astype(np.uint8))
        exchange_rows(u, flags, S, rank, world)
        ok = (torch.equal(u[:n, :l], torch.from_numpy(u_ref)) and bool((u[:n, l:] == 0).all())
              and bool((u[n:] == 0).all()) and torch.equal(flags[:n], torch.from_numpy(zv_ref.astype(np.uint8)))
              and bool((flags[n:] == 0).all()))
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if rank == 0:
            result_q.put(all(oks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,l", [(2, 300, 9), (2, 100, 5), (3, 700, 6)])
def test_row_exchange_reassembles_u(world, n, l):
    from paper_1605_01584_b200.distributed import row_slices

    slices, S = row_slices(n, world)
    assert S % 128 == 0 and world * S >= -(-n // 128) * 128
    assert slices[0][0] == 0 and slices[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(slices, slices[1:]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, n, l, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10)
