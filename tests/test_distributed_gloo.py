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
