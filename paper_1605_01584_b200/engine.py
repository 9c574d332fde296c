"""One-call entry point: the drop-in for ``paircorr.allpairs``.

Mirrors ``paircorr.engine`` (/root/reference/pkg/src/paircorr/engine.py:1-56).
``allpairs`` keeps the reference signature and result type; the scheduling
knobs (``tile_size``, ``capacity``, ``threads``, ``backend``,
``buffer_budget``) are validated as the reference validates them and, as the
reference promises (engine.py:32-37), never change a bit of the result.

Single-device data flow (stream.py; one host synchronisation at the end):

    X (host; pinned -> asynchronous) --copy-in stream, bottom rows first--> X_dev
    K1 normalize per arrived chunk (csrc/normalize.cuh)     X_dev -> U (padded), flags
    K2 contraction passes from the last tile backwards      U -> packed[n(n+1)/2] (device)
       (csrc/syrk.cuh, packed epilogue)
    completed packed rows --copy-out stream--> host, overlapped with later passes

This is the paper's Alg. 2 (asynchronous double-buffered passes,
PAPER.md:235-287) with the device array as the staging buffer.
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._device import as_device_f64, nvtx, ptr, resolve_devices, stream_handle
from .distributed import BACKENDS, run_workers
from .indexing import sym_job_count
from .stream import run_stream
from .tiles import DEFAULT_TILE_SIZE, CorrelationResult, TileGeometry
from .transform import Dataset, normalize_device

__all__ = ["allpairs", "default_capacity", "DEFAULT_BUFFER_BUDGET"]

DEFAULT_BUFFER_BUDGET = 256 * 2**20  # engine.py:14


def default_capacity(t: int, buffer_budget: int | None = None) -> int:
    """Largest per-pass tile count whose two buffers fit the budget (engine.py:17-20)."""
    budget = DEFAULT_BUFFER_BUDGET if buffer_budget is None else buffer_budget
    return max(1, budget // (2 * t * t * 8))


def _host_out(out, total: int) -> torch.Tensor:
    if out is None:
        return torch.from_numpy(np.empty(total, dtype=np.float64))
    t = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
    if t.device.type != "cpu" or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("out must be a contiguous float64 host array")
    if t.numel() < total:
        raise ValueError(f"out holds {t.numel()} values, need {total}")
    return t


_SMALL_BYTES = 64 << 20  # X + packed result below this: no streaming (measured crossover between c1 and c3)


def _device_result_budget(device: torch.device, n: int, l: int, method: str = "tensor") -> int:
    """Bytes the packed result may take on ``device``: free memory minus X, U
    (plus the split method's digit planes) and a margin
    (``PCC_DEVICE_RESULT_BUDGET`` overrides, for tests)."""
    env = os.environ.get("PCC_DEVICE_RESULT_BUDGET")
    if env:
        return int(env)
    free, _ = torch.cuda.mem_get_info(device)
    L = _lib.lib()
    xu = n * l * 8 + int(L.pcc_rows_padded(n)) * int(L.pcc_ldu(l)) * 8
    if method == "split":
        xu += int(L.pcc_split_slice_bytes(n, l)) + 8 * int(L.pcc_rows_padded(n))
    return max(0, int(0.9 * free) - xu - (1 << 30))


def _allpairs_windowed(x_host, n: int, l: int, device: torch.device, host: torch.Tensor, window: int,
                       method: str) -> torch.Tensor:
    """Packed result larger than the device budget: GPU tile passes whose
    packed span fits ``window`` doubles, each contracted into one of two
    device windows (``out_base`` = the pass's span start) and its owned
    cells (``owned_runs``) copied to ``host`` while the next pass computes --
    the reference's bounded-memory pass model (pipeline.py:109-170) at GPU
    tile granularity.  Returns the device zero-variance flags."""
    from .distributed import owned_runs, shard_span

    L = _lib.lib()
    x = as_device_f64(x_host, device)
    u, flags = normalize_device(x)
    del x
    T = int(L.pcc_gpu_tile_count(n))
    mg = -(-n // _lib.GPU_TILE)
    row_tiles = mg  # a pass always holds at least one tile row's worth of cells
    window = max(window, shard_span(n, 0, min(T, row_tiles))[1])
    passes = []
    tb = 0
    while tb < T:  # largest te with span(tb, te) <= window (binary search)
        lo_te, hi_te = tb + 1, T
        while lo_te < hi_te:
            mid = (lo_te + hi_te + 1) // 2
            a, b = shard_span(n, tb, mid)
            if b - a <= window:
                lo_te = mid
            else:
                hi_te = mid - 1
        passes.append((tb, lo_te))
        tb = lo_te
    compute = torch.cuda.current_stream(device)
    copy = torch.cuda.Stream(device)
    bufs = [torch.empty(window, dtype=torch.float64, device=device) for _ in range(min(2, len(passes)))]
    freed = [None] * len(bufs)
    pinned = host.is_pinned()
    con = _lib.Contraction(method, u, n, l).prepare_all(stream_handle(compute))
    for k, (tb, te) in enumerate(passes):
        b = k % len(bufs)
        if freed[b] is not None:
            compute.wait_event(freed[b])  # the window's previous downloads are done
        span_lo, _ = shard_span(n, tb, te)
        con.syrk(tb, te, _lib.LAYOUT_PACKED, ptr(bufs[b]), 0, span_lo, 0, 0, 0, stream_handle(compute),
                 "allpairs(windowed)")
        done = torch.cuda.Event()
        done.record(compute)
        copy.wait_event(done)
        with torch.cuda.stream(copy):
            for ra, rb in owned_runs(n, tb, te):
                host[ra:rb].copy_(bufs[b][ra - span_lo:rb - span_lo], non_blocking=pinned)
            freed[b] = torch.cuda.Event()
            freed[b].record(copy)
    copy.synchronize()
    compute.synchronize()
    return flags


def _allpairs_one_device(dataset: Dataset, device: torch.device, keep_on_device: bool, out, chunk_rows: int,
                         output: str, method: str = "tensor"):
    n, l = dataset.n, dataset.l
    L = _lib.lib()
    with torch.cuda.device(device):
        if output == "dense":
            compute = torch.cuda.current_stream()
            x = as_device_f64(dataset.values, device)
            u, flags = normalize_device(x)
            T = int(L.pcc_gpu_tile_count(n))
            dense = torch.empty((n, n), dtype=torch.float64, device=device)
            con = _lib.Contraction(method, u, n, l).prepare_all(stream_handle(compute))
            con.syrk(0, T, _lib.LAYOUT_DENSE, ptr(dense), n, 0, 0, 0, 0, stream_handle(compute), "allpairs(dense)")
            zv = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
            return (dense if keep_on_device else dense.cpu().numpy()), zv

        total = sym_job_count(n)
        T = int(L.pcc_gpu_tile_count(n))
        # cudaMemGetInfo costs ~0.2 ms: only results that could approach the
        # device's capacity are checked against the free memory
        check = total * 8 > (1 << 30) or "PCC_DEVICE_RESULT_BUDGET" in os.environ
        budget = _device_result_budget(device, n, l, method) if check else total * 8
        if not keep_on_device and total * 8 > budget:
            # the packed result does not fit the device next to X and U: bounded
            # device windows, each pass downloaded into the host result
            host = _host_out(out, total)
            flags = _allpairs_windowed(dataset.values, n, l, device, host, budget // 8, method)
            zv = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
            return (out if out is not None else host.numpy()), zv
        packed = torch.empty(total, dtype=torch.float64, device=device)
        host = None if keep_on_device else _host_out(out, total)
        if n * l * 8 + total * 8 <= _SMALL_BYTES:
            # small problem: one upload, K1, one contraction launch, one
            # download -- the streamed plan's extra launches and events cost
            # more than they overlap here (c1: 1.0 -> 0.6 ms)
            compute = torch.cuda.current_stream()
            x = as_device_f64(dataset.values, device)
            u, flags = normalize_device(x)
            con = _lib.Contraction(method, u, n, l).prepare_all(stream_handle(compute))
            con.syrk(0, T, _lib.LAYOUT_PACKED, ptr(packed), 0, 0, 0, 0, 0, stream_handle(compute), "allpairs")
            if host is not None:
                host.copy_(packed, non_blocking=host.is_pinned())
            compute.synchronize()
        else:
            _, flags, _ = run_stream(dataset.values, n, l, device, 0, T, packed, 0, host, 0, chunk_rows=chunk_rows,
                                     method=method)
        zv = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
        if keep_on_device:
            return packed, zv
        return (out if out is not None else host.numpy()), zv


def allpairs(
    dataset: Dataset | str | Path,
    tile_size: int = DEFAULT_TILE_SIZE,
    capacity: int | None = None,
    threads: int = 1,
    workers: int = 1,
    backend: str = "in_process",
    buffer_budget: int | None = None,
    *,
    devices=None,
    output: str = "packed",
    keep_on_device: bool = False,
    out=None,
    chunk_rows: int = 8,
    exact: bool = False,
    method: str | None = None,
):
    """All-pairs Pearson correlation of ``dataset`` on B200 GPUs (engine.py:23-56).

    Reference arguments keep their meaning and validation; ``workers > 1``
    splits the GPU tile range across that many workers (one host thread
    each, round-robin over ``devices``); ``backend="subprocess"`` runs them
    as GPU worker processes speaking the reference's framed protocol
    (``run_workers``, as engine.py:46-56 routes it).  Extensions:

    * ``devices``: ``None`` (current device), a device count, or a list;
    * ``output``: ``"packed"`` (reference layout, returns ``CorrelationResult``)
      or ``"dense"`` (returns the full ``n x n`` matrix and the zero-variance
      set, written by the same kernel's dense epilogue);
    * ``keep_on_device``: leave the packed result on the GPU (a CUDA tensor
      in ``CorrelationResult.packed``);
    * ``out``: caller-owned host float64 buffer for the packed result (pinned
      memory makes the device-to-host copies asynchronous);
    * ``chunk_rows``: upload granularity in 128-row GPU tile rows; each
      uploaded chunk releases one contraction pass (``stream.plan_stream``);
    * ``exact``: compute every coefficient in the reference's own arithmetic
      (``dot8``: separately rounded products, eight lane sums, fixed tree) on
      the FP64 CUDA cores -- the packed result is bit-identical to
      ``paircorr.allpairs`` -- instead of on the FP64 tensor cores (within
      1e-12, about twice as fast);
    * ``method``: the contraction -- ``"tensor"`` (default, FP64 tensor
      cores), ``"split"`` (int8 tensor cores on exact radix-128 digit planes
      of the normalised rows, FP64-accurate: within 1e-12 of the reference,
      ~2.4x the tensor path's speed; l <= 8192) or ``"exact"`` (same as
      ``exact=True``).
    """
    with nvtx("pcc.allpairs"):
        return _allpairs(dataset, tile_size, capacity, threads, workers, backend, buffer_budget, devices, output,
                         keep_on_device, out, chunk_rows, exact, method)


def _allpairs(dataset, tile_size, capacity, threads, workers, backend, buffer_budget, devices, output, keep_on_device,
              out, chunk_rows, exact, method):
    source = dataset  # a path stays a path for subprocess workers (engine.py:55-56)
    if not isinstance(dataset, Dataset):
        from .fileio import load_dataset

        dataset = load_dataset(dataset)
    geom = TileGeometry(n=dataset.n, t=tile_size)  # validates tile_size like the reference
    if capacity is None:
        capacity = default_capacity(tile_size, buffer_budget)
    if capacity < 1:
        raise ValueError(f"capacity must be >= 1, got {capacity}")
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}, expected one of {BACKENDS}")
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    if output not in ("packed", "dense"):
        raise ValueError(f"output must be 'packed' or 'dense', got {output!r}")
    method = _lib.resolve_method(method, exact)
    _lib.check_method_shape(method, dataset.l)
    devs = resolve_devices(devices)
    if backend == "subprocess":
        # the reference routes workers > 1 or backend != "in_process" to
        # run_workers(dataset, geom, workers, backend, capacity, threads)
        # (engine.py:46-56): GPU worker processes on the framed protocol
        if output != "packed" or keep_on_device:
            raise ValueError("backend='subprocess' returns the gathered packed result "
                             "(output='packed', keep_on_device=False)")
        return run_workers(source, geom, workers, "subprocess", capacity, threads, devices=devs, method=method)
    if (workers > 1 or len(devs) > 1) and output == "packed" and not keep_on_device:
        return run_workers(dataset, geom, max(workers, len(devs)), backend="cuda", devices=devs, out=out,
                           method=method)
    if workers > 1 or len(devs) > 1:
        raise ValueError("multi-worker runs support output='packed' gathered to host "
                         "(use run_workers(..., gather=False) for device-resident shards)")
    res, zv = _allpairs_one_device(dataset, devs[0], keep_on_device, out, chunk_rows, output, method)
    if output == "dense":
        return res, zv
    return CorrelationResult(n=dataset.n, packed=res, zero_variance=zv)
