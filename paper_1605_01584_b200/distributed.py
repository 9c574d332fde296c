"""Static distribution of GPU tile jobs across devices.

Mirrors ``paircorr.distributed`` (/root/reference/pkg/src/paircorr/distributed.py):
``partition`` is the reference's rule verbatim in meaning -- ``p``
contiguous chunks of ``ceil(T/p)`` tile ids, trailing workers possibly empty
(distributed.py:76-92; the paper's static distribution) --
applied to the 128 x 128 GPU tile matrix.  A worker is one GPU driven by one
host thread (ctypes releases the GIL).  With several devices each device
uploads only its block of rows of X and one broadcast normalisation kernel
writes the normalised rows into every device's U over NVLink peer memory
(``normalize_on_devices``); the workers then contract only their tile
ranges, so there is no collective in the contraction.
Results stay sharded on the devices (``ShardedResult``) or are gathered
into one packed host array; every packed cell belongs to exactly one tile
and every tile to exactly one worker, so the gathered result is bitwise
identical for any worker count.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import tempfile
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._device import as_device_f64, nvtx, ptr, resolve_devices, stream_handle
from .errors import IntegrityError, WorkerError
from .indexing import sym_job_coord, sym_job_count
from .tiles import CorrelationResult, TileGeometry
from .stream import run_stream
from .transform import Dataset, normalize_device

__all__ = [
    "BACKENDS",
    "WorkerAssignment",
    "WorkerReport",
    "merge",
    "Shard",
    "ShardedResult",
    "partition",
    "make_assignments",
    "shard_span",
    "owned_runs",
    "run_workers",
    "compute_worker",
    "check_coverage",
    "row_slices",
    "exchange_rows",
    "exchange_normalize",
    "clear_exchange_cache",
]

BACKENDS = ("in_process", "subprocess", "cuda")


def partition(total_tiles: int, p: int) -> list[tuple[int, int]]:
    """``p`` contiguous ranges covering ``[0, total_tiles)`` (distributed.py:76-92)."""
    if p < 1:
        raise ValueError(f"worker count must be >= 1, got {p}")
    if total_tiles < 0:
        raise ValueError(f"total tile count must be >= 0, got {total_tiles}")
    chunk = -(-total_tiles // p) if total_tiles else 0
    return [(min(total_tiles, i * chunk), min(total_tiles, (i + 1) * chunk)) for i in range(p)]


@dataclass(frozen=True)
class WorkerAssignment:
    """Tile range of one worker (distributed.py:55-64); ``geometry`` is the GPU tile geometry."""

    worker_index: int
    start: int
    stop: int
    geometry: TileGeometry
    capacity: int = 0

    @property
    def tile_count(self) -> int:
        return self.stop - self.start


@dataclass
class WorkerReport:
    """Blocks a worker delivered (distributed.py:67-73), for ``merge``."""

    worker_index: int
    tiles_done: int = 0
    blocks: list = field(default_factory=list)
    status: str = "ok"
    message: str = ""


def gpu_geometry(n: int) -> TileGeometry:
    return TileGeometry(n=n, t=_lib.GPU_TILE)


def make_assignments(geom: TileGeometry, p: int, capacity: int = 0) -> list[WorkerAssignment]:
    """distributed.py:95-99 over ``geom`` (normally the GPU geometry)."""
    return [WorkerAssignment(i, lo, hi, geom, capacity) for i, (lo, hi) in enumerate(partition(geom.total_tiles, p))]


def _F(n: int, y: int) -> int:
    return (y * (2 * n + 1 - y)) >> 1


def shard_span(n: int, tile_begin: int, tile_end: int) -> tuple[int, int]:
    """Packed-index span ``[lo, hi)`` covering every cell of GPU tiles ``[tile_begin, tile_end)``."""
    if tile_end <= tile_begin:
        return (0, 0)
    T = _lib.GPU_TILE
    mg = -(-n // T)
    y0, x0 = sym_job_coord(mg, tile_begin)
    y1, x1 = sym_job_coord(mg, tile_end - 1)
    ya, xa = y0 * T, x0 * T
    y_last = min(n, (y1 + 1) * T) - 1
    x_end = min(n, (x1 + 1) * T)
    return _F(n, ya) + xa - ya, _F(n, y_last) + x_end - y_last


def owned_runs(n: int, tile_begin: int, tile_end: int) -> list[tuple[int, int]]:
    """Maximal contiguous packed-index runs owned by GPU tiles ``[tile_begin, tile_end)``.

    Whole tile-row bands own whole packed rows (one run); the partial bands
    at the two ends of the range contribute one run per job row.
    """
    if tile_end <= tile_begin:
        return []
    T = _lib.GPU_TILE
    mg = -(-n // T)
    Y0, X0 = sym_job_coord(mg, tile_begin)
    Y1, X1 = sym_job_coord(mg, tile_end - 1)
    runs: list[tuple[int, int]] = []

    def add(lo: int, hi: int) -> None:
        if hi <= lo:
            return
        if runs and runs[-1][1] == lo:
            runs[-1] = (runs[-1][0], hi)
        else:
            runs.append((lo, hi))

    for Y in range(Y0, Y1 + 1):
        xa = X0 if Y == Y0 else Y
        xb = X1 if Y == Y1 else mg - 1
        full = xa == Y and xb == mg - 1
        y_lo, y_hi = Y * T, min(n, (Y + 1) * T)
        if full:
            add(_F(n, y_lo), _F(n, y_hi))
            continue
        for y in range(y_lo, y_hi):
            c_lo = max(y, xa * T)
            c_hi = min(n, (xb + 1) * T)
            add(_F(n, y) + c_lo - y, _F(n, y) + c_hi - y)
    return runs


@dataclass
class Shard:
    """One worker's contiguous GPU tile range and its device-resident packed span."""

    worker_index: int
    device: torch.device
    tile_begin: int
    tile_end: int
    base: int                      # packed index of values[0]
    values: torch.Tensor | None    # device float64[span], cells of other shards unspecified
    zero_variance: frozenset[int] = field(default_factory=frozenset)

    def runs(self, n: int) -> list[tuple[int, int]]:
        return owned_runs(n, self.tile_begin, self.tile_end)


@dataclass
class ShardedResult:
    """Per-device packed shards of one all-pairs result (kept on device)."""

    n: int
    shards: list[Shard]
    zero_variance: frozenset[int] = field(default_factory=frozenset)

    def gather(self, out: np.ndarray | torch.Tensor | None = None) -> CorrelationResult:
        """Copy every shard's owned cells into one packed host array."""
        total = sym_job_count(self.n)
        if out is None:
            host = torch.from_numpy(np.empty(total, dtype=np.float64))
        else:
            host = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
            if host.numel() < total:
                raise ValueError(f"out holds {host.numel()} values, need {total}")
        for sh in self.shards:
            if sh.values is None:
                continue
            with torch.cuda.device(sh.device):
                for lo, hi in sh.runs(self.n):
                    host[lo:hi].copy_(sh.values[lo - sh.base : hi - sh.base], non_blocking=host.is_pinned())
                torch.cuda.current_stream().synchronize()
        packed = out if out is not None else host.numpy()
        return CorrelationResult(n=self.n, packed=packed, zero_variance=self.zero_variance)


def check_coverage(spans: list[tuple[int, int, int]], total: int) -> None:
    """Each span is (start, delivered_up_to, stop); demand an exact cover (distributed.py:321-335)."""
    covered = 0
    expected = 0
    for start, delivered, stop in spans:
        if start != expected:
            raise IntegrityError(f"tile ranges not contiguous: expected start {expected}, got {start}")
        if delivered != stop:
            raise IntegrityError(f"tiles [{delivered}, {stop}) never delivered")
        covered += stop - start
        expected = stop
    if covered != total:
        raise IntegrityError(f"covered {covered} tiles of {total}")


def merge(reports: list[WorkerReport], geom: TileGeometry, zero_variance: frozenset[int] = frozenset()) -> CorrelationResult:
    """Assemble retained worker blocks, demanding every tile exactly once (distributed.py:338-373)."""
    from .tiles import empty_result, scatter

    for r in reports:
        if r.status != "ok":
            raise WorkerError(f"cannot merge: worker {r.worker_index} status {r.status!r}: {r.message}",
                              worker_index=r.worker_index)
    total = geom.total_tiles
    seen = np.zeros(total, dtype=np.int64)
    for r in reports:
        for b in r.blocks:
            if not 0 <= b.tile_id < total:
                raise IntegrityError(f"tile id {b.tile_id} out of range [0, {total})")
            seen[b.tile_id] += 1
    dup = np.flatnonzero(seen > 1)
    if dup.size:
        raise IntegrityError(f"duplicated tiles: {dup.tolist()[:20]}")
    missing = np.flatnonzero(seen == 0)
    if missing.size:
        raise IntegrityError(f"missing tiles: {missing.tolist()[:20]}")
    result = empty_result(geom.n, zero_variance)
    for r in reports:
        scatter(r.blocks, geom, result)
    return result


def _run_subprocess(dataset: Dataset, dataset_path: str, geom: TileGeometry, p: int, capacity: int,
                    threads: int, devs: list[torch.device], method: str = "tensor") -> CorrelationResult:
    """One GPU worker process per assignment, the reference's wire protocol
    (distributed.py:209-318): BLOCKS frames are scattered into one packed
    result as they arrive; a failing worker raises ``WorkerError`` with its
    undelivered range."""
    from . import protocol
    from .tiles import _scatter_host, empty_result

    assignments = make_assignments(geom, p, capacity)
    with torch.cuda.device(devs[0]):
        _, flags = normalize_device(as_device_f64(dataset.values, devs[0]))
        zv = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
    result = empty_result(geom.n, zv)
    lock = threading.Lock()
    cursors = [a.start for a in assignments]
    errors: list[WorkerError | None] = [None] * len(assignments)
    root = str(Path(__file__).resolve().parent.parent)

    def reader(a: WorkerAssignment, proc: subprocess.Popen) -> None:
        i = a.worker_index
        try:
            done = False
            while True:
                frame = protocol.read_frame(proc.stdout)
                if frame is None:
                    if not done:
                        raise protocol.ProtocolError("worker exited before DONE")
                    break
                kind, payload = frame
                if kind == protocol.FRAME_BLOCKS:
                    first, count, values = protocol.decode_blocks(payload, geom.t)
                    if first != cursors[i]:
                        raise IntegrityError(f"worker {i} sent tiles from {first}, expected {cursors[i]}")
                    if first + count > a.stop:
                        raise IntegrityError(f"worker {i} overran its range: [{first}, {first + count})")
                    with lock:
                        _scatter_host(result.packed, values, first, count, geom)
                    cursors[i] = first + count
                elif kind == protocol.FRAME_DONE:
                    n_done = protocol.decode_done(payload)
                    if n_done != a.tile_count or cursors[i] != a.stop:
                        raise IntegrityError(f"worker {i} reported {n_done} tiles done but delivered up to "
                                             f"{cursors[i]} of [{a.start}, {a.stop})")
                    done = True
                elif kind == protocol.FRAME_ERROR:
                    raise WorkerError(f"worker {i} reported: {protocol.decode_error(payload)}", worker_index=i,
                                      unfinished_range=(cursors[i], a.stop))
                else:
                    raise protocol.ProtocolError(f"unexpected frame type 0x{kind:02x} from worker {i}")
        except WorkerError as err:
            errors[i] = err
        except Exception as exc:  # noqa: BLE001
            errors[i] = WorkerError(f"worker {i} failed with tiles [{cursors[i]}, {a.stop}) unassembled: {exc}",
                                    worker_index=i, unfinished_range=(cursors[i], a.stop))

    procs, readers = [], []
    try:
        for a in assignments:
            env = dict(os.environ, PAIRCORR_THREADS=str(threads),
                       PCC_DEVICE=str(devs[a.worker_index % len(devs)].index), PCC_METHOD=method,
                       PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
            procs.append(subprocess.Popen([sys.executable, "-m", "paper_1605_01584_b200.worker"],
                                          stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                                          stderr=subprocess.DEVNULL, env=env))
        for a, proc in zip(assignments, procs):
            try:
                protocol.write_frame(proc.stdin, protocol.FRAME_ASSIGN,
                                     protocol.encode_assign(a.start, a.stop, geom.t, a.capacity, dataset_path))
                proc.stdin.close()
            except OSError:
                pass  # the reader reports the early exit
            t = threading.Thread(target=reader, args=(a, proc), daemon=True)
            t.start()
            readers.append(t)
        for t in readers:
            t.join()
        for proc in procs:
            proc.wait()
    finally:
        for proc in procs:
            if proc.poll() is None:
                proc.kill()
                proc.wait()
    for err in errors:
        if err is not None:
            raise err
    check_coverage([(a.start, cursors[a.worker_index], a.stop) for a in assignments], geom.total_tiles)
    return result


def compute_shard(x_host, n: int, l: int, a: WorkerAssignment, device: torch.device,
                  x_device: torch.Tensor | None = None, method: str = "tensor",
                  normalized: tuple | None = None) -> tuple[Shard, torch.Tensor]:
    """Worker body: contract ``a``'s tile range on ``device``.

    ``normalized`` = ``(u, flags)`` already on the device (``normalize_on_devices``),
    or ``(u, flags, contraction)`` to share one prepared ``_lib.Contraction``
    between the workers of a device; else X is uploaded and normalised here.
    Returns the shard and the device zero-variance flags; asynchronous on
    the device's current stream.
    """
    with torch.cuda.device(device):
        if normalized is None:
            x = x_device if x_device is not None else as_device_f64(x_host, device)
            u, flags = normalize_device(x)
            con = None
        else:
            u, flags = normalized[0], normalized[1]
            con = normalized[2] if len(normalized) > 2 else None
        lo, hi = shard_span(n, a.start, a.stop)
        vals = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=device)
        if a.stop > a.start:
            if con is None:
                con = _lib.Contraction(method, u, n, l).prepare_all(stream_handle())
            con.syrk(a.start, a.stop, _lib.LAYOUT_PACKED, ptr(vals), 0, lo, 0, 0, 0, stream_handle(),
                     f"worker {a.worker_index}")
        return Shard(a.worker_index, device, a.start, a.stop, lo, vals), flags


def _rows_of(x_host, r0: int, r1: int) -> torch.Tensor:
    """Rows [r0, r1) of the host / device matrix as a float64 torch tensor view."""
    if isinstance(x_host, torch.Tensor):
        t = x_host if x_host.dtype == torch.float64 else x_host.to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x_host, dtype=np.float64))
    return t[r0:r1]


def normalize_on_devices(x_host, n: int, l: int, devs: list[torch.device]) -> list[tuple[torch.Tensor, torch.Tensor]]:
    """K1 for in-process workers: one ``(u, flags)`` per entry of ``devs``.

    One entry: upload X, normalise (``normalize_device``).  Several: entry q
    uploads only its ``row_slices`` block of X (1/p of it over its own PCIe
    link) and ONE broadcast K1 kernel (``pcc_normalize_rows_bcast_f64``)
    stores each normalised row into every entry's U -- peer stores over
    NVLink between distinct GPUs (``pcc_enable_peer_access``), local stores
    when entries share a device.  U has ``p S`` rows (pad rows zero), flags
    ``p S`` entries.  Same bits as ``normalize_device`` on every entry.
    """
    L = _lib.lib()
    p = len(devs)
    if p == 1:
        with torch.cuda.device(devs[0]):
            return [normalize_device(as_device_f64(x_host, devs[0]))]
    if p > 16:  # kMaxNormDests
        out = []
        for d in devs:
            with torch.cuda.device(d):
                out.append(normalize_device(as_device_f64(x_host, d)))
        return out
    slices, S = row_slices(n, p)
    ldu = int(L.pcc_ldu(l))
    bufs = []
    for d in devs:
        with torch.cuda.device(d):
            u = torch.empty((p * S, ldu), dtype=torch.float64, device=d)
            flags = torch.zeros(p * S, dtype=torch.uint8, device=d)
            _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, p * S, stream_handle()), "pad rows")
            bufs.append((u, flags))
    idx = sorted({d.index for d in devs})
    for a in idx:
        for b in idx:
            _lib.check(L.pcc_enable_peer_access(a, b), f"peer access {a} -> {b}")
    for d in idx:  # every buffer allocated and zero-padded before any peer writes
        torch.cuda.synchronize(d)
    errors: list[BaseException | None] = [None] * p

    def run(q: int) -> None:
        d = devs[q]
        r0, r1 = slices[q]
        try:
            if r1 <= r0:
                return
            with torch.cuda.device(d):
                xd = as_device_f64(_rows_of(x_host, r0, r1), d)
                uarr = (ctypes.c_void_p * p)(*[ptr(u) + 8 * r0 * ldu for u, _ in bufs])
                farr = (ctypes.c_void_p * p)(*[ptr(f) + r0 for _, f in bufs])
                _lib.check(L.pcc_normalize_rows_bcast_f64(ptr(xd), xd.stride(0), uarr, farr, p, ldu, l, 0, r1 - r0,
                                                          stream_handle()), f"device slot {q} normalize+broadcast")
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors[q] = exc

    ts = [threading.Thread(target=run, args=(q,)) for q in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for q, exc in enumerate(errors):
        if exc is not None:
            raise WorkerError(f"device slot {q} failed to normalise rows {slices[q]}: {exc}", worker_index=q) from exc
    return bufs


def stream_shard(x_host, n: int, l: int, a: WorkerAssignment, device: torch.device, host_out=None,
                 method: str = "tensor"):
    """Worker body with overlapped upload / contraction / download (stream.run_stream).

    Uploads and normalises only the rows the range touches (>= its first
    tile row); ``host_out`` (span-sized, pinned for async copies) receives
    the shard's packed span.  Returns the shard and the device flags, valid
    for rows ``[row_lo, n)`` (worker 0 covers every row).
    """
    lo, hi = shard_span(n, a.start, a.stop)
    with torch.cuda.device(device):
        vals = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=device)
        _, flags, _ = run_stream(x_host, n, l, device, a.start, a.stop, vals, lo, host_out, lo, method=method)
    return Shard(a.worker_index, device, a.start, a.stop, lo, vals), flags


def row_slices(n: int, p: int) -> tuple[list[tuple[int, int]], int]:
    """Rows ``[lo, hi)`` each of ``p`` ranks uploads and normalises in exchange
    mode, and the padded block size ``S`` of the all-gather.

    Blocks are whole 128-row GPU tile bands, ``S = ceil(m_g / p) * 128`` rows
    each, so rank r owns rows ``[r S, (r+1) S)`` of a ``p S``-row U (clipped to
    ``n``; trailing ranks may own only pad rows).
    """
    if p < 1:
        raise ValueError(f"rank count must be >= 1, got {p}")
    T = _lib.GPU_TILE
    mg = -(-n // T)
    S = -(-mg // p) * T
    return [(min(n, r * S), min(n, (r + 1) * S)) for r in range(p)], S


def exchange_rows(u: torch.Tensor, flags: torch.Tensor, S: int, rank: int, world: int, group=None) -> None:
    """All-gather every rank's ``S``-row block of ``u`` (rows ``[rank S, (rank+1) S)``)
    and of the zero-variance ``flags`` into all ranks, in place.

    NCCL (one GPU per rank): ``all_gather_into_tensor`` straight between the
    devices over NVLink.  Any other backend (gloo: CPU tests, or functional
    runs with several ranks sharing one GPU) stages through host memory.
    """
    import torch.distributed as dist

    if world == 1:
        return
    backend = dist.get_backend(group)
    blk = slice(rank * S, (rank + 1) * S)
    if backend == "nccl":
        dist.all_gather_into_tensor(u, u[blk].clone(), group=group)
        dist.all_gather_into_tensor(flags, flags[blk].clone(), group=group)
        return
    for t in (u, flags):
        host = t.cpu() if t.is_cuda else t
        dist.all_gather_into_tensor(host, host[blk].clone(), group=group)
        if t.is_cuda:
            t.copy_(host)


EXCHANGES = ("p2p", "collective")


# Exchange buffers and peer mappings of the last p2p exchange, reused while
# the shape, rank layout and group stay the same (cudaMalloc of U and 2 (p-1)
# cudaIpcOpenMemHandle calls per allpairs call would otherwise cost several
# ms each time).  One entry; ``clear_exchange_cache()`` releases it.
_P2P_CACHE: dict = {}


def clear_exchange_cache() -> None:
    """Release the cached p2p exchange buffers and peer mappings."""
    for entry in _P2P_CACHE.values():
        for pu, pf in entry["peers"].values():
            pu.close()
            pf.close()
    _P2P_CACHE.clear()


def _p2p_buffers(n: int, ldu: int, S: int, rank: int, world: int, device: torch.device, group):
    import torch.distributed as dist

    key = (n, ldu, S, rank, world, device.index, id(group))
    entry = _P2P_CACHE.get(key)
    if entry is not None:
        return entry
    clear_exchange_cache()
    L = _lib.lib()
    s = stream_handle()
    ubuf = _lib.DeviceBuffer(world * S * ldu * 8)
    fbuf = _lib.DeviceBuffer(world * S)
    u = ubuf.tensor((world * S, ldu), "<f8")
    flags = fbuf.tensor((world * S,), "|u1")
    # rows past n are written by nobody: each rank zeroes its own buffer's once
    _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, world * S, s), "pad rows")
    flags[n:].zero_()
    handles = [None] * world
    dist.all_gather_object(handles, (ubuf.ipc_handle(), fbuf.ipc_handle()), group=group)
    peers = {q: (_lib.DeviceBuffer(handle=hu), _lib.DeviceBuffer(handle=hf))
             for q, (hu, hf) in enumerate(handles) if q != rank}
    us = [ubuf.address if q == rank else peers[q][0].address for q in range(world)]
    fs = [fbuf.address if q == rank else peers[q][1].address for q in range(world)]
    entry = {"ubuf": ubuf, "fbuf": fbuf, "u": u, "flags": flags, "peers": peers, "us": us, "fs": fs}
    _P2P_CACHE[key] = entry
    return entry


def _exchange_normalize_p2p(x_host, n: int, l: int, rank: int, world: int, device: torch.device, group):
    """K1 fused with the all-gather of U over peer memory: every rank maps
    every other rank's U (CUDA IPC handles swapped over ``group``, cached
    across calls) and one broadcast K1 kernel (``pcc_normalize_rows_bcast_f64``)
    stores each normalised row of this rank's block into all ``p`` buffers --
    over NVLink when the ranks sit on different GPUs of one node.  Two
    ``group`` barriers bracket the writes (every rank done with the previous
    use of its U before, every rank's rows landed after); no kernel ever
    waits on another rank.  The returned ``u`` is the cached buffer: the
    next exchange of the same shape overwrites it."""
    import torch.distributed as dist

    L = _lib.lib()
    slices, S = row_slices(n, world)
    r0, r1 = slices[rank]
    ldu = int(L.pcc_ldu(l))
    with torch.cuda.device(device):
        s = stream_handle()
        e = _p2p_buffers(n, ldu, S, rank, world, device, group)
        xd = None
        if r1 > r0:
            xh = x_host if isinstance(x_host, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x_host))
            xd = torch.empty((r1 - r0, l), dtype=torch.float64, device=device)
            xd.copy_(xh[r0:r1], non_blocking=xh.is_pinned())
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)  # every rank is done with the previous use of its U; buffers mapped
        if r1 > r0:
            uarr = (ctypes.c_void_p * world)(*[a + 8 * r0 * ldu for a in e["us"]])
            farr = (ctypes.c_void_p * world)(*[a + r0 for a in e["fs"]])
            _lib.check(L.pcc_normalize_rows_bcast_f64(ptr(xd), l, uarr, farr, world, ldu, l, 0, r1 - r0, s),
                       f"rank {rank} normalize+broadcast")
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)  # every rank's rows have landed everywhere
    return e["u"], e["flags"]


def exchange_normalize(x_host, n: int, l: int, rank: int, world: int, device: torch.device, group=None,
                       exchange: str = "collective"):
    """Exchange-mode K1: this rank uploads and normalises only its row block
    (``row_slices``), then the blocks are all-gathered so every rank holds
    all of U -- 1/p of X over each GPU's own PCIe link instead of (almost)
    all of it, and the rest over NVLink.  Returns ``(u, flags)`` with
    ``u`` of ``p S`` rows (pad rows zero) and ``flags`` of ``p S`` entries.
    ``exchange``: ``"collective"`` -- K1, then ``all_gather_into_tensor``
    (NCCL; host-staged over gloo); ``"p2p"`` -- one K1 kernel that stores
    the rows straight into every rank's U over peer memory
    (``_exchange_normalize_p2p``).
    """
    if exchange not in EXCHANGES:
        raise ValueError(f"unknown exchange {exchange!r}, expected one of {EXCHANGES}")
    if exchange == "p2p" and world > 1:
        return _exchange_normalize_p2p(x_host, n, l, rank, world, device, group)
    L = _lib.lib()
    slices, S = row_slices(n, world)
    r0, r1 = slices[rank]
    ldu = int(L.pcc_ldu(l))
    with torch.cuda.device(device):
        s = stream_handle()
        u = torch.empty((world * S, ldu), dtype=torch.float64, device=device)
        flags = torch.zeros(world * S, dtype=torch.uint8, device=device)
        if r1 > r0:
            xh = x_host if isinstance(x_host, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x_host))
            xd = torch.empty((r1 - r0, l), dtype=torch.float64, device=device)
            xd.copy_(xh[r0:r1], non_blocking=xh.is_pinned())
            _lib.check(L.pcc_normalize_rows_f64(ptr(xd), l, ptr(u) + 8 * r0 * ldu, ldu, ptr(flags) + r0, l, 0,
                                                r1 - r0, s), f"rank {rank} normalize")
        pad_lo = max(n, rank * S)
        _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, min(pad_lo, (rank + 1) * S), (rank + 1) * S, s), "pad rows")
        exchange_rows(u, flags, S, rank, world, group)
    return u, flags


def compute_worker(dataset: Dataset, p: int, worker_index: int, device=None, out=None, group=None,
                   exact: bool = False, exchange: str = "collective", method: str | None = None):
    """Run worker ``worker_index`` of a ``p``-way split as a standalone call.

    The one-process-per-GPU form of ``run_workers`` (torchrun ranks): upload,
    normalise, contract this worker's GPU tile range; with ``out`` (host
    float64 buffer of ``shard_span`` size, pinned for async copies) its owned
    packed cells are downloaded to ``out[index - span_lo]``.  Returns the
    device ``Shard``; ``Shard.zero_variance`` holds the constant rows.

    ``group``: a ``torch.distributed`` group of the ``p`` workers (rank =
    ``worker_index``).  With it, X is not uploaded whole by every worker:
    each uploads and normalises its ``row_slices`` block and the blocks are
    all-gathered (``exchange_normalize``) before the contraction.
    ``exact`` / ``method``: the contraction (see ``allpairs``).
    """
    method = _lib.resolve_method(method, exact)
    _lib.check_method_shape(method, dataset.l)
    if not 0 <= worker_index < p:
        raise ValueError(f"worker index {worker_index} outside [0, {p})")
    n, l = dataset.n, dataset.l
    a = make_assignments(gpu_geometry(n), p)[worker_index]
    dev = resolve_devices(None if device is None else [device])[0]
    host = None
    if out is not None:
        host = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        lo_span, hi_span = shard_span(n, a.start, a.stop)
        if host.numel() < hi_span - lo_span:
            raise ValueError(f"out holds {host.numel()} values, shard needs {hi_span - lo_span}")
    if group is not None and p > 1:
        with nvtx("pcc.compute_worker.exchange_normalize"):
            u, flags = exchange_normalize(dataset.values, n, l, worker_index, p, dev, group, exchange=exchange)
        lo, hi = shard_span(n, a.start, a.stop)
        with torch.cuda.device(dev):
            vals = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=dev)
            run_stream(None, n, l, dev, a.start, a.stop, vals, lo, host, lo, resident=(u, flags), method=method)
        shard = Shard(a.worker_index, dev, a.start, a.stop, lo, vals)
        flags = flags[:n]
    else:
        shard, flags = stream_shard(dataset.values, n, l, a, dev, host, method=method)
    shard.zero_variance = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
    return shard


def run_workers(
    dataset: Dataset,
    geom: TileGeometry | None,
    p: int,
    backend: str = "cuda",
    capacity: int | None = None,
    threads: int = 1,
    devices=None,
    gather: bool = True,
    out=None,
    exact: bool = False,
    method: str | None = None,
):
    """Partition the work across ``p`` workers on ``devices`` (distributed.py:117-151).

    ``backend="in_process"`` / ``"cuda"``: worker ``i`` is a host thread
    driving ``devices[i % len(devices)]`` over a contiguous range of GPU
    tiles; ``geom`` (the caller's reference tiling) only fixes ``n``.
    Returns a gathered ``CorrelationResult`` (``gather=True``) or the
    device-resident ``ShardedResult``.  ``backend="subprocess"``: one GPU
    worker process per range of the caller's t x t tiles, speaking the
    reference's framed protocol (``worker.py``), gathered on the host.  A
    failing worker raises ``WorkerError`` with its index and unfinished range.
    ``exact`` / ``method``: the contraction (see ``allpairs``).
    """
    method = _lib.resolve_method(method, exact)
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}, expected one of {BACKENDS}")
    dataset_path = None
    if not isinstance(dataset, Dataset):
        from .fileio import load_dataset

        dataset_path = str(dataset)
        dataset = load_dataset(dataset)
    if geom is not None and dataset.n != geom.n:
        raise ValueError(f"geometry is for n={geom.n} but dataset has n={dataset.n}")
    _lib.check_method_shape(method, dataset.l)
    devs = resolve_devices(devices)
    if backend == "subprocess":
        # the reference's worker-process model: reference t x t tiles over the wire
        from .engine import default_capacity
        from .fileio import save_dataset

        geom = geom if geom is not None else TileGeometry(n=dataset.n)
        capacity = default_capacity(geom.t) if capacity is None else capacity
        if dataset_path is not None:
            return _run_subprocess(dataset, dataset_path, geom, p, capacity, threads, devs, method)
        with tempfile.NamedTemporaryFile(suffix=".lpcc", delete=False) as tmp:
            tmp_path = tmp.name
        try:
            save_dataset(tmp_path, dataset)
            return _run_subprocess(dataset, tmp_path, geom, p, capacity, threads, devs, method)
        finally:
            os.unlink(tmp_path)
    n, l = dataset.n, dataset.l
    assignments = make_assignments(gpu_geometry(n), p)
    shards: list[Shard | None] = [None] * p
    flags: list[torch.Tensor | None] = [None] * p
    errors: list[BaseException | None] = [None] * p
    # one device slot per entry of devs (at most one per worker): K1 once per
    # slot -- row blocks + broadcast over NVLink with several -- then every
    # worker contracts its range against its slot's U
    slots = devs[:p]
    with nvtx("pcc.run_workers.normalize_on_devices"):
        normed = normalize_on_devices(dataset.values, n, l, slots)
    cons: list = [None] * len(slots)

    def run_one(a: WorkerAssignment) -> None:
        q = a.worker_index % len(slots)
        dev = slots[q]
        try:
            u, fl = normed[q]
            shards[a.worker_index], flags[a.worker_index] = compute_shard(
                dataset.values, n, l, a, dev, method=method, normalized=(u, fl, cons[q]))
            with torch.cuda.device(dev):
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001 - re-raised as WorkerError below
            errors[a.worker_index] = exc

    for q, (u, _) in enumerate(normed):  # split method: digit planes once per slot
        with torch.cuda.device(slots[q]):
            cons[q] = _lib.Contraction(method, u, n, l).prepare_all(stream_handle())
    if len(slots) == 1:
        with nvtx("pcc.run_workers.contract"):
            for a in assignments:
                run_one(a)
    else:
        ts = [threading.Thread(target=run_one, args=(a,)) for a in assignments]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    for a in assignments:
        exc = errors[a.worker_index]
        if exc is not None:
            raise WorkerError(
                f"worker {a.worker_index} failed with tiles [{a.start}, {a.stop}) unassembled: {exc}",
                worker_index=a.worker_index,
                unfinished_range=(a.start, a.stop),
            ) from exc
    check_coverage([(a.start, a.stop, a.stop) for a in assignments], gpu_geometry(n).total_tiles)
    zv = frozenset(np.flatnonzero(normed[0][1][:n].cpu().numpy()).tolist())
    result = ShardedResult(n=n, shards=[s for s in shards if s is not None], zero_variance=zv)
    return result.gather(out) if gather else result
