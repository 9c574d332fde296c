"""Tiles, results and the compute_pass / scatter seam of the reference.

Mirrors ``paircorr.tiles`` (/root/reference/pkg/src/paircorr/tiles.py:44-242):
``TileGeometry``, ``TileBlock``, ``BlockList``, ``CorrelationResult``,
``empty_result``, ``tile_coord``, ``compute_pass``, ``scatter`` and
``scatter_pass`` keep the reference's names, argument meaning, layouts and
errors, so ``run_pipeline`` / ``ResultSink`` consumers work unchanged.

Two tile sizes coexist:
* the reference's ``t x t`` tiles (default t=4, ``TileGeometry``) define the
  pass-buffer layout of ``compute_pass`` -- tile J at ``(J - j_start) t^2``,
  row-major inside, zeros below the diagonal and past ``n``;
* the engine schedules 128 x 128 GPU tiles (``PCC_GPU_TILE``) numbered by
  the same bijection; the fused epilogue writes either the packed triangle
  directly (``allpairs``) or the reference's t x t pass layout
  (``compute_pass``, via ``pcc_compute_pass_f64``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import ptr, stream_handle
from .errors import IntegrityError
from .indexing import Coord, sym_job_coord, sym_job_coords, sym_job_count, sym_job_id
from .transform import NormalizedDataset

__all__ = [
    "DEFAULT_TILE_SIZE",
    "TileGeometry",
    "TileBlock",
    "BlockList",
    "CorrelationResult",
    "empty_result",
    "tile_coord",
    "compute_pass",
    "compute_pass_device",
    "scatter",
    "scatter_pass",
    "gpu_tile_rows_span",
]

DEFAULT_TILE_SIZE = 4  # tiles.py:44


@dataclass(frozen=True)
class TileGeometry:
    """``t x t`` tiling of the ``n x n`` job matrix (tiles.py:47-71)."""

    n: int
    t: int = DEFAULT_TILE_SIZE

    def __post_init__(self) -> None:
        if self.n < 1:
            raise ValueError(f"n must be >= 1, got {self.n}")
        if self.t < 1:
            raise ValueError(f"tile size must be >= 1, got {self.t}")

    @property
    def m(self) -> int:
        return -(-self.n // self.t)

    @property
    def total_tiles(self) -> int:
        return sym_job_count(self.m)

    @property
    def job_count(self) -> int:
        return sym_job_count(self.n)


@dataclass
class TileBlock:
    """One tile's ``t*t`` values; may view a shared pass buffer (tiles.py:74-79)."""

    tile_id: int
    values: np.ndarray


class BlockList(list):
    """Blocks of one pass in tile order; ``flat`` views the whole pass buffer (tiles.py:82-90)."""

    flat: np.ndarray | None = None


@dataclass
class CorrelationResult:
    """Upper triangle packed in job-id order (tiles.py:93-116).

    ``packed`` is a host ``np.ndarray`` (the reference's type) or, with
    ``allpairs(..., keep_on_device=True)``, a CUDA ``torch.Tensor``.
    """

    n: int
    packed: object
    zero_variance: frozenset[int] = field(default_factory=frozenset)

    def get(self, i: int, j: int) -> float:
        if not (0 <= i < self.n and 0 <= j < self.n):
            raise ValueError(f"pair ({i}, {j}) outside [0, {self.n})")
        return float(self.packed[sym_job_id(self.n, min(i, j), max(i, j))])

    def host_packed(self) -> np.ndarray:
        p = self.packed
        return p.cpu().numpy() if isinstance(p, torch.Tensor) else p

    def to_dense(self) -> np.ndarray:
        """Full symmetric ``n x n`` matrix (tiles.py:107-116)."""
        packed = self.host_packed()
        full = np.empty((self.n, self.n), dtype=np.float64)
        k = 0
        for y in range(self.n):
            row = packed[k : k + self.n - y]
            full[y, y:] = row
            full[y:, y] = row
            k += self.n - y
        return full


def empty_result(n: int, zero_variance: frozenset[int] = frozenset()) -> CorrelationResult:
    """Zero-filled host packed result (tiles.py:119-125)."""
    return CorrelationResult(n=n, packed=np.zeros(sym_job_count(n), dtype=np.float64),
                             zero_variance=zero_variance)


def tile_coord(m: int, tile_id: int) -> Coord:
    """Tile-matrix coordinate of ``tile_id`` (tiles.py:128-130)."""
    return sym_job_coord(m, tile_id)


def gpu_tile_rows_span(n: int, tile_begin: int, tile_end: int) -> tuple[int, int]:
    """Job rows ``[y_lo, y_hi)`` touched by GPU tiles ``[tile_begin, tile_end)``."""
    if tile_end <= tile_begin:
        return (0, 0)
    mg = -(-n // _lib.GPU_TILE)
    ya = sym_job_coord(mg, tile_begin).y
    yb = sym_job_coord(mg, tile_end - 1).y
    return ya * _lib.GPU_TILE, min(n, (yb + 1) * _lib.GPU_TILE)


def _check_range(geom: TileGeometry, j_start: int, j_end: int) -> None:
    if not 0 <= j_start <= j_end <= geom.total_tiles:
        raise ValueError(f"tile range [{j_start}, {j_end}) invalid for {geom.total_tiles} tiles")


def compute_pass_device(u: NormalizedDataset, geom: TileGeometry, j_start: int, j_end: int,
                        out: torch.Tensor, stream: torch.cuda.Stream | None = None, exact: bool = False,
                        method: str | None = None, contraction: "_lib.Contraction | None" = None) -> None:
    """Fill the device buffer ``out`` with the pass layout of tiles ``[j_start, j_end)``
    (``exact``: bit-identical to the reference's ``compute_tile_range``;
    ``method``: see ``allpairs``; ``contraction``: a prepared
    ``_lib.Contraction`` over ``u`` to reuse across passes)."""
    _check_range(geom, j_start, j_end)
    if geom.n != u.n:
        raise ValueError(f"geometry is for n={geom.n} but data has n={u.n}")
    need = (j_end - j_start) * geom.t * geom.t
    if out.numel() < need:
        raise ValueError(f"pass buffer too small: {out.numel()} < {need}")
    if need == 0:
        return
    with torch.cuda.device(u.device):
        s = stream_handle(stream)
        con = contraction
        if con is None:
            con = _lib.Contraction(_lib.resolve_method(method, exact), u.u_device, u.n, u.l).prepare_all(s)
        con.compute_pass(geom.t, j_start, j_end, ptr(out), s)


def compute_pass(
    u: NormalizedDataset,
    geom: TileGeometry,
    j_start: int,
    j_end: int,
    threads: int = 1,
    out=None,
    pool=None,
    *,
    exact: bool = False,
    method: str | None = None,
) -> BlockList:
    """Compute tiles ``[j_start, j_end)`` on the GPU into a flat pass buffer (tiles.py:133-199).

    ``out`` (host float64 array of at least ``(j_end - j_start) t^2``
    values) is filled in place, else a fresh one is returned; ``threads`` and
    ``pool`` are accepted for compatibility and change nothing.  Returns the
    reference's ``BlockList`` of per-tile views with ``flat`` set.
    ``exact``: the bit-exact dot8 contraction (the reference's pass buffer,
    bit for bit); ``method``: the contraction (see ``allpairs``).
    """
    _check_range(geom, j_start, j_end)
    count = j_end - j_start
    t2 = geom.t * geom.t
    need = count * t2
    if out is None:
        out = np.empty(need, dtype=np.float64)
    elif out.shape[0] < need:
        raise ValueError(f"pass buffer too small: {out.shape[0]} < {need}")
    if count == 0:
        return BlockList()
    dev = torch.empty(need, dtype=torch.float64, device=u.device)
    compute_pass_device(u, geom, j_start, j_end, dev, exact=exact, method=method)
    if isinstance(out, torch.Tensor):
        out[:need].copy_(dev)
        host = out
    else:
        torch.from_numpy(out[:need]).copy_(dev)
        host = out
    blocks = BlockList(TileBlock(tile_id=j_start + k, values=host[k * t2 : (k + 1) * t2]) for k in range(count))
    blocks.flat = host[:need]
    return blocks


def _scatter_host(packed: np.ndarray, flat: np.ndarray, first_tile: int, count: int, geom: TileGeometry) -> None:
    # Coordinate-driven (never value-driven) copy of cells y <= x < n of
    # `count` consecutive tiles (_kernels.py:322-348), vectorised indexing.
    t, n, m = geom.t, geom.n, geom.m
    ids = np.arange(first_tile, first_tile + count, dtype=np.uint64)
    yt, xt = sym_job_coords(m, ids)
    r = np.arange(t, dtype=np.int64)
    y = (yt.astype(np.int64)[:, None, None] * t + r[None, :, None])
    x = (xt.astype(np.int64)[:, None, None] * t + r[None, None, :])
    y, x = np.broadcast_arrays(y, x)
    keep = (y <= x) & (x < n)
    yk, xk = y[keep], x[keep]
    idx = (yk * (2 * n + 1 - yk)) // 2 + xk - yk
    packed[idx] = flat[: count * t * t].reshape(count, t, t)[keep]


def scatter(blocks, geom: TileGeometry, result: CorrelationResult) -> CorrelationResult:
    """Write tile blocks into ``result``, coordinate-driven (tiles.py:202-229)."""
    seen: set[int] = set()
    checked = []
    for block in blocks:
        if block.tile_id in seen:
            raise IntegrityError(f"tile {block.tile_id} scattered twice in one call")
        if not 0 <= block.tile_id < geom.total_tiles:
            raise ValueError(f"tile id {block.tile_id} outside [0, {geom.total_tiles})")
        seen.add(block.tile_id)
        values = np.ascontiguousarray(block.values, dtype=np.float64)
        if values.shape != (geom.t * geom.t,):
            raise ValueError(
                f"tile {block.tile_id} carries {values.shape} values, expected ({geom.t * geom.t},)"
            )
        checked.append((block.tile_id, values))
    for tile_id, values in checked:
        _scatter_into(result, values, tile_id, 1, geom)
    return result


def _scatter_into(result: CorrelationResult, flat, first_tile: int, count: int, geom: TileGeometry) -> None:
    packed = result.packed
    if isinstance(packed, torch.Tensor):
        vals = flat if isinstance(flat, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(flat))
        vals = vals.to(packed.device)
        with torch.cuda.device(packed.device):
            _lib.check(_lib.lib().pcc_scatter_range_f64(ptr(packed), ptr(vals), first_tile, count, geom.t, geom.n,
                                                        stream_handle()), "scatter_range")
    else:
        host = flat.cpu().numpy() if isinstance(flat, torch.Tensor) else flat
        _scatter_host(packed, host, first_tile, count, geom)


def scatter_pass(blocks, geom: TileGeometry, result: CorrelationResult) -> None:
    """Scatter one pass, flat fast path when available (tiles.py:232-242)."""
    flat = getattr(blocks, "flat", None)
    if flat is None or not blocks or flat.shape[0] != len(blocks) * geom.t * geom.t:
        scatter(blocks, geom, result)
        return
    _scatter_into(result, flat, blocks[0].tile_id, len(blocks), geom)
