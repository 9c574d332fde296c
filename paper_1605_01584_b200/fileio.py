"""The reference's binary containers, so ``allpairs(path)`` and result files interoperate.

Formats (little-endian, documented in the reference README "File formats"
and fileio.py:1-20):

* dataset ``LPCC``: ``"LPCC" | version u32 = 1 | n u64 | l u64 | n*l f64``
* packed result ``LPCR``: ``"LPCR" | version u32 = 1 | n u64 | zv_count u64 |
  zv_count sorted u64 | n(n+1)/2 f64`` in job-id order, so a pair lookup is
  one seek at a bijection-computed offset (``query_pair``).

Streaming the result to disk: ``PackedFileWriterSink``
is the reference's ``ResultSink`` that writes each pass's owned cells into
the file (fileio.py:233-274), for ``run_pipeline``; ``allpairs_to_file`` is the
GPU fast path -- the streamed engine downloads finished packed rows straight
into a memory map of the file's payload.  Text ingestion stays out of scope.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import DataError
from .indexing import sym_job_count, sym_job_id
from .pipeline import ResultSink
from .tiles import CorrelationResult, TileGeometry, _scatter_host
from .transform import Dataset

__all__ = ["save_dataset", "load_dataset", "save_result", "load_result", "query_pair", "PackedResultReader",
           "PackedFileWriterSink", "allpairs_to_file", "gen_synthetic"]

_HDR = struct.Struct("<4sIQQ")
_VERSION = 1


def gen_synthetic(n: int, l: int, seed: int = 0) -> Dataset:
    """Deterministic uniform [0, 1) dataset (fileio.py:295-305): element k of
    the row-major array is splitmix64(seed + (k+1) * golden) >> 11 * 2^-53,
    bit-identical to the reference (tests/golden/helpers.json)."""
    from .workloads import gen_uniform_splitmix64

    return Dataset(values=gen_uniform_splitmix64(n, l, seed))


def save_dataset(path, dataset: Dataset) -> None:
    v = dataset.values
    v = v.cpu().numpy() if hasattr(v, "cpu") else v
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"LPCC", _VERSION, dataset.n, dataset.l))
        np.ascontiguousarray(v, dtype="<f8").tofile(f)


def load_dataset(path, format: str = "auto") -> Dataset:
    """Load a dataset (fileio.py:65-78): ``format`` is ``auto`` (magic bytes
    decide), ``binary`` (the LPCC container) or ``tsv`` (whitespace-separated
    text, optional label column)."""
    path = Path(path)
    if format not in ("auto", "binary", "tsv"):
        raise ValueError(f"unknown format {format!r}")
    if format == "auto":
        with open(path, "rb") as f:
            format = "binary" if f.read(4) == b"LPCC" else "tsv"
    if format == "tsv":
        return _load_dataset_tsv(path)
    size = path.stat().st_size
    with open(path, "rb") as f:
        head = f.read(_HDR.size)
        if len(head) < _HDR.size:
            raise DataError(f"{path}: truncated header")
        magic, version, n, l = _HDR.unpack(head)
        if magic != b"LPCC":
            raise DataError(f"{path}: bad magic {magic!r}")
        if version != _VERSION:
            raise DataError(f"{path}: unsupported version {version}")
        if size != _HDR.size + 8 * n * l:
            raise DataError(f"{path}: file is {size} bytes but header declares {_HDR.size + 8 * n * l}")
        values = np.fromfile(f, dtype="<f8", count=n * l)
    return Dataset(values=values.astype(np.float64, copy=False).reshape(n, l))


def _is_number(text: str) -> bool:
    try:
        float(text)
    except ValueError:
        return False
    return True


def _load_dataset_tsv(path: Path) -> Dataset:
    """Text rows of numbers, whitespace separated; a non-numeric first field
    on the first row makes column 1 a label column for every row
    (fileio.py:102-141, same checks and messages)."""
    import math

    rows: list[list[float]] = []
    ids: list[str] = []
    labeled = None
    width = None
    with open(path, "r", encoding="utf-8") as f:
        for lineno, line in enumerate(f, start=1):
            fields = line.split()
            if not fields:
                continue
            if labeled is None:
                labeled = not _is_number(fields[0])
            if labeled:
                if _is_number(fields[0]):
                    raise DataError(f"{path}:{lineno}: expected a label in column 1, got {fields[0]!r}")
                ids.append(fields[0])
                fields = fields[1:]
            row = []
            for col, field in enumerate(fields, start=2 if labeled else 1):
                try:
                    value = float(field)
                except ValueError:
                    raise DataError(f"{path}:{lineno}: column {col}: {field!r} is not a number") from None
                if not math.isfinite(value):
                    raise DataError(f"{path}:{lineno}: column {col}: non-finite value {field!r}")
                row.append(value)
            if width is None:
                width = len(row)
            elif len(row) != width:
                raise DataError(f"{path}:{lineno}: ragged row of {len(row)} samples, expected {width}")
            rows.append(row)
    if not rows:
        raise DataError(f"{path}: empty dataset")
    return Dataset(values=np.array(rows, dtype=np.float64), ids=ids if labeled else None)


def save_result(path, result: CorrelationResult) -> None:
    zv = np.array(sorted(result.zero_variance), dtype="<u8")
    packed = result.host_packed()
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"LPCR", _VERSION, result.n, zv.size))
        f.write(zv.tobytes())
        np.ascontiguousarray(packed, dtype="<f8").tofile(f)


def _result_header(f, path):
    head = f.read(_HDR.size)
    if len(head) < _HDR.size:
        raise DataError(f"{path}: truncated header")
    magic, version, n, zc = _HDR.unpack(head)
    if magic != b"LPCR":
        raise DataError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise DataError(f"{path}: unsupported version {version}")
    return n, zc


def load_result(path) -> CorrelationResult:
    path = Path(path)
    with open(path, "rb") as f:
        n, zc = _result_header(f, path)
        zv = np.fromfile(f, dtype="<u8", count=zc)
        packed = np.fromfile(f, dtype="<f8", count=sym_job_count(n))
    if packed.size != sym_job_count(n):
        raise DataError(f"{path}: truncated packed payload")
    return CorrelationResult(n=n, packed=packed.astype(np.float64, copy=False),
                             zero_variance=frozenset(int(i) for i in zv))


def query_pair(result_path, i: int, j: int) -> float:
    """One seek: offset = header + 8 * (zv_count + job_id(min, max))."""
    path = Path(result_path)
    with open(path, "rb") as f:
        n, zc = _result_header(f, path)
        if not (0 <= i < n and 0 <= j < n):
            raise ValueError(f"pair ({i}, {j}) outside [0, {n})")
        f.seek(_HDR.size + 8 * (zc + sym_job_id(n, min(i, j), max(i, j))))
        return float(np.frombuffer(f.read(8), dtype="<f8")[0])


class PackedResultReader:
    """Seek-based random access to an ``LPCR`` file (fileio.py:175-230)."""

    def __init__(self, path):
        self.path = Path(path)
        self._f = open(self.path, "rb")
        try:
            self.n, zc = _result_header(self._f, self.path)
            zv = np.fromfile(self._f, dtype="<u8", count=zc)
            if zv.size != zc:
                raise DataError(f"{self.path}: truncated zero-variance index list")
            self.zero_variance = frozenset(int(i) for i in zv)
            self._data_offset = _HDR.size + 8 * zc
            expected = self._data_offset + 8 * sym_job_count(self.n)
            if self.path.stat().st_size != expected:
                raise DataError(f"{self.path}: file is {self.path.stat().st_size} bytes but header declares {expected}")
        except Exception:
            self._f.close()
            raise

    def query(self, i: int, j: int) -> float:
        if not (0 <= i < self.n and 0 <= j < self.n):
            raise ValueError(f"pair ({i}, {j}) outside [0, {self.n})")
        self._f.seek(self._data_offset + 8 * sym_job_id(self.n, min(i, j), max(i, j)))
        return float(np.frombuffer(self._f.read(8), dtype="<f8")[0])

    def read_all(self) -> np.ndarray:
        self._f.seek(self._data_offset)
        return np.fromfile(self._f, dtype="<f8", count=sym_job_count(self.n)).astype(np.float64, copy=False)

    def close(self) -> None:
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc_info):
        self.close()


def _create_result_file(path, n: int, zero_variance: frozenset[int]) -> np.memmap:
    zv = np.array(sorted(zero_variance), dtype="<u8")
    offset = _HDR.size + 8 * zv.size
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"LPCR", _VERSION, n, zv.size))
        f.write(zv.tobytes())
        f.truncate(offset + 8 * sym_job_count(n))
    return np.memmap(path, dtype="<f8", mode="r+", offset=offset, shape=(sym_job_count(n),))


class PackedFileWriterSink(ResultSink):
    """``ResultSink`` streaming each pass into an ``LPCR`` file (fileio.py:233-274).

    Header and zero-filled payload are created up front; every consumed pass
    scatters only the cells its tiles own (coordinate-driven), through a
    memory map of the payload.
    """

    def __init__(self, path, geom: TileGeometry, zero_variance: frozenset[int] = frozenset()):
        self.geom = geom
        self._map = _create_result_file(path, geom.n, zero_variance)

    def consume(self, pass_range, blocks) -> None:
        flat = getattr(blocks, "flat", None)
        t2 = self.geom.t * self.geom.t
        if flat is not None and blocks and flat.shape[0] == len(blocks) * t2:
            _scatter_host(self._map, np.asarray(flat), blocks[0].tile_id, len(blocks), self.geom)
            return
        for block in blocks:
            _scatter_host(self._map, np.ascontiguousarray(block.values, dtype=np.float64), block.tile_id, 1, self.geom)

    def close(self) -> None:
        self._map.flush()
        del self._map

    def __enter__(self):
        return self

    def __exit__(self, *exc_info):
        self.close()


def allpairs_to_file(dataset: Dataset, path, device=None, *, exact: bool = False,
                     method: str | None = None) -> frozenset[int]:
    """All-pairs PCC of ``dataset`` written straight to an ``LPCR`` file.

    The zero-variance set (needed for the header, which precedes the
    payload) comes from one normalisation pass; the streamed engine then
    downloads finished packed rows directly into the file's memory map.
    ``exact`` / ``method``: the contraction (see ``allpairs``).  Returns the
    zero-variance set.
    """
    import torch

    from . import _lib
    from ._device import as_device_f64, resolve_devices
    from .stream import run_stream
    from .transform import normalize_device

    method = _lib.resolve_method(method, exact)
    _lib.check_method_shape(method, dataset.l)
    dev = resolve_devices(None if device is None else [device])[0]
    n, l = dataset.n, dataset.l
    with torch.cuda.device(dev):
        x = as_device_f64(dataset.values, dev)
        _, flags = normalize_device(x)
        zv = frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())
        payload = _create_result_file(path, n, zv)
        T = int(_lib.lib().pcc_gpu_tile_count(n))
        packed = torch.empty(sym_job_count(n), dtype=torch.float64, device=dev)
        run_stream(x, n, l, dev, 0, T, packed, 0, torch.from_numpy(payload), 0, method=method)
        payload.flush()
        del payload
    return zv
