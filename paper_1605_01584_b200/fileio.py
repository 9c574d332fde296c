"""The reference's binary containers, so ``allpairs(path)`` and result files interoperate.

Formats (little-endian, documented in the reference README "File formats"
and fileio.py:1-20):

* dataset ``LPCC``: ``"LPCC" | version u32 = 1 | n u64 | l u64 | n*l f64``
* packed result ``LPCR``: ``"LPCR" | version u32 = 1 | n u64 | zv_count u64 |
  zv_count sorted u64 | n(n+1)/2 f64`` in job-id order, so a pair lookup is
  one seek at a bijection-computed offset (``query_pair``).

Only the binary dataset container and the packed result file are provided;
text ingestion, the streaming ``PackedFileWriterSink`` and ``verify`` are
outside this build's hot-path scope.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import DataError
from .indexing import sym_job_count, sym_job_id
from .tiles import CorrelationResult
from .transform import Dataset

__all__ = ["save_dataset", "load_dataset", "save_result", "load_result", "query_pair"]

_HDR = struct.Struct("<4sIQQ")
_VERSION = 1


def save_dataset(path, dataset: Dataset) -> None:
    v = dataset.values
    v = v.cpu().numpy() if hasattr(v, "cpu") else v
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"LPCC", _VERSION, dataset.n, dataset.l))
        np.ascontiguousarray(v, dtype="<f8").tofile(f)


def load_dataset(path, format: str = "auto") -> Dataset:
    """Read an ``LPCC`` dataset (fileio.py:65-99, binary container)."""
    path = Path(path)
    if format not in ("auto", "binary"):
        raise ValueError(f"unsupported format {format!r} (this build reads the binary LPCC container)")
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
