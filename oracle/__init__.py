"""CPU oracle for the all-pairs PCC hot path -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/libpcc_oracle.so`` (built from
``oracle/pcc_oracle.c`` by ``oracle/Makefile`` or ``__graft_entry__.build()``),
a bit-exact C restatement of the reference package's numba kernels
(``/root/reference/pkg/src/paircorr/_kernels.py``) and their thread drivers.

Who may import this: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- as the checker
or the reported CPU baseline, never as the thing measured or shipped.  The
product package ``paper_1605_01584_b200`` never imports it.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
bit-for-bit against fixtures generated from the real reference
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libpcc_oracle.so"
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> Path:
    """Compile the oracle shared library in place (gcc, no FMA contraction)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        l = ctypes.CDLL(str(_LIB_PATH))
        l.oracle_dot8.restype = ctypes.c_double
        l.oracle_dot8.argtypes = [_dp, _dp, _i64]
        l.oracle_sum8.restype = ctypes.c_double
        l.oracle_sum8.argtypes = [_dp, _i64]
        l.oracle_ssd8.restype = ctypes.c_double
        l.oracle_ssd8.argtypes = [_dp, _i64, ctypes.c_double]
        l.oracle_covar8.restype = ctypes.c_double
        l.oracle_covar8.argtypes = [_dp, _dp, _i64, ctypes.c_double, ctypes.c_double]
        l.oracle_is_constant.restype = ctypes.c_int
        l.oracle_is_constant.argtypes = [_dp, _i64]
        l.oracle_pcc_naive_pair.restype = ctypes.c_double
        l.oracle_pcc_naive_pair.argtypes = [_dp, _dp, _i64]
        l.oracle_tile_row.restype = _i64
        l.oracle_tile_row.argtypes = [_i64, _i64]
        l.oracle_normalize_rows.argtypes = [_dp, _dp, _u8p, _i64, _i64, _i64]
        l.oracle_normalize.argtypes = [_dp, _i64, _i64, _dp, _u8p, ctypes.c_int]
        l.oracle_compute_pass.argtypes = [_dp, _i64, _i64, _i64, _i64, _i64, _dp, ctypes.c_int]
        l.oracle_compute_tile_range.argtypes = [_dp, _i64, _dp, _i64, _i64, _i64, _i64, _i64, _i64]
        l.oracle_scatter_range.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _i64]
        l.oracle_scatter_range_span.argtypes = [_dp, _i64, _dp, _i64, _i64, _i64, _i64, _i64]
        l.oracle_allpairs_naive.argtypes = [_dp, _i64, _i64, _dp, ctypes.c_int]
        l.oracle_constant_row_flags.argtypes = [_dp, _i64, _i64, _u8p]
        l.oracle_allpairs.restype = ctypes.c_int
        l.oracle_allpairs.argtypes = [_dp, _i64, _i64, _i64, _i64, _dp, _u8p, _dp, _dp, ctypes.c_int]
        _lib = l
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _u8(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# -- per-vector kernels (_kernels.py:30-223) --------------------------------

def dot8(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return lib().oracle_dot8(_d(a), _d(b), a.shape[0])


def sum8(a) -> float:
    a = _f64(a)
    return lib().oracle_sum8(_d(a), a.shape[0])


def ssd8(a, mean: float) -> float:
    a = _f64(a)
    return lib().oracle_ssd8(_d(a), a.shape[0], mean)


def covar8(a, b, mean_a: float, mean_b: float) -> float:
    a, b = _f64(a), _f64(b)
    return lib().oracle_covar8(_d(a), _d(b), a.shape[0], mean_a, mean_b)


def is_constant(a) -> bool:
    a = _f64(a)
    return bool(lib().oracle_is_constant(_d(a), a.shape[0]))


def pcc_naive_pair(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return lib().oracle_pcc_naive_pair(_d(a), _d(b), a.shape[0])


def tile_row(m: int, tile_id: int) -> int:
    return int(lib().oracle_tile_row(m, tile_id))


# -- row / tile drivers (transform.py, tiles.py, engine.py) -----------------

def normalize(x, threads: int | None = None):
    """transform.py:99-124 -> (u, zero_variance bool[n])."""
    x = _f64(x)
    n, l = x.shape
    u = np.empty_like(x)
    flags = np.zeros(n, dtype=np.uint8)
    lib().oracle_normalize(_d(x), n, l, _d(u), _u8(flags), threads or default_threads())
    return u, flags.astype(bool)


def constant_row_flags(x) -> np.ndarray:
    x = _f64(x)
    flags = np.zeros(x.shape[0], dtype=np.uint8)
    lib().oracle_constant_row_flags(_d(x), x.shape[0], x.shape[1], _u8(flags))
    return flags.astype(bool)


def compute_pass(u, t: int, j_start: int, j_end: int, threads: int | None = None) -> np.ndarray:
    """tiles.py:133-199 flat buffer: tile J at (J - j_start) * t * t."""
    u = _f64(u)
    n, l = u.shape
    out = np.empty(max(0, j_end - j_start) * t * t, dtype=np.float64)
    if j_end > j_start:
        lib().oracle_compute_pass(_d(u), n, l, t, j_start, j_end, _d(out), threads or default_threads())
    return out


def scatter_range(packed: np.ndarray, values, first_tile: int, count: int, m: int, t: int, n: int) -> None:
    values = _f64(values)
    lib().oracle_scatter_range(_d(packed), _d(values), first_tile, count, m, t, n)


def packed_rows_span(u, y_lo: int, y_hi: int, t: int = 4, threads: int | None = None) -> np.ndarray:
    """The reference's packed values of rows [y_lo, y_hi) -- the packed span
    [F(y_lo), F(y_hi)) -- computed exactly as its engine does: compute_pass
    over the t x t tile rows covering those rows (tiles.py:133-199) and
    scatter_range of them (_kernels.py:322-348) into the span (sampled
    full-size parity; ``y_lo`` and ``y_hi`` multiples of t, or y_hi = n)."""
    u = _f64(u)
    n = u.shape[0]
    if not (0 <= y_lo < y_hi <= n) or y_lo % t or (y_hi % t and y_hi != n):
        raise ValueError(f"row range [{y_lo}, {y_hi}) must be t-aligned inside [0, {n}]")
    m = -(-n // t)
    tr_lo, tr_hi = y_lo // t, -(-y_hi // t)
    j_lo = tr_lo * (2 * m - tr_lo + 1) // 2
    j_hi = tr_hi * (2 * m - tr_hi + 1) // 2
    flat = compute_pass(u, t, j_lo, j_hi, threads)
    lo = y_lo * (2 * n - y_lo + 1) // 2
    hi = y_hi * (2 * n - y_hi + 1) // 2
    span = np.full(hi - lo, np.nan, dtype=np.float64)
    lib().oracle_scatter_range_span(_d(span), lo, _d(flat), j_lo, j_hi - j_lo, m, t, n)
    return span


def allpairs(x, t: int = 4, capacity: int | None = None, threads: int | None = None,
             buffer_budget: int = 256 * 2**20):
    """engine.py:23-56 (workers=1): -> (packed f64[n(n+1)/2], zero_variance bool[n])."""
    x = _f64(x)
    n, l = x.shape
    if capacity is None:
        capacity = max(1, buffer_budget // (2 * t * t * 8))  # engine.py:17-20
    m = -(-n // t)
    total = m * (m + 1) // 2
    capacity = max(1, min(capacity, total))
    u = np.empty_like(x)
    flags = np.zeros(n, dtype=np.uint8)
    buf = np.empty(capacity * t * t, dtype=np.float64)
    packed = np.empty(n * (n + 1) // 2, dtype=np.float64)
    lib().oracle_allpairs(_d(x), n, l, t, capacity, _d(u), _u8(flags), _d(buf), _d(packed),
                          threads or default_threads())
    return packed, flags.astype(bool)


def allpairs_naive(x, threads: int | None = None):
    """transform.py:163-179 brute-force oracle -> (packed, zero_variance bool[n])."""
    x = _f64(x)
    n, l = x.shape
    packed = np.empty(n * (n + 1) // 2, dtype=np.float64)
    lib().oracle_allpairs_naive(_d(x), n, l, _d(packed), threads or default_threads())
    return packed, constant_row_flags(x)


def packed_rows(u, rows, threads: int | None = None):
    """Reference dot8 values for selected packed rows (sampled parity at scale).

    Returns {y: f64[n - y]} with entry x - y = dot8(u[y], u[x]) -- exactly the
    value the reference's compute_tile_range writes for cell (y, x)
    (_kernels.py:366-373), whatever the tile size.
    """
    u = _f64(u)
    n = u.shape[0]
    out = {}
    for y in rows:
        y = int(y)
        # t = n-wide single tile row: compute_tile_range over tile (0, 0) of a
        # 1-row view is awkward; evaluate dot8 directly per cell instead.
        seg = np.empty(n - y, dtype=np.float64)
        _row_dots(u, y, seg, threads or default_threads())
        out[y] = seg
    return out


def _row_dots(u: np.ndarray, y: int, seg: np.ndarray, threads: int) -> None:
    # One reference tile per cell with t=1: compute_tile_range over the
    # contiguous tile ids of row y in the t=1 tile matrix (m = n).
    n, l = u.shape
    first = y * (2 * n - y + 1) // 2
    lib().oracle_compute_tile_range(_d(u), l, _d(seg), n, 1, n, first, first + (n - y), first)
