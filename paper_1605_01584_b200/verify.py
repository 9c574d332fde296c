"""Brute-force verification on the GPU: the reference's ``verify``
(fileio.py:314-367) with its oracle ``allpairs_naive`` (transform.py:163-179)
evaluated by csrc/verify.cuh -- the definition of Pearson's r (paper Eq. (1))
per pair, bit-identical to ``_kernels.pcc_naive_pair`` -- so results of any
size can be checked without the CPU oracle's O(n^2 l) host cost
(SURVEY.md §8f rank 4).  It shares no kernel with the engine it verifies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device_f64, ptr, require_cuda, stream_handle
from .errors import VerificationError
from .indexing import sym_job_coord, sym_job_count
from .tiles import CorrelationResult
from .transform import Dataset

__all__ = ["VerifyReport", "verify", "naive_pairs", "naive_zero_variance"]


@dataclass
class VerifyReport:
    """Same fields as the reference's report (fileio.py:314-326)."""

    n: int
    tolerance: float
    max_abs_deviation: float
    worst_pair: tuple[int, int]
    first_bad_pair: tuple[int, int] | None
    zero_variance_match: bool
    pairs_checked: int = 0

    @property
    def ok(self) -> bool:
        return self.first_bad_pair is None and self.zero_variance_match


class _Naive:
    """Device copy of X plus per-row statistics for the naive oracle."""

    def __init__(self, dataset: Dataset, device=None):
        require_cuda()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.l = dataset.n, dataset.l
        with torch.cuda.device(self.device):
            self.x = as_device_f64(dataset.values, self.device)
            self.mean = torch.empty(self.n, dtype=torch.float64, device=self.device)
            self.ssd = torch.empty(self.n, dtype=torch.float64, device=self.device)
            self.const = torch.empty(self.n, dtype=torch.uint8, device=self.device)
            _lib.check(_lib.lib().pcc_row_stats_f64(ptr(self.x), self.x.stride(0), self.n, self.l, ptr(self.mean),
                                                    ptr(self.ssd), ptr(self.const), stream_handle()), "row_stats")

    def pairs(self, id_lo: int, id_hi: int) -> torch.Tensor:
        with torch.cuda.device(self.device):
            out = torch.empty(max(0, id_hi - id_lo), dtype=torch.float64, device=self.device)
            _lib.check(_lib.lib().pcc_naive_pairs_f64(ptr(self.x), self.x.stride(0), self.n, self.l, ptr(self.mean),
                                                      ptr(self.ssd), ptr(self.const), id_lo, id_hi, ptr(out),
                                                      stream_handle()), "naive_pairs")
            return out

    def zero_variance(self) -> frozenset[int]:
        flags = (self.const.bool() | (self.ssd == 0.0)).cpu().numpy()
        return frozenset(np.flatnonzero(flags).tolist())


def naive_pairs(dataset: Dataset, id_lo: int = 0, id_hi: int | None = None, device=None) -> torch.Tensor:
    """``pcc_naive_pair`` for packed job ids ``[id_lo, id_hi)`` (device tensor)."""
    nv = _Naive(dataset, device)
    total = sym_job_count(nv.n)
    id_hi = total if id_hi is None else id_hi
    if not 0 <= id_lo <= id_hi <= total:
        raise ValueError(f"job id range [{id_lo}, {id_hi}) outside [0, {total})")
    return nv.pairs(id_lo, id_hi)


def naive_zero_variance(dataset: Dataset, device=None) -> frozenset[int]:
    """``constant_row_flags`` as a set (_kernels.py:278-288)."""
    return _Naive(dataset, device).zero_variance()


def verify(dataset: Dataset, result: CorrelationResult, tolerance: float = 1e-10, raise_on_failure: bool = True,
           rows=None, device=None, chunk: int = 1 << 26) -> VerifyReport:
    """Compare ``result`` against the definition-based oracle, on the GPU.

    ``rows=None`` checks every pair (as the reference does); a list of rows
    checks those rows' packed segments (all pairs (y, x >= y)).  Raises
    ``VerificationError`` (report attached) like the reference.
    """
    if result.n != dataset.n:
        raise ValueError(f"result is for n={result.n}, dataset has n={dataset.n}")
    nv = _Naive(dataset, device)
    n = nv.n
    if rows is None:
        spans = [(lo, min(lo + chunk, sym_job_count(n))) for lo in range(0, sym_job_count(n), chunk)]
    else:
        spans = []
        for y in sorted({int(r) for r in rows}):
            if not 0 <= y < n:
                raise ValueError(f"row {y} outside [0, {n})")
            lo = (y * (2 * n + 1 - y)) // 2
            spans.extend((a, min(a + chunk, lo + n - y)) for a in range(lo, lo + n - y, chunk))
    packed = result.packed
    worst_dev, worst_id, first_bad, checked = 0.0, 0, None, 0
    with torch.cuda.device(nv.device):
        for lo, hi in spans:
            ref = nv.pairs(lo, hi)
            if isinstance(packed, torch.Tensor):
                got = packed[lo:hi].to(nv.device, torch.float64)
            else:
                got = torch.from_numpy(np.ascontiguousarray(packed[lo:hi], dtype=np.float64)).to(nv.device)
            dev = (got - ref).abs()
            dev = torch.where(torch.isnan(dev), torch.full_like(dev, float("inf")), dev)
            m, i = torch.max(dev, 0)
            m = float(m)
            if m > worst_dev or checked == 0:
                if m >= worst_dev:
                    worst_dev, worst_id = m, lo + int(i)
            if first_bad is None and m > tolerance:
                first_bad = lo + int(torch.nonzero(dev > tolerance)[0, 0])
            checked += hi - lo
    wy, wx = sym_job_coord(n, worst_id) if checked else (0, 0)
    fb = tuple(sym_job_coord(n, first_bad)) if first_bad is not None else None
    report = VerifyReport(n=n, tolerance=tolerance, max_abs_deviation=worst_dev, worst_pair=(wy, wx),
                          first_bad_pair=fb, zero_variance_match=result.zero_variance == nv.zero_variance(),
                          pairs_checked=checked)
    if raise_on_failure and not report.ok:
        if report.first_bad_pair is not None:
            raise VerificationError(
                f"pair {report.first_bad_pair} deviates by more than {tolerance} "
                f"(max deviation {report.max_abs_deviation:.3e} at {report.worst_pair})", report=report)
        raise VerificationError("zero-variance row sets disagree between engine and oracle", report=report)
    return report
