"""Per-variable normalisation on the GPU (stage 1 of the hot path).

Mirrors the reference's ``paircorr.transform`` surface
(/root/reference/pkg/src/paircorr/transform.py:52-193): ``Dataset`` with the
same validation and errors, ``NormalizedDataset``, ``normalize`` and
``estimate_cost``.  The arithmetic is the K1 kernel
(csrc/normalize.cuh), bit-identical to ``_kernels.normalize_rows``
(_kernels.py:226-252): mean and centred sum of squares in the fixed 8-lane
order, exact constant-row test, ``ssd == 0.0`` guard, IEEE division and
square root.

Device layout of U: ``pcc_rows_padded(n) x pcc_ldu(l)`` row-major float64
(rows padded to the 128-row GPU tile, K padded to PCC_K_ALIGN = 32 doubles =
256 bytes so every row starts on a cache-line pair and every TMA box of the
contraction stays in bounds); the pad is zero, which leaves every dot product
unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import as_device_f64, ptr, require_cuda, stream_handle
from .errors import DataError

__all__ = [
    "Dataset",
    "NormalizedDataset",
    "normalize",
    "normalize_device",
    "estimate_cost",
    "pcc_normalized",
    "pcc_naive",
    "allpairs_naive",
]


@dataclass
class Dataset:
    """``n`` variables (rows) of ``l`` samples each (transform.py:52-80).

    ``values`` may be a numpy array (coerced to C-contiguous float64, as the
    reference does) or a torch tensor (kept as is -- a pinned CPU tensor
    stays pinned for asynchronous upload, a CUDA tensor stays resident).
    """

    values: object
    ids: list[str] | None = None

    def __post_init__(self) -> None:
        v = self.values
        if isinstance(v, torch.Tensor):
            if v.dtype != torch.float64:
                v = v.to(torch.float64)
            v = v.contiguous()
            if v.dim() != 2:
                raise DataError(f"dataset must be 2-D (rows=variables), got ndim={v.dim()}")
            shape = tuple(v.shape)
            finite = bool(torch.isfinite(v).all()) if v.numel() else True
            if not finite:
                bad = torch.nonzero(~torch.isfinite(v))[0].tolist()
        else:
            v = np.ascontiguousarray(v, dtype=np.float64)
            if v.ndim != 2:
                raise DataError(f"dataset must be 2-D (rows=variables), got ndim={v.ndim}")
            shape = v.shape
            finite = bool(np.isfinite(v).all())
            if not finite:
                bad = np.argwhere(~np.isfinite(v))[0].tolist()
        if shape[0] < 1:
            raise DataError("dataset needs at least one variable")
        if shape[1] < 2:
            raise DataError(f"need at least 2 samples per variable, got {shape[1]}")
        if not finite:
            raise DataError(f"non-finite value at row {bad[0]}, column {bad[1]}")
        if self.ids is not None and len(self.ids) != shape[0]:
            raise DataError("ids length does not match variable count")
        self.values = v

    @property
    def n(self) -> int:
        return int(self.values.shape[0])

    @property
    def l(self) -> int:
        return int(self.values.shape[1])


@dataclass
class NormalizedDataset:
    """Normalised variables resident on a device, plus the constant rows.

    ``u_device`` is the padded ``rows_padded x ldu`` workspace the
    contraction reads; ``u`` is the reference-shaped ``n x l`` host copy
    (made on first access), ``zero_variance`` the flagged rows.
    """

    u_device: torch.Tensor
    n_rows: int
    n_samples: int
    zero_variance: frozenset[int] = field(default_factory=frozenset)
    zero_flags: torch.Tensor | None = None
    _u_host: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.n_rows

    @property
    def l(self) -> int:
        return self.n_samples

    @property
    def ldu(self) -> int:
        return int(self.u_device.shape[1])

    @property
    def device(self) -> torch.device:
        return self.u_device.device

    @property
    def u(self) -> np.ndarray:
        if self._u_host is None:
            self._u_host = self.u_device[: self.n_rows, : self.n_samples].cpu().numpy()
        return self._u_host


def normalize_device(x: torch.Tensor, stream: torch.cuda.Stream | None = None):
    """K1 on a device-resident ``n x l`` float64 tensor.

    Returns ``(u_padded, flags_u8)`` without synchronising the host.
    """
    n, l = int(x.shape[0]), int(x.shape[1])
    L = _lib.lib()
    rows_pad = int(L.pcc_rows_padded(n))
    ldu = int(L.pcc_ldu(l))
    u = torch.empty((rows_pad, ldu), dtype=torch.float64, device=x.device)
    flags = torch.empty(n, dtype=torch.uint8, device=x.device)
    s = stream_handle(stream)
    with torch.cuda.device(x.device):
        _lib.check(L.pcc_normalize_rows_f64(ptr(x), x.stride(0), ptr(u), ldu, ptr(flags), l, 0, n, s),
                   "normalize")
        _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, rows_pad, s), "normalize pad rows")
    return u, flags


def _flags_to_set(flags: torch.Tensor) -> frozenset[int]:
    return frozenset(np.flatnonzero(flags.cpu().numpy()).tolist())


def normalize(dataset: Dataset, threads: int = 1, device=None) -> NormalizedDataset:
    """Normalise every row of ``dataset`` on ``device`` (transform.py:99-124).

    ``threads`` is accepted for signature compatibility; as in the reference
    it never changes a bit of the output (rows are independent).
    """
    if not isinstance(dataset, Dataset):
        raise TypeError("normalize expects a Dataset")
    require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    x = as_device_f64(dataset.values, dev)
    u, flags = normalize_device(x)
    return NormalizedDataset(u_device=u, n_rows=dataset.n, n_samples=dataset.l,
                             zero_variance=_flags_to_set(flags), zero_flags=flags)


def estimate_cost(n: int, l: int) -> int:
    """Unit operations of the transformed computation (transform.py:182-193):
    ``5 l n`` for the row transforms plus ``l`` per each of the ``n(n+1)/2`` pairs."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if l < 1:
        raise ValueError(f"l must be >= 1, got {l}")
    return 5 * l * n + l * n * (n + 1) // 2


# ---------------------------------------------------------------------------
# The reference's per-pair helpers (transform.py:127-179), on the GPU.

def _as_row(v) -> np.ndarray:
    row = np.ascontiguousarray(v.cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
    if row.ndim != 1:
        raise ValueError("expected a 1-D vector")
    return row


class _Rows:
    """Unvalidated ``n x l`` rows for the naive kernels (the reference's
    per-pair helpers take raw vectors, not a ``Dataset``)."""

    def __init__(self, values: np.ndarray):
        self.values = values
        self.n, self.l = int(values.shape[0]), int(values.shape[1])


def pcc_normalized(u_i, u_j) -> float:
    """Correlation of two already-normalised rows (transform.py:134-144): their
    fixed-order ``dot8``, computed by the engine's bit-exact contraction
    (``pcc_syrk_exact_f64`` on a two-row U) -- bit-identical to the
    reference.  A zero-variance (all-zero) row gives 0.0."""
    a, b = _as_row(u_i), _as_row(u_j)
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"length mismatch: {a.shape[0]} vs {b.shape[0]}")
    require_cuda()
    L = _lib.lib()
    l = int(a.shape[0])
    if l == 0:
        return 0.0
    dev = torch.device("cuda", torch.cuda.current_device())
    ldu = int(L.pcc_ldu(l))
    u = torch.zeros((int(L.pcc_rows_padded(2)), ldu), dtype=torch.float64, device=dev)
    u[0, :l] = torch.from_numpy(a).to(dev)
    u[1, :l] = torch.from_numpy(b).to(dev)
    out = torch.empty(3, dtype=torch.float64, device=dev)
    _lib.check(L.pcc_syrk_exact_f64(ptr(u), 2, l, ldu, 0, 1, _lib.LAYOUT_PACKED, ptr(out), 0, 0, 0, 0, 0,
                                    stream_handle()), "pcc_normalized")
    return float(out[1].item())


def pcc_naive(u, v) -> float:
    """Pearson correlation straight from the definition (transform.py:147-160),
    evaluated by the GPU oracle kernel (csrc/verify.cuh) -- bit-identical to
    the reference's ``pcc_naive_pair``; 0.0 if either vector is constant."""
    from .verify import _Naive

    a, b = _as_row(u), _as_row(v)
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"length mismatch: {a.shape[0]} vs {b.shape[0]}")
    if a.shape[0] < 2:
        raise ValueError("need at least 2 samples")
    return float(_Naive(_Rows(np.stack([a, b]))).pairs(1, 2)[0].item())


def allpairs_naive(dataset: Dataset):
    """Brute-force oracle (transform.py:163-179): every upper-triangle pair from
    the definition, on the GPU (bit-identical to the reference's
    ``naive_allpairs_packed``); ``zero_variance`` = ``constant_row_flags``
    (_kernels.py:276-286: exactly constant, or ssd == 0.0), as in the reference."""
    from .indexing import sym_job_count
    from .tiles import CorrelationResult
    from .verify import _Naive

    if not isinstance(dataset, Dataset):
        raise TypeError("allpairs_naive expects a Dataset")
    nv = _Naive(dataset)
    packed = nv.pairs(0, sym_job_count(nv.n)).cpu().numpy()
    return CorrelationResult(n=nv.n, packed=packed, zero_variance=nv.zero_variance())
