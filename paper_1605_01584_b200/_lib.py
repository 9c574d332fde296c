"""ctypes binding of the C ABI in ``include/pcc_b200.h`` (libpcc_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``) into
``paper_1605_01584_b200/lib/libpcc_b200.so``.  There is no fallback: if the
library is missing or no B200 is visible, every compute entry point raises.
ctypes releases the GIL for the duration of each call, so one host thread per
device drives devices concurrently (SURVEY.md §5 "Distributed communication
backend").
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import DeviceError

__all__ = [
    "LIB_PATH",
    "lib",
    "check",
    "DeviceInfo",
    "GPU_TILE",
    "K_ALIGN",
    "LAYOUT_PACKED",
    "LAYOUT_DENSE",
    "LAYOUT_TILES",
    "EXPORTED_SYMBOLS",
]

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpcc_b200.so"

PCC_OK, PCC_EINVAL, PCC_ECUDA = 0, 1, 2
GPU_TILE = 128
K_ALIGN = 32
LAYOUT_PACKED, LAYOUT_DENSE, LAYOUT_TILES = 0, 1, 2
VARIANT_EXACT = 100  # PCC_VARIANT_EXACT: the bit-exact dot8 contraction

# Every symbol include/pcc_b200.h declares (tests check the .so exports them).
EXPORTED_SYMBOLS = (
    "pcc_last_error",
    "pcc_version",
    "pcc_device_info",
    "pcc_rows_padded",
    "pcc_ldu",
    "pcc_gpu_tile_count",
    "pcc_normalize_rows_f64",
    "pcc_normalize_rows_bcast_f64",
    "pcc_device_alloc",
    "pcc_device_free",
    "pcc_ipc_get_handle",
    "pcc_ipc_open_handle",
    "pcc_ipc_close_handle",
    "pcc_enable_peer_access",
    "pcc_zero_rows_f64",
    "pcc_syrk_f64",
    "pcc_syrk_f64_variant",
    "pcc_syrk_exact_f64",
    "pcc_split_slice_bytes",
    "pcc_split_rows_f64",
    "pcc_normalize_split_rows_f64",
    "pcc_syrk_split_f64",
    "pcc_compute_pass_f64",
    "pcc_compute_pass_exact_f64",
    "pcc_compute_pass_split_f64",
    "pcc_scatter_range_f64",
    "pcc_allpairs_f64",
    "pcc_row_stats_f64",
    "pcc_naive_pairs_f64",
    "pcc_tile_schedule",
    "pcc_syrk_launches",
    "pcc_probe_fp64_peak",
)


class DeviceInfo(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("sm_count", ctypes.c_int),
        ("cc_major", ctypes.c_int),
        ("cc_minor", ctypes.c_int),
        ("max_smem_optin", ctypes.c_int),
        ("syrk_ctas_per_sm", ctypes.c_int),
        ("syrk_smem_bytes", ctypes.c_int),
        ("gpu_tile", ctypes.c_int),
        ("total_mem", ctypes.c_size_t),
    ]


_lock = threading.Lock()
_lib = None

_i32, _i64, _u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_vp = ctypes.c_void_p


def _bind(l: ctypes.CDLL) -> None:
    sig = {
        "pcc_last_error": (ctypes.c_char_p, []),
        "pcc_version": (ctypes.c_int, []),
        "pcc_device_info": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(DeviceInfo)]),
        "pcc_rows_padded": (_i64, [_i64]),
        "pcc_ldu": (_i64, [_i64]),
        "pcc_gpu_tile_count": (_u64, [_i64]),
        "pcc_normalize_rows_f64": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _vp]),
        "pcc_zero_rows_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp]),
        "pcc_normalize_rows_bcast_f64": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i32,
                                                        _i64, _i64, _i64, _i64, _vp]),
        "pcc_device_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_vp)]),
        "pcc_device_free": (ctypes.c_int, [_vp]),
        "pcc_ipc_get_handle": (ctypes.c_int, [_vp, ctypes.c_char_p]),
        "pcc_ipc_open_handle": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
        "pcc_ipc_close_handle": (ctypes.c_int, [_vp]),
        "pcc_enable_peer_access": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
        "pcc_syrk_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _u64, _u64, _i32, _vp, _i64, _u64, _i32, _u64, _u64, _vp]),
        "pcc_syrk_f64_variant": (ctypes.c_int, [_i32, _vp, _i64, _i64, _i64, _u64, _u64, _i32, _vp, _i64, _u64, _i32, _u64, _u64, _vp]),
        "pcc_syrk_exact_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _u64, _u64, _i32, _vp, _i64, _u64, _i32, _u64, _u64, _vp]),
        "pcc_split_slice_bytes": (_u64, [_i64, _i64]),
        "pcc_split_rows_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
        "pcc_normalize_split_rows_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp]),
        "pcc_syrk_split_f64": (ctypes.c_int, [_vp, _vp, _i64, _i64, _u64, _u64, _i32, _vp, _i64, _u64, _i32, _u64, _u64, _vp]),
        "pcc_compute_pass_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i64, _u64, _u64, _vp, _vp]),
        "pcc_compute_pass_exact_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i64, _u64, _u64, _vp, _vp]),
        "pcc_compute_pass_split_f64": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _u64, _u64, _vp, _vp]),
        "pcc_scatter_range_f64": (ctypes.c_int, [_vp, _vp, _u64, _u64, _i64, _i64, _vp]),
        "pcc_allpairs_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _u64, _u64, _i32, _vp, _i64, _u64, _vp]),
        "pcc_row_stats_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
        "pcc_naive_pairs_f64": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _u64, _u64, _vp, _vp]),
        "pcc_tile_schedule": (ctypes.c_int, [_i64, _u64, _u64, ctypes.c_uint32, _vp, _vp]),
        "pcc_syrk_launches": (ctypes.c_int, [_i64, _u64, _u64, ctypes.POINTER(ctypes.c_int32)]),
        "pcc_probe_fp64_peak": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(l, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> ctypes.CDLL:
    """Load (once) and return the engine library; raise DeviceError if absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise DeviceError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)"
                    )
                l = ctypes.CDLL(str(LIB_PATH))
                _bind(l)
                _lib = l
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception conventions."""
    if rc == PCC_OK:
        return
    msg = lib().pcc_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == PCC_EINVAL:
        raise ValueError(msg)
    raise DeviceError(msg)


def device_info(device: int) -> DeviceInfo:
    info = DeviceInfo()
    check(lib().pcc_device_info(device, ctypes.byref(info)), "pcc_device_info")
    return info


def probe_fp64_peak() -> float:
    """Measured DMMA (FP64 tensor pipe) TFLOP/s of the current device."""
    v = ctypes.c_double(0.0)
    check(lib().pcc_probe_fp64_peak(ctypes.byref(v)), "pcc_probe_fp64_peak")
    return v.value


def syrk_launches(n: int, tile_begin: int, tile_end: int) -> int:
    """Kernels ``pcc_syrk_f64`` launches for GPU tiles ``[tile_begin, tile_end)`` on the current device."""
    v = ctypes.c_int32(0)
    check(lib().pcc_syrk_launches(n, tile_begin, tile_end, ctypes.byref(v)), "pcc_syrk_launches")
    return v.value


def syrk_fn(exact: bool = False):
    """The contraction entry point: the tensor-core path (``pcc_syrk_f64``) or
    the bit-exact dot8 path (``pcc_syrk_exact_f64``); same arguments."""
    return lib().pcc_syrk_exact_f64 if exact else lib().pcc_syrk_f64


# Contraction methods (``allpairs(..., method=)``):
#   "tensor" -- FP64 tensor cores (DMMA), within 1e-12 of the reference (default);
#   "split"  -- int8 tensor cores (tcgen05.mma kind::i8) on exact radix-128
#               digit planes of U (the Ozaki scheme), within 1e-12, l <= 8192;
#   "exact"  -- the reference's dot8 arithmetic on the FP64 CUDA cores, bit-identical.
METHODS = ("tensor", "split", "exact")
SPLIT_MAX_L = 8192
SPLIT_ROW_BYTES = 64  # digit-plane layout int8 [ceil(l/64)][7][rows][64] (split.cuh)


def resolve_method(method: str | None = None, exact: bool = False) -> str:
    """``method`` name from the public arguments (``exact=True`` is ``"exact"``)."""
    if exact:
        if method not in (None, "exact"):
            raise ValueError(f"exact=True conflicts with method={method!r}")
        return "exact"
    m = "tensor" if method is None else method
    if m not in METHODS:
        raise ValueError(f"unknown contraction method {m!r}, expected one of {METHODS}")
    return m


def check_method_shape(method: str, l: int) -> None:
    if method == "split" and l > SPLIT_MAX_L:
        raise ValueError(f"method='split' is bounded to l <= {SPLIT_MAX_L} samples (its 1e-12 error bound); "
                         f"got l={l}: use method='tensor'")


def split_products(scale, n: int, l: int, tile_begin: int, tile_end: int) -> int:
    """int8 products (tcgen05.mma of 128 x 128 x 32 per K step) the split
    contraction issues per K step summed over GPU tiles [tile_begin,
    tile_end): 34 per tile, 28 where the tile pair's rows allow dropping the
    sd = 7 diagonal (split.cuh ``split_drop_top``, same arithmetic)."""
    import numpy as np

    s = np.asarray(scale.cpu() if hasattr(scale, "cpu") else scale, dtype=np.float64)
    mg = -(-n // GPU_TILE)
    tmax = s[:mg * GPU_TILE].reshape(mg, GPU_TILE).max(axis=1)
    iy, ix = np.triu_indices(mg)  # row-major upper triangle = the bijection's id order
    iy, ix = iy[tile_begin:tile_end], ix[tile_begin:tile_end]
    sy, sx = tmax[iy], tmax[ix]
    bound = sy * sx * float(l) * (6.04 * 2.0 ** -37) + (sy + sx) * 2.0 ** -43 * np.sqrt(float(l))
    drop = bound <= 5e-13
    return int(34 * drop.size - 6 * int(drop.sum()))


class Contraction:
    """The contraction over one normalised U (``pcc_rows_padded(n) x ldu``
    f64 on a CUDA device, pad rows zero) by ``method`` (``METHODS``).

    ``prepare(row_lo, row_hi, stream)`` must follow the normalisation of those
    rows and precede any contraction that reads them: the split method
    writes their int8 digit planes and scales (``pcc_split_rows_f64``; a
    range reaching row n - 1 also covers the pad rows), the other methods
    read U directly and do nothing.  ``syrk`` / ``compute_pass`` take the
    arguments of ``pcc_syrk_f64`` / ``pcc_compute_pass_f64`` after U and
    raise ``DeviceError`` on failure."""

    def __init__(self, method: str, u, n: int, l: int, device=None):
        import torch

        if method not in METHODS:
            raise ValueError(f"unknown contraction method {method!r}, expected one of {METHODS}")
        check_method_shape(method, l)
        if u is None and method != "split":
            raise ValueError("only the split method runs without U (normalize_split)")
        self.method, self.u, self.n, self.l = method, u, int(n), int(l)
        # U may carry extra zero rows (the multi-GPU exchange pads to p blocks);
        # the digit planes cover pcc_rows_padded(n) rows
        rows_pad = int(lib().pcc_rows_padded(n))
        self.ldu = int(u.shape[1]) if u is not None else 0
        self.rows = min(int(u.shape[0]), rows_pad) if u is not None else rows_pad
        dev = u.device if u is not None else device
        if method == "split":
            self.slices = torch.empty(int(lib().pcc_split_slice_bytes(n, l)), dtype=torch.uint8, device=dev)
            self.scale = torch.empty(self.rows, dtype=torch.float64, device=dev)

    def normalize_split(self, x, ldx: int, flags, row_lo: int, row_hi: int, stream) -> None:
        """Split method without U: normalise rows [row_lo, row_hi) of the
        device matrix ``x`` straight into the digit planes
        (``pcc_normalize_split_rows_f64``: the same bits as K1 followed by
        ``prepare``); a range ending at row n also clears the pad rows."""
        check(lib().pcc_normalize_split_rows_f64(x.data_ptr(), ldx, self.n, self.l, flags.data_ptr(), row_lo, row_hi,
                                                 self.slices.data_ptr(), self.scale.data_ptr(), stream),
              "normalize_split")

    def prepare(self, row_lo: int, row_hi: int, stream) -> None:
        if self.method != "split" or row_hi <= row_lo:
            return
        if row_hi >= self.n:
            row_hi = self.rows
        check(lib().pcc_split_rows_f64(self.u.data_ptr(), self.n, self.l, self.ldu, row_lo, row_hi,
                                       self.slices.data_ptr(), self.scale.data_ptr(), stream), "split_rows")

    def prepare_all(self, stream) -> "Contraction":
        self.prepare(0, self.n, stream)
        return self

    def syrk(self, tile_begin: int, tile_end: int, layout: int, out: int, ld_out: int, out_base: int,
             ref_t: int, ref_begin: int, ref_end: int, stream, what: str = "syrk") -> None:
        L = lib()
        if self.method == "split":
            rc = L.pcc_syrk_split_f64(self.slices.data_ptr(), self.scale.data_ptr(), self.n, self.l, tile_begin,
                                      tile_end, layout, out, ld_out, out_base, ref_t, ref_begin, ref_end, stream)
        else:
            rc = syrk_fn(self.method == "exact")(self.u.data_ptr(), self.n, self.l, self.ldu, tile_begin, tile_end,
                                                 layout, out, ld_out, out_base, ref_t, ref_begin, ref_end, stream)
        check(rc, what)

    def compute_pass(self, t: int, j_lo: int, j_hi: int, out: int, stream) -> None:
        L = lib()
        if self.method == "split":
            rc = L.pcc_compute_pass_split_f64(self.slices.data_ptr(), self.scale.data_ptr(), self.n, self.l, t,
                                              j_lo, j_hi, out, stream)
        else:
            fn = L.pcc_compute_pass_exact_f64 if self.method == "exact" else L.pcc_compute_pass_f64
            rc = fn(self.u.data_ptr(), self.n, self.l, self.ldu, t, j_lo, j_hi, out, stream)
        check(rc, "compute_pass")


IPC_HANDLE_BYTES = 64


class DeviceBuffer:
    """Raw ``cudaMalloc`` buffer (``pcc_device_alloc``), or a peer buffer opened
    from a CUDA IPC handle; ``tensor()`` views it as a torch tensor through
    ``__cuda_array_interface__`` (the view keeps the buffer alive)."""

    def __init__(self, nbytes: int = 0, handle: bytes | None = None):
        self.ptr = ctypes.c_void_p()
        self.nbytes = nbytes
        self.opened = handle is not None
        if handle is None:
            check(lib().pcc_device_alloc(nbytes, ctypes.byref(self.ptr)), "pcc_device_alloc")
        else:
            check(lib().pcc_ipc_open_handle(handle, ctypes.byref(self.ptr)), "pcc_ipc_open_handle")
        self._shape = None

    @property
    def address(self) -> int:
        return int(self.ptr.value or 0)

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        check(lib().pcc_ipc_get_handle(self.ptr, buf), "pcc_ipc_get_handle")
        return buf.raw

    def tensor(self, shape, typestr: str):
        import torch

        self._shape = (tuple(shape), typestr)
        return torch.as_tensor(self, device="cuda")

    @property
    def __cuda_array_interface__(self):
        shape, typestr = self._shape
        return {"shape": shape, "typestr": typestr, "data": (self.address, False), "version": 3}

    def close(self) -> None:
        if self.ptr.value:
            if self.opened:
                lib().pcc_ipc_close_handle(self.ptr)
            else:
                lib().pcc_device_free(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass
