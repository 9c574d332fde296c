"""Device plumbing: resolving devices, streams and host<->device staging.

PyTorch is used only for device memory, streams and events; every
arithmetic step of the hot path runs in libpcc_b200.so (see _lib.py).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import DeviceError

__all__ = ["require_cuda", "resolve_devices", "stream_handle", "as_device_f64", "ptr", "nvtx"]


def nvtx(name: str):
    """NVTX range around a host-side phase (visible in Nsight Systems / ncu
    --nvtx timelines): ``with nvtx("pcc.allpairs"): ...``."""
    return torch.cuda.nvtx.range(name)


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible: the B200 engine has no CPU fallback")


def resolve_devices(devices=None) -> list[torch.device]:
    """``None`` -> [current device]; int -> first k devices; list -> those devices."""
    require_cuda()
    if devices is None:
        return [torch.device("cuda", torch.cuda.current_device())]
    if isinstance(devices, int):
        if devices < 1:
            raise ValueError(f"device count must be >= 1, got {devices}")
        avail = torch.cuda.device_count()
        if devices > avail:
            raise ValueError(f"{devices} devices requested but only {avail} visible")
        return [torch.device("cuda", i) for i in range(devices)]
    out = []
    for d in devices:
        d = torch.device(d) if not isinstance(d, int) else torch.device("cuda", d)
        if d.type != "cuda":
            raise ValueError(f"device {d} is not a CUDA device")
        out.append(d)
    if not out:
        raise ValueError("empty device list")
    return out


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr())


def as_device_f64(values, device: torch.device, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """C-contiguous float64 copy of ``values`` on ``device`` (async from pinned memory)."""
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64))
    if t.device == device:
        return t.contiguous()
    with torch.cuda.stream(stream) if stream is not None else _null():
        return t.to(device, non_blocking=t.is_pinned()).contiguous()


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
