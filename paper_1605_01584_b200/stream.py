"""Streamed single-device execution of a GPU tile range: the paper's Alg. 2
(asynchronous double-buffered passes) rebuilt for one
B200 with three engines working at once.

    copy-in stream   X row chunks, host -> HBM, bottom rows first
    compute stream   K1 normalize per arrived chunk, then K2 contraction
                     passes over the tile range from the END backwards
    copy-out stream  each pass's completed packed rows, HBM -> host

Why bottom-up: tile (Y, X) needs the row bands Y and X >= Y, so a tile row Y
is computable as soon as rows >= 128 Y are resident.  Uploading the bottom
rows first lets the contraction start after a fraction of the upload, and
the packed rows of finished tile rows leave the device while later passes
run.  Pass sizes are whole waves (SMs x resident CTAs) so no pass ends on a
partially idle wave; they ramp up (start early) and down (a short final pass
leaves little copy-out exposed at the end).

Results do not depend on the schedule: every cell's K order is fixed by the
kernel (see csrc/syrk.cuh), so this path is bitwise identical to a single
launch over the whole range.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import ptr, stream_handle
from .indexing import sym_job_coord

__all__ = ["wave_plan", "plan_stream", "StreamPlan", "run_stream"]

T_G = _lib.GPU_TILE


def _F(n: int, y: int) -> int:
    return (y * (2 * n + 1 - y)) >> 1


def wave_plan(waves: int, mid: int = 8) -> list[int]:
    """Pass sizes in waves: 1, 1, 2, 4, ... up to ``mid``, ``mid`` x k, ..., 4, 2, 1, 1."""
    if waves <= 0:
        return []
    if waves <= 4:
        return [1] * waves
    m = max(1, min(mid, waves // 6))
    up = [1]
    while up[-1] * 2 <= m and sum(up) + up[-1] * 2 <= waves // 2:
        up.append(up[-1] * 2)
    up = [1] + up if len(up) > 1 else up
    down = list(reversed(up))
    rest = waves - sum(up) - sum(down)
    while rest < 0:
        down.pop(0) if down else up.pop()
        rest = waves - sum(up) - sum(down)
    middle = [m] * (rest // m) + ([rest % m] if rest % m else [])
    return up + middle + down


@dataclass(frozen=True)
class StreamPlan:
    row_lo: int                         # first job row the range needs (upload/normalise [row_lo, n))
    chunks: tuple[tuple[int, int], ...]  # upload/normalise order: bottom-up row chunks
    passes: tuple[tuple[int, int, int, int], ...]  # (tile_lo, tile_hi, need_row, copy_lo_row) in launch order


def plan_stream(n: int, tile_begin: int, tile_end: int, wave: int, chunks: int = 16, mid: int = 8) -> StreamPlan:
    """Plan the streamed execution of GPU tiles ``[tile_begin, tile_end)``.

    ``need_row``: rows ``[need_row, n)`` must be normalised before the pass;
    ``copy_lo_row``: after the pass, packed rows ``>= copy_lo_row`` (within
    the range's span) are final.
    """
    mg = -(-n // T_G)
    if tile_end <= tile_begin:
        return StreamPlan(n, (), ())
    y_first = sym_job_coord(mg, tile_begin).y
    row_lo = y_first * T_G
    # bottom-up row chunks aligned to the GPU tile
    bands = mg - y_first
    k = max(1, min(chunks, bands))
    per = -(-bands // k)
    cuts = []
    top = mg
    while top > y_first:
        b = max(y_first, top - per)
        cuts.append((b * T_G, min(n, top * T_G)))
        top = b
    total = tile_end - tile_begin
    waves = -(-total // wave)
    sizes = [w * wave for w in wave_plan(waves, mid)]
    # the partial wave goes to the first (bottom-most) pass, hidden under the upload
    excess = sum(sizes) - total
    sizes[0] -= excess
    if sizes[0] <= 0:
        sizes[1] += sizes[0]
        sizes.pop(0)
    passes = []
    hi = tile_end
    for s in sizes:
        lo = hi - s
        y_lo, x_lo = sym_job_coord(mg, lo)
        need = y_lo * T_G
        # tile rows fully done once every tile from the row's first tile up is computed
        row_first = _F(mg, y_lo)
        done_y = y_lo if lo == row_first else y_lo + 1
        passes.append((lo, hi, need, min(n, done_y * T_G)))
        hi = lo
    assert hi == tile_begin
    return StreamPlan(row_lo, tuple(cuts), tuple(passes))


def run_stream(x, n: int, l: int, device: torch.device, tile_begin: int, tile_end: int,
               out_dev: torch.Tensor, out_base: int, host_out: torch.Tensor | None,
               host_base: int = 0, chunks: int = 16):
    """Execute GPU tiles ``[tile_begin, tile_end)`` with overlapped upload,
    normalisation, contraction and download.

    ``x``: host tensor/array (pinned for asynchronous upload) or a device
    tensor (already resident: no upload).  ``out_dev``: device packed span,
    ``out_dev[i - out_base]`` holds packed cell ``i``.  ``host_out``: if given,
    ``host_out[i - host_base]`` receives every packed cell of the range's span.
    Returns ``(u, flags)`` (device) after the host has synchronised.
    """
    L = _lib.lib()
    with torch.cuda.device(device):
        info = _lib.device_info(device.index)
        wave = info.sm_count * info.syrk_ctas_per_sm
        plan = plan_stream(n, tile_begin, tile_end, wave, chunks)
        compute = torch.cuda.current_stream()
        s = stream_handle(compute)
        rows_pad = int(L.pcc_rows_padded(n))
        ldu = int(L.pcc_ldu(l))
        u = torch.empty((rows_pad, ldu), dtype=torch.float64, device=device)
        flags = torch.zeros(n, dtype=torch.uint8, device=device)
        _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, rows_pad, s), "pad rows")

        on_device = isinstance(x, torch.Tensor) and x.is_cuda
        if on_device:
            xd = x if x.dtype == torch.float64 else x.to(torch.float64)
            xd = xd.contiguous()
            up_events = None
        else:
            xh = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            pinned = xh.is_pinned()
            xd = torch.empty((n, l), dtype=torch.float64, device=device)
            copy_in = torch.cuda.Stream(device)
            copy_in.wait_stream(compute)  # xd's memory is free from the compute stream's view
            up_events = []
            with torch.cuda.stream(copy_in):
                for lo, hi in plan.chunks:
                    xd[lo:hi].copy_(xh[lo:hi], non_blocking=pinned)
                    ev = torch.cuda.Event()
                    ev.record(copy_in)
                    up_events.append(ev)
        if host_out is not None:
            copy_out = torch.cuda.Stream(device)
            pinned_out = host_out.is_pinned()

        span_lo = out_base
        span_hi = out_base + out_dev.numel()
        normalized = 0  # chunks normalised so far (bottom-up)
        copied_to_row = n  # packed rows >= this are already downloaded
        for p_lo, p_hi, need_row, done_row in plan.passes:
            while normalized < len(plan.chunks) and plan.chunks[normalized][1] > need_row:
                lo, hi = plan.chunks[normalized]
                if up_events is not None:
                    compute.wait_event(up_events[normalized])
                _lib.check(L.pcc_normalize_rows_f64(ptr(xd), xd.stride(0), ptr(u), ldu, ptr(flags), l, lo, hi, s),
                           "normalize")
                normalized += 1
            _lib.check(L.pcc_syrk_f64(ptr(u), n, l, ldu, p_lo, p_hi, _lib.LAYOUT_PACKED, ptr(out_dev), 0, out_base,
                                      0, 0, 0, s), "syrk")
            if host_out is not None and done_row < copied_to_row:
                a = max(span_lo, _F(n, done_row))
                b = min(span_hi, _F(n, copied_to_row))
                if b > a:
                    ev = torch.cuda.Event()
                    ev.record(compute)
                    copy_out.wait_event(ev)
                    with torch.cuda.stream(copy_out):
                        host_out[a - host_base:b - host_base].copy_(out_dev[a - out_base:b - out_base],
                                                                    non_blocking=pinned_out)
                copied_to_row = done_row
        # any rows the range did not finish (its first, partial tile row) and
        # never-normalised chunks (rows the range does not touch)
        while normalized < len(plan.chunks):
            lo, hi = plan.chunks[normalized]
            if up_events is not None:
                compute.wait_event(up_events[normalized])
            _lib.check(L.pcc_normalize_rows_f64(ptr(xd), xd.stride(0), ptr(u), ldu, ptr(flags), l, lo, hi, s),
                       "normalize")
            normalized += 1
        if host_out is not None:
            a = span_lo
            b = min(span_hi, _F(n, copied_to_row))
            if b > a:
                ev = torch.cuda.Event()
                ev.record(compute)
                copy_out.wait_event(ev)
                with torch.cuda.stream(copy_out):
                    host_out[a - host_base:b - host_base].copy_(out_dev[a - out_base:b - out_base],
                                                                non_blocking=pinned_out)
            copy_out.synchronize()
        compute.synchronize()
        return u, flags, xd
