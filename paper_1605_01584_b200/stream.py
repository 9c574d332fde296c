"""Streamed single-device execution of a GPU tile range: the paper's Alg. 2
(asynchronous double-buffered passes) rebuilt for one
B200 with three engines working at once.

    copy-in stream   X row chunks, host -> HBM, bottom rows first
    compute stream   K1 normalize per arrived chunk
    pass streams     K2 contraction passes over the tile range from the END
                     backwards, each released by the chunk it needs (4
                     rotating streams: small early passes run concurrently)
    copy-out stream  each pass's completed packed rows, HBM -> host

Why bottom-up: tile (Y, X) needs the row bands Y and X >= Y, so a tile row Y
is computable as soon as rows >= 128 Y are resident.  Uploading the bottom
rows first lets the contraction start after a fraction of the upload, and
the packed rows of finished tile rows leave the device while later passes
run.  Pass sizes are whole waves (SMs x resident CTAs) so no pass ends on a
partially idle wave; they ramp up (start early) and down (a short final pass
leaves little copy-out exposed at the end).  Passes of different streams
overlap, so a pass's partial last wave is filled by the next pass's CTAs.

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
    row_lo: int                          # first job row the range needs (upload/normalise [row_lo, n))
    chunks: tuple[tuple[int, int], ...]  # upload/normalise order: bottom-up row chunks
    # launch order: (tile_lo, tile_hi, chunks_needed, dl_row_lo, dl_row_hi, phase):
    # the pass may start once the first `chunks_needed` chunks are
    # normalised; once it and every earlier pass are done, job rows
    # [dl_row_lo, dl_row_hi) are final (empty when dl_row_lo >= dl_row_hi)
    passes: tuple[tuple[int, int, int, int, int, int], ...]


# FP64-equivalent contraction rate (n^2 l / t) per method on one B200, for
# the bottom-up share of the streamed plan
METHOD_RATE = {"tensor": 35e12, "split": 95e12, "exact": 15e12}


def lead_fraction(n: int, resident: bool = False, rate: float = METHOD_RATE["tensor"]) -> float:
    """Share of the range's work done bottom-up while X is still uploading.

    Upload time / contraction time ~= 8 B * FP64 rate / (n * PCIe rate)
    (``rate``, the method's FP64-equivalent contraction rate, ``METHOD_RATE``:
    ~35 TFLOP/s on the FP64 tensor path vs ~50 GB/s); the bottom-up phase should just
    outlast the upload so the top-down phase never waits for data.  The
    1.15 margin is a measured choice (c2 e2e within noise for 0.9-2.0,
    PCC_STREAM_LEAD_SCALE overrides it for experiments).
    """
    if resident:
        return 0.05
    import os

    scale = float(os.environ.get("PCC_STREAM_LEAD_SCALE", "1.15"))  # tuning experiments
    return min(0.95, max(0.05, scale * 8 * rate / (n * 50e9)))


def plan_stream(n: int, tile_begin: int, tile_end: int, wave: int, chunk_rows: int = 8, mid: int = 8,
                lead: float | None = None, half_tail: bool = True,
                rate: float = METHOD_RATE["tensor"]) -> StreamPlan:
    """Plan the streamed execution of GPU tiles ``[tile_begin, tile_end)``.

    X arrives bottom-up in chunks of GPU tile rows -- 2, 2, 4, 4 rows first
    (the contraction can start early), then ``chunk_rows``.  Phase 1 (the
    last ``lead`` share of the range's tiles, bottom rows): each chunk
    releases the tiles whose row bands it completes (tile row Y needs bands
    >= Y only) as one pass, on rotating streams so small early passes share
    the GPU.  Phase 2 (the rest, after the upload): ``mid``-wave passes from
    the TOP row downwards on one stream, ending in a ramp (4, 2, 1, 1/2, 1/2
    waves), so the rows finishing last -- and the download left after the
    final pass -- are short middle rows instead of the longest top rows.
    """
    mg = -(-n // T_G)
    if tile_end <= tile_begin:
        return StreamPlan(n, (), ())
    lead = lead_fraction(n, rate=rate) if lead is None else lead
    y_first = sym_job_coord(mg, tile_begin).y
    row_lo = y_first * T_G
    chunk_rows = max(1, chunk_rows)
    ramp = [r for r in (2, 2, 4, 4) if r < chunk_rows]
    # mostly bottom-up plans (fast methods: the upload and the download are
    # the critical path) end with small top bands (4, 2, 1 tile rows), so the
    # work and the download released by the upload's last chunk are short
    import os

    ramp_on = os.environ.get("PCC_STREAM_TOP_RAMP")  # A/B knob: "0" / "1" force it off / on
    top_ramp = [1, 2, 4] if (lead > 0.5 if ramp_on is None else ramp_on == "1") else []
    top_ramp = [r for r in top_ramp if r < chunk_rows]
    reserved = min(sum(top_ramp), max(0, mg - y_first - sum(ramp)))
    bands = []  # bottom-up tile-row bands [b, t)
    top = mg
    while top > y_first + reserved:
        size = ramp[len(bands)] if len(bands) < len(ramp) else chunk_rows
        b = max(y_first + reserved, top - size)
        bands.append((b, top))
        top = b
    for size in reversed(top_ramp):
        if top <= y_first:
            break
        b = max(y_first, top - size)
        bands.append((b, top))
        top = b
    chunks = tuple((b * T_G, min(n, t * T_G)) for b, t in bands)

    def chunk_of(y: int) -> int:  # 1-based count of chunks needed for rows >= y * 128
        for c, (b, t) in enumerate(bands):
            if b <= y < t:
                return c + 1
        return len(bands)

    total = tile_end - tile_begin
    split = tile_end - min(total, max(0, int(round(lead * total))))  # phase 1 = [split, tile_end)
    passes = []
    # phase 1: bottom-up, one pass per released chunk
    prev_row = n
    for c, (b, t) in enumerate(bands):
        lo = max(split, tile_begin, _F(mg, b))
        hi = min(tile_end, _F(mg, t))
        if hi <= lo:
            continue
        y_lo = sym_job_coord(mg, lo).y
        done_row = min(n, (y_lo if lo == _F(mg, y_lo) else y_lo + 1) * T_G)
        passes.append((lo, hi, c + 1, done_row, prev_row, 1))
        prev_row = min(prev_row, done_row)
    # phase 2: top-down whole waves over [tile_begin, split), ramp at the end
    if split > tile_begin:
        waves = -(-(split - tile_begin) // wave)
        # mid-sized passes, then a ramp down (..., 4, 2, 1, 1 waves)
        tail = [w for w in (4, 2, 1, 1) if w < mid]
        sizes = []
        left = waves
        for w in reversed(tail):
            if left - w >= 1:
                sizes.insert(0, w)
                left -= w
        sizes = [mid] * (left // mid) + ([left % mid] if left % mid else []) + sizes
        sizes = [w * wave for w in sizes]
        excess = sum(sizes) - (split - tile_begin)
        sizes[0] -= excess
        sizes = [s for s in sizes if s > 0]
        if half_tail and len(sizes) > 1 and sizes[-1] == wave and wave >= 2:
            # last wave as two half-wave passes: each runs as one round of
            # 64 x 64 quadrants (half a tile time, csrc/pcc_b200.cu tail
            # kernel), so the download left after the final pass halves
            sizes[-1:] = [wave // 2, wave - wave // 2]
        lo = tile_begin
        top_row = row_lo
        for s_ in sizes:
            hi = lo + s_
            y_h = sym_job_coord(mg, hi).y if hi < _F(mg, mg) else mg
            comp_row = min(n, y_h * T_G)  # rows above the first unprocessed tile's row are final
            passes.append((lo, hi, chunk_of(sym_job_coord(mg, lo).y), top_row, comp_row, 2))
            top_row = max(top_row, comp_row)
            lo = hi
    return StreamPlan(row_lo, chunks, tuple(passes))


def run_stream(x, n: int, l: int, device: torch.device, tile_begin: int, tile_end: int,
               out_dev: torch.Tensor, out_base: int, host_out: torch.Tensor | None,
               host_base: int = 0, chunk_rows: int = 8, trace: list | None = None, resident=None,
               method: str = "tensor"):
    """Execute GPU tiles ``[tile_begin, tile_end)`` with overlapped upload,
    normalisation, contraction and download.

    ``x``: host tensor/array (pinned for asynchronous upload) or a device
    tensor (already resident: no upload).  ``out_dev``: device packed span,
    ``out_dev[i - out_base]`` holds packed cell ``i``.  ``host_out``: if given,
    ``host_out[i - host_base]`` receives every packed cell of the range's span.
    ``trace``: if a list is given, ``(label, cuda.Event)`` pairs are appended
    for the upload, pass and download milestones (tools/trace_stream.py).
    ``resident``: ``(u, flags)`` already normalised on ``device`` (e.g. after
    the multi-GPU row exchange); ``x`` is then ignored and only the
    contraction passes and downloads run (top-down, no upload phase).
    ``method``: the contraction (``_lib.METHODS``; ``"exact"`` = the bit-exact
    dot8 kernel, ``"split"`` = int8 digit planes written chunk by chunk by
    the normaliser itself -- no U; the returned ``u`` is then None).
    Returns ``(u, flags, x_device)`` after the host has synchronised
    (``x_device`` is None with ``resident``).
    """

    def mark(label, stream):
        torch.cuda.nvtx.mark(f"pcc.stream.{label}")
        if trace is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            trace.append((label, ev))

    L = _lib.lib()
    with torch.cuda.device(device):
        info = _lib.device_info(device.index)
        wave = info.sm_count * info.syrk_ctas_per_sm
        plan = plan_stream(n, tile_begin, tile_end, wave, chunk_rows, lead=0.0 if resident is not None else None,
                           rate=METHOD_RATE[method])
        compute = torch.cuda.current_stream()
        s = stream_handle(compute)
        mark("start", compute)
        if resident is not None:
            u, flags = resident
            ldu = int(u.shape[1])
        elif method == "split":
            # no U: each chunk is normalised straight into the digit planes
            u, ldu = None, 0
            flags = torch.zeros(n, dtype=torch.uint8, device=device)
        else:
            rows_pad = int(L.pcc_rows_padded(n))
            ldu = int(L.pcc_ldu(l))
            u = torch.empty((rows_pad, ldu), dtype=torch.float64, device=device)
            flags = torch.zeros(n, dtype=torch.uint8, device=device)
            _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, rows_pad, s), "pad rows")
        con = _lib.Contraction(method, u, n, l, device=device)
        if resident is not None:
            con.prepare_all(s)

        on_device = resident is not None or (isinstance(x, torch.Tensor) and x.is_cuda)
        if resident is not None:
            xd = None
        elif on_device:
            xd = x if x.dtype == torch.float64 else x.to(torch.float64)
            xd = xd.contiguous()
        else:
            xh = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            pinned_in = xh.is_pinned()
            xd = torch.empty((n, l), dtype=torch.float64, device=device)
            copy_in = torch.cuda.Stream(device)
            copy_in.wait_stream(compute)  # xd's memory is free from the compute stream's view
            if not pinned_in:
                # pageable source: two pinned staging slots (torch's caching host
                # allocator keeps them across calls); the host copies chunk c+1
                # (multi-threaded) while chunk c uploads
                max_rows = max((hi_ - lo_ for lo_, hi_ in plan.chunks), default=0)
                stage_in = [torch.empty(max(1, max_rows * l), dtype=torch.float64, pin_memory=True)
                            for _ in range(2)]
                stage_in_ev = [None, None]
        pinned_out = host_out is not None and host_out.is_pinned()
        if host_out is not None:
            copy_out = torch.cuda.Stream(device)

        span_lo = out_base
        span_hi = out_base + out_dev.numel()
        workers = [torch.cuda.Stream(device) for _ in range(min(4, max(1, len(plan.passes))))]
        for w in workers:
            w.wait_stream(compute)  # u / out_dev allocations precede every pass
        pass_done = []  # (event, dl_row_lo, dl_row_hi) per launched pass, in plan order
        downloaded = []  # job-row intervals already copied

        if host_out is not None and not pinned_out:
            # pageable destination: D2H into two pinned staging slots, the host
            # copies each piece out (multi-threaded; first touch of the pages
            # included) while the next piece transfers
            piece = int(min(max(1, span_hi - span_lo), 1 << 24))  # <= 128 MB per piece
            stage_out = [torch.empty(piece, dtype=torch.float64, pin_memory=True) for _ in range(2)]
            out_pending = []  # (event, slot, a, b) in issue order
            out_next = [0]

        def drain_one() -> None:
            ev, sl, a, b = out_pending.pop(0)
            ev.synchronize()
            host_out[a - host_base:b - host_base].copy_(stage_out[sl][:b - a])

        def copy_rows(r_lo: int, r_hi: int, label: str) -> None:
            a = max(span_lo, _F(n, r_lo))
            b = min(span_hi, _F(n, r_hi))
            if b > a:
                if pinned_out:
                    with torch.cuda.stream(copy_out):
                        host_out[a - host_base:b - host_base].copy_(out_dev[a - out_base:b - out_base],
                                                                    non_blocking=True)
                else:
                    for pa in range(a, b, piece):
                        pb = min(b, pa + piece)
                        if len(out_pending) == 2:
                            drain_one()  # frees the slot used two pieces ago
                        sl = out_next[0] % 2
                        out_next[0] += 1
                        with torch.cuda.stream(copy_out):
                            stage_out[sl][:pb - pa].copy_(out_dev[pa - out_base:pb - out_base], non_blocking=True)
                            ev = torch.cuda.Event()
                            ev.record(copy_out)
                        out_pending.append((ev, sl, pa, pb))
                mark(f"download {8 * (b - a) / 1e6:.0f} MB{label}", copy_out)
            downloaded.append((r_lo, r_hi))

        dl_next = [0]  # next pass_done entry to download (a list, not a function
        #               attribute: a self-referencing closure would keep this call's
        #               device buffers alive until the cyclic GC runs)

        def download(upto: int) -> None:
            # in-order waits: a copy runs only after its pass and every earlier pass
            while dl_next[0] < upto:
                ev, r_lo, r_hi = pass_done[dl_next[0]]
                dl_next[0] += 1
                copy_out.wait_event(ev)
                if r_hi > r_lo:
                    copy_rows(r_lo, r_hi, "")

        k = 0
        for c, (lo, hi) in enumerate(plan.chunks):
            # upload (pageable sources block here while the GPU runs earlier passes)
            if not on_device:
                if pinned_in:
                    src = xh[lo:hi]
                else:
                    sl = c % 2
                    if stage_in_ev[sl] is not None:
                        stage_in_ev[sl].synchronize()  # the slot's previous upload has finished
                    src = stage_in[sl][:(hi - lo) * l].view(hi - lo, l)
                    src.copy_(xh[lo:hi])
                with torch.cuda.stream(copy_in):
                    xd[lo:hi].copy_(src, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(copy_in)
                    mark(f"upload rows [{lo},{hi})", copy_in)
                if not pinned_in:
                    stage_in_ev[c % 2] = up
                compute.wait_event(up)
            if resident is None and u is None:
                con.normalize_split(xd, xd.stride(0), flags, lo, hi, s)
            elif resident is None:
                _lib.check(L.pcc_normalize_rows_f64(ptr(xd), xd.stride(0), ptr(u), ldu, ptr(flags), l, lo, hi, s),
                           "normalize")
            normed = torch.cuda.Event()
            normed.record(compute)
            # every pass whose rows are now normalised, in plan order
            while k < len(plan.passes) and plan.passes[k][2] <= c + 1:
                p_lo, p_hi, _, dl_lo, dl_hi, phase = plan.passes[k]
                # phase 1 (upload-limited, small passes): rotating streams run them
                # side by side; phase 2: one stream, so passes -- and their
                # downloads -- complete in order
                ws = workers[k % len(workers)] if phase == 1 else workers[0]
                ws.wait_event(normed)
                mark(f"  start [{p_lo},{p_hi})", ws)
                con.syrk(p_lo, p_hi, _lib.LAYOUT_PACKED, ptr(out_dev), 0, out_base, 0, 0, 0, stream_handle(ws))
                done = torch.cuda.Event()
                done.record(ws)
                mark(f"pass tiles [{p_lo},{p_hi})", ws)
                pass_done.append((done, dl_lo, dl_hi))
                k += 1
            if pinned_out:
                download(len(pass_done))
        assert k == len(plan.passes)
        for w in workers:
            compute.wait_stream(w)
        if host_out is not None:
            download(len(pass_done))  # pageable destinations: staged copies once all work is queued
            copy_out.wait_stream(compute)
            # rows no pass completed on its own (a row split between the two phases)
            cur = plan.row_lo
            for a, b in sorted(downloaded) + [(n, n)]:
                if a > cur:
                    copy_rows(cur, a, " (final)")
                cur = max(cur, b)
            if not pinned_out:
                while out_pending:
                    drain_one()
            copy_out.synchronize()
        compute.synchronize()
        return u, flags, xd
