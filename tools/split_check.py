"""Split mode (int8 tensor cores, Ozaki digits) against the FP64 tensor path
on one GPU: max |split - dmma| over the whole packed result, plus device
times of the slicing kernel and both contractions.

    python tools/split_check.py --config c2 [--reps 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200.workloads import make_config

p = argparse.ArgumentParser()
p.add_argument("--config", default="c1")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--skip-dmma", action="store_true")
p.add_argument("--sustain", type=int, default=0, help="also time N back-to-back split launches with clock sampling")
p.add_argument("--hash", action="store_true", help="print the sha256 of the split result (A/B bit-identity checks)")
a = p.parse_args()
L = _lib.lib()
x = torch.from_numpy(make_config(a.config)).cuda()
n, l = x.shape
R, ldu = L.pcc_rows_padded(n), L.pcc_ldu(l)
u = torch.zeros((R, ldu), dtype=torch.float64, device="cuda")
zv = torch.empty(n, dtype=torch.uint8, device="cuda")
s0 = torch.cuda.current_stream().cuda_stream
_lib.check(L.pcc_normalize_rows_f64(x.data_ptr(), l, u.data_ptr(), ldu, zv.data_ptr(), l, 0, n, s0), "normalize")
slices = torch.empty(L.pcc_split_slice_bytes(n, l), dtype=torch.uint8, device="cuda")
scale = torch.empty(R, dtype=torch.float64, device="cuda")
tiles = L.pcc_gpu_tile_count(n)
pairs = n * (n + 1) // 2
out_s = torch.full((pairs,), float("nan"), dtype=torch.float64, device="cuda")
out_d = torch.full((pairs,), float("nan"), dtype=torch.float64, device="cuda")


def timed(fn):
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


t_split_rows = timed(lambda: _lib.check(L.pcc_split_rows_f64(u.data_ptr(), n, l, ldu, 0, R, slices.data_ptr(),
                                                               scale.data_ptr(), s0), "split_rows"))
t_split = timed(lambda: _lib.check(L.pcc_syrk_split_f64(slices.data_ptr(), scale.data_ptr(), n, l, 0, tiles,
                                                        _lib.LAYOUT_PACKED, out_s.data_ptr(), 0, 0, 0, 0, 0, s0),
                                   "syrk_split"))
flops = float(n) * n * l
prod = _lib.split_products(scale, n, l, 0, tiles)
print(f"{a.config}: products per tile {prod / tiles:.2f} (34 = full depth, 28 = adaptive depth everywhere)")
print(f"{a.config}: n={n} l={l}  split_rows {t_split_rows:.3f} ms  split syrk {t_split:.3f} ms "
      f"({flops / t_split / 1e9:.1f} TFLOP/s-equivalent n^2 l/t)", flush=True)
if a.hash:
    import hashlib
    print(f"  split result sha256 {hashlib.sha256(out_s.cpu().numpy().tobytes()).hexdigest()[:24]}", flush=True)
if not a.skip_dmma:
    t_d = timed(lambda: _lib.check(L.pcc_syrk_f64(u.data_ptr(), n, l, ldu, 0, tiles, _lib.LAYOUT_PACKED,
                                                  out_d.data_ptr(), 0, 0, 0, 0, 0, s0), "syrk"))
    d = (out_s - out_d).abs()
    print(f"  dmma syrk {t_d:.3f} ms ({flops / t_d / 1e9:.1f} TFLOP/s)  speed-up {t_d / t_split:.2f}x", flush=True)
    print(f"  nan in split: {int(torch.isnan(out_s).sum())}  max|split - dmma| = {float(d.max()):.3e}  "
          f"mean = {float(d.mean()):.3e}", flush=True)

if a.sustain:
    from bench import ClockSampler

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.sustain)]
    torch.cuda.synchronize()
    with ClockSampler(0) as cs:
        for e0, e1 in evs:
            e0.record()
            _lib.check(L.pcc_syrk_split_f64(slices.data_ptr(), scale.data_ptr(), n, l, 0, tiles, _lib.LAYOUT_PACKED,
                                            out_s.data_ptr(), 0, 0, 0, 0, 0, s0), "syrk_split")
            e1.record()
        torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) for e0, e1 in evs]
    print(f"  sustained x{a.sustain}: first {ts[0]:.3f} ms, median {sorted(ts)[len(ts) // 2]:.3f} ms, "
          f"last {ts[-1]:.3f} ms; clocks {cs.summary()}", flush=True)
