"""Device time of the exact-mode contraction (pcc_syrk_exact_f64, packed) per
config, min of N launches, and its fraction of the FP64 ALU peak (DMUL +
DADD per term = half the DMMA probe in FLOP/s).
    python tools/time_exact.py --configs c2,c3"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1605_01584_b200 import _lib  # noqa: E402
from paper_1605_01584_b200._device import ptr, stream_handle  # noqa: E402
from paper_1605_01584_b200.transform import normalize_device  # noqa: E402
from paper_1605_01584_b200.workloads import CONFIGS, make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--configs", default="c2,c3")
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
L = _lib.lib()
peak = _lib.probe_fp64_peak()
for cfg in a.configs.split(","):
    n, l = CONFIGS[cfg].n, CONFIGS[cfg].l
    x = torch.from_numpy(make_config(cfg)).cuda()
    u, _ = normalize_device(x)
    T = int(L.pcc_gpu_tile_count(n))
    out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda")
    best = 1e30
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.pcc_syrk_exact_f64(ptr(u), n, l, u.shape[1], 0, T, 0, ptr(out), 0, 0, 0, 0, 0, stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        if r:
            best = min(best, e0.elapsed_time(e1))
    tf = 2.0 * l * n * (n + 1) / 2 / (best * 1e-3) / 1e12
    print(f"{cfg}: exact {best:8.3f} ms  {tf:6.2f} TFLOP/s  {tf / (peak / 2) * 100:5.1f}% of the FP64 ALU peak", flush=True)
    del x, u, out
    torch.cuda.empty_cache()
