"""Minimal driver for ncu: W warm-up + K device steps (normalize + syrk) of a config.

    python tools/profile_step.py --config c2 --steps 2
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
        python tools/profile_step.py --config c2 --steps 2

Same kernels and arguments as bench.py's timed region, without the e2e,
CPU-baseline and clock-sampling legs.
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1605_01584_b200 import _lib  # noqa: E402
from paper_1605_01584_b200._device import ptr, stream_handle  # noqa: E402
from paper_1605_01584_b200.transform import normalize_device  # noqa: E402
from paper_1605_01584_b200.workloads import CONFIGS, make_config  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--l", type=int, default=None)
    a = p.parse_args()
    spec = CONFIGS[a.config]
    n = a.n or spec.n
    l = a.l or spec.l
    x = torch.from_numpy(make_config(a.config, n=n, l=l)).cuda()
    L = _lib.lib()
    T = int(L.pcc_gpu_tile_count(n))
    out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda")
    s = stream_handle()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(a.warmup + a.steps):
        u, flags = normalize_device(x)
        ev[0].record()
        _lib.check(L.pcc_syrk_f64(ptr(u), n, l, u.shape[1], 0, T, 0, ptr(out), 0, 0, 0, 0, 0, s))
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1])
        print(f"step {i}: syrk {ms:.3f} ms  {float(n) * n * l / ms / 1e9:.2f} TFLOP/s (n^2 l)")


if __name__ == "__main__":
    main()
