"""Time every contraction kernel shape (pcc_syrk_f64_variant) on the BASELINE
configs and check they agree bit for bit.  Prints one line per (config, variant).

The tuning shapes 1..14 are not in the product library: this tool loads the
tools build (``make -C tools`` -> tools/libpcc_tune.so, the same source with
-DPCC_TUNING_VARIANTS)."""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_1605_01584_b200 import _lib  # noqa: E402
from paper_1605_01584_b200._device import ptr, stream_handle  # noqa: E402
from paper_1605_01584_b200.transform import normalize_device  # noqa: E402
from paper_1605_01584_b200.workloads import CONFIGS, make_config  # noqa: E402


def _check(L, rc):
    if rc != 0:
        raise RuntimeError(L.pcc_last_error().decode())


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="c2,c3")
    p.add_argument("--variants", default="0,1,2,3,4")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    tune_path = Path(__file__).resolve().parent / "libpcc_tune.so"
    if not tune_path.exists():
        raise SystemExit("build the tools library first: make -C tools")
    L = ctypes.CDLL(str(tune_path))
    _lib._bind(L)
    peak = _lib.probe_fp64_peak()
    print(f"DMMA probe peak {peak:.2f} TFLOP/s", flush=True)
    for cfg in a.configs.split(","):
        spec = CONFIGS[cfg]
        n, l = spec.n, spec.l
        x = torch.from_numpy(make_config(cfg)).cuda()
        u, _ = normalize_device(x)
        T = int(L.pcc_gpu_tile_count(n))
        ref = None
        for v in map(int, a.variants.split(",")):
            out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device="cuda")
            s = stream_handle()
            best = 1e30
            for r in range(a.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _check(L, L.pcc_syrk_f64_variant(v, ptr(u), n, l, u.shape[1], 0, T, 0, ptr(out), 0, 0, 0, 0, 0, s))
                e1.record()
                torch.cuda.synchronize()
                if r:
                    best = min(best, e0.elapsed_time(e1))
            tf = float(n) * n * l / (best * 1e-3) / 1e12
            same = "ref" if ref is None else ("bitwise-equal" if torch.equal(out, ref) else "DIFFERENT")
            if ref is None:
                ref = out
            print(f"{cfg} variant {v}: {best:8.3f} ms  {tf:6.2f} TFLOP/s (n^2 l)  {tf / peak * 100:5.1f}% of probe  {same}",
                  flush=True)
            del out
        del ref, u, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
