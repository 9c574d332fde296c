"""Time K1 (pcc_normalize_rows_f64) per config: CUDA events, best of N, and
the achieved algorithmic HBM bandwidth (read X once + write U once)."""
import argparse, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200._device import ptr, stream_handle
from paper_1605_01584_b200.workloads import CONFIGS, make_config

def main():
    p = argparse.ArgumentParser(); p.add_argument("--configs", default="c1,c2,c3,c4,c5"); p.add_argument("--reps", type=int, default=5)
    p.add_argument("--check", action="store_true", help="also compare U and the flags bit for bit with the CPU oracle")
    a = p.parse_args()
    L = _lib.lib()
    peaks = {}
    try:
        peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())
    except OSError:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    for cfg in a.configs.split(","):
        spec = CONFIGS[cfg]; n, l = spec.n, spec.l
        x = torch.from_numpy(make_config(cfg)).cuda()
        ldu = int(L.pcc_ldu(l)); rows = int(L.pcc_rows_padded(n))
        u = torch.empty((rows, ldu), dtype=torch.float64, device="cuda")
        fl = torch.empty(n, dtype=torch.uint8, device="cuda")
        s = stream_handle()
        best = 1e9
        for r in range(a.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(u), ldu, ptr(fl), l, 0, n, s))
            e1.record(); torch.cuda.synchronize()
            if r: best = min(best, e0.elapsed_time(e1))
        byt = 8.0 * n * l * 2
        if a.check:
            import numpy as np
            sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
            import oracle
            xh = make_config(cfg)
            u_ref, zv_ref = oracle.normalize(xh)
            same = np.array_equal(u[:n, :l].cpu().numpy().view(np.uint64), u_ref.view(np.uint64)) and \
                np.array_equal(fl.cpu().numpy().astype(bool), zv_ref) and float(u[:, l:].abs().max() if ldu > l else 0) == 0.0
            print(f"{cfg}: bit-exact vs oracle: {same}", flush=True)
        print(f"{cfg}: normalize {best*1e3:8.1f} us  {byt/best/1e6:7.1f} GB/s algorithmic  {byt/best/1e6/hbm*100:5.1f}% of HBM {hbm:.0f} GB/s", flush=True)
        del x, u, fl; torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
