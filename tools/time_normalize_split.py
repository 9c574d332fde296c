"""Device time of the fused normaliser -> digit planes (pcc_normalize_split_rows_f64)
on BASELINE configs (min of 5 launches):  python tools/time_normalize_split.py --configs c2,c4,c5"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200.workloads import make_config

p = argparse.ArgumentParser()
p.add_argument("--configs", default="c2,c4,c5")
a = p.parse_args()
out = []
for cfg in a.configs.split(","):
    x = torch.from_numpy(make_config(cfg)).cuda()
    n, l = x.shape
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    con = _lib.Contraction("split", None, n, l, device=x.device)
    s = torch.cuda.current_stream().cuda_stream
    best = 1e30
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        con.normalize_split(x, l, flags, 0, n, s)
        e1.record()
        torch.cuda.synchronize()
        if r:
            best = min(best, e0.elapsed_time(e1))
    out.append(f"{cfg} {best * 1e3:.1f} us")
    del x, con
print("  ".join(out))
