"""allpairs() end to end from plain numpy input (pageable host memory, result
allocated by the call) -- what a drop-in caller of the reference API does --
next to the pinned-buffer path bench.py reports."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200.workloads import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
x = make_config(cfg)
ds = pc.Dataset(values=x)
for label, kw in (("numpy in, result allocated by the call", {}),
                  ("numpy in, caller-owned numpy out", {"out": np.empty(x.shape[0] * (x.shape[0] + 1) // 2)})):
    ts = []
    for i in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = pc.allpairs(ds, **kw)
        ts.append((time.perf_counter() - t) * 1e3)
    s = sorted(ts[1:])
    print(f"{cfg} {label}: median {s[len(s)//2]:.1f} ms  min {s[0]:.1f}", flush=True)
