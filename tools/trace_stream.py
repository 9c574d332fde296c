"""Timeline of one streamed allpairs call (stream.run_stream milestones)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200.stream import run_stream
from paper_1605_01584_b200.workloads import CONFIGS, make_config

p = argparse.ArgumentParser(); p.add_argument("--config", default="c2"); p.add_argument("--chunk-rows", type=int, default=4)
p.add_argument("--method", default="tensor")
a = p.parse_args()
spec = CONFIGS[a.config]; n, l = spec.n, spec.l
x = torch.from_numpy(make_config(a.config)).pin_memory()
T = int(_lib.lib().pcc_gpu_tile_count(n))
dev = torch.device("cuda", 0)
out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=dev)
host = torch.empty(n * (n + 1) // 2, dtype=torch.float64).pin_memory()
for it in range(3):
    tr = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_stream(x, n, l, dev, 0, T, out, 0, host, 0, chunk_rows=a.chunk_rows, trace=tr, method=a.method)
    wall = time.perf_counter() - t0
    torch.cuda.synchronize()
    if it == 2:
        s0 = tr[0][1]
        for label, ev in sorted(tr, key=lambda t: s0.elapsed_time(t[1])):
            print(f"{s0.elapsed_time(ev):8.2f} ms  {label}")
    print(f"wall {wall*1e3:.2f} ms")
