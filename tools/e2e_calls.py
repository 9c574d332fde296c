"""Wall time of repeated allpairs(Dataset(pinned X), out=pinned) calls (the
bench e2e leg), one line per call -- to see the spread, not just the median."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200.workloads import make_config

p = argparse.ArgumentParser(); p.add_argument("--config", default="c2"); p.add_argument("--calls", type=int, default=20)
p.add_argument("--chunk-rows", type=int, default=8); p.add_argument("--quiet", action="store_true")
a = p.parse_args()
x = torch.from_numpy(make_config(a.config)).pin_memory()
n = x.shape[0]
ds = pc.Dataset(values=x)
out = torch.empty(n * (n + 1) // 2, dtype=torch.float64).pin_memory()
ts = []
for i in range(a.calls):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    pc.allpairs(ds, out=out, chunk_rows=a.chunk_rows)
    ts.append((time.perf_counter() - t) * 1e3)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    st = torch.cuda.memory_stats()
    if not a.quiet: print(f"call {i}: {ts[-1]:.1f} ms (device stream span {gpu_ms:.1f} ms) reserved {torch.cuda.memory_reserved() / 2**30:.2f} GiB "
          f"retries {st.get('num_alloc_retries', 0)} cudaMalloc {st.get('num_device_alloc', 0)} "
          f"cudaFree {st.get('num_device_free', 0)}", flush=True)
print(" ".join(f"{v:.1f}" for v in ts))
s = sorted(ts[1:])
print(f"median {s[len(s)//2]:.2f} ms  min {s[0]:.2f}  max {s[-1]:.2f}")
