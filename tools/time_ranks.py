"""Device time of one rank's share (K1 over the rows it needs + K2 over its
partition(T, p) tile range) -- the per-GPU step of an N-GPU run, timed on one
GPU -- and the implied strong-scaling efficiency t(1) / (p * max_rank t(p))."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200._device import ptr, stream_handle
from paper_1605_01584_b200.distributed import partition, shard_span
from paper_1605_01584_b200.transform import normalize_device
from paper_1605_01584_b200.workloads import CONFIGS, make_config

p = argparse.ArgumentParser(); p.add_argument("--configs", default="c1,c2,c3"); p.add_argument("--reps", type=int, default=3)
p.add_argument("--ps", default="1,2,4,8")
p.add_argument("--method", default="tensor", choices=("tensor", "split"))
a = p.parse_args()
L = _lib.lib()
for cfg in a.configs.split(","):
    spec = CONFIGS[cfg]; n, l = spec.n, spec.l
    x = torch.from_numpy(make_config(cfg)).cuda()
    T = int(L.pcc_gpu_tile_count(n))
    def timed(fn):
        best = 1e30
        for r in range(a.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if r: best = min(best, e0.elapsed_time(e1))
        return best
    t1 = None
    for P in map(int, a.ps.split(",")):
        worst = 0.0
        for rank in range(P):
            tb, te = partition(T, P)[rank]
            if te == tb:
                continue
            lo, hi = shard_span(n, tb, te)
            out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            if a.method == "split":
                flags = torch.empty(n, dtype=torch.uint8, device="cuda")

                def step():  # K1 fused with the digit planes + the split contraction
                    con = _lib.Contraction("split", None, n, l, device=x.device)
                    con.normalize_split(x, l, flags, 0, n, stream_handle())
                    con.syrk(tb, te, 0, ptr(out), 0, lo, 0, 0, 0, stream_handle())
            else:
                def step():
                    u, f = normalize_device(x)
                    _lib.check(L.pcc_syrk_f64(ptr(u), n, l, u.shape[1], tb, te, 0, ptr(out), 0, lo, 0, 0, 0,
                                              stream_handle()))
            worst = max(worst, timed(step))
            del out
        if P == 1:
            t1 = worst
        print(f"{cfg} {a.method} p={P}: max rank step {worst:9.3f} ms   efficiency {t1 / (P * worst) * 100:6.1f}%", flush=True)
    del x; torch.cuda.empty_cache()
