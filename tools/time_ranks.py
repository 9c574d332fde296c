"""Device time of one rank's share of an N-GPU run, timed on one GPU: K1 over
the rows the rank normalises + K2 over its partition(T, p) tile range, and the
implied strong-scaling efficiency t(1) / (p * max_rank t(p)).

--k1 needed (bench.py --u-exchange local): the rank normalises, from its
   resident X, every row its tile range reads (rank 0: all rows).
--k1 block  (bench.py --u-exchange p2p): the rank normalises only its 1/p row
   block (row_slices); the broadcast of the block into the other p - 1 GPUs' U
   rides on NVLink and cannot be timed on one GPU, so it is added as a model:
   (p - 1) / p of U at --nvlink-gbs (peer-store bandwidth; 775 GB/s measured
   for kernel stores on 8x B300 NVLink 5, B300_MICROARCH.md)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1605_01584_b200 import _lib  # noqa: E402
from paper_1605_01584_b200._device import ptr, stream_handle  # noqa: E402
from paper_1605_01584_b200.distributed import partition, row_slices, shard_span  # noqa: E402
from paper_1605_01584_b200.indexing import sym_job_coord  # noqa: E402
from paper_1605_01584_b200.workloads import CONFIGS, make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--configs", default="c1,c2,c3")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--ps", default="1,2,4,8")
p.add_argument("--method", default="tensor", choices=("tensor", "split"))
p.add_argument("--k1", default="needed", choices=("needed", "block"))
p.add_argument("--nvlink-gbs", type=float, default=775.0)
a = p.parse_args()
L = _lib.lib()
for cfg in a.configs.split(","):
    spec = CONFIGS[cfg]
    n, l = spec.n, spec.l
    x = torch.from_numpy(make_config(cfg)).cuda()
    T = int(L.pcc_gpu_tile_count(n))
    mg = -(-n // _lib.GPU_TILE)
    ldu, rows_pad = int(L.pcc_ldu(l)), int(L.pcc_rows_padded(n))
    u = torch.zeros((rows_pad, ldu), dtype=torch.float64, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")

    def timed(fn):
        best = 1e30
        for r in range(a.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r:
                best = min(best, e0.elapsed_time(e1))
        return best

    t1 = None
    for P in map(int, a.ps.split(",")):
        worst, worst_k1 = 0.0, 0.0
        for rank in range(P):
            tb, te = partition(T, P)[rank]
            if te == tb:
                continue
            lo, hi = shard_span(n, tb, te)
            out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            if a.k1 == "needed" or P == 1:
                r0, r1 = sym_job_coord(mg, tb)[0] * _lib.GPU_TILE, n
                exch_ms = 0.0
            else:
                r0, r1 = row_slices(n, P)[0][rank]
                exch_ms = (P - 1) / P * n * ldu * 8 / (a.nvlink_gbs * 1e9) * 1e3
            if a.method == "split":
                con = _lib.Contraction("split", None, n, l, device=x.device)

                def k1():
                    con.normalize_split(x, l, flags, r0, r1, stream_handle())

                def step():  # K1 fused with the digit planes + the split contraction
                    k1()
                    con.syrk(tb, te, 0, ptr(out), 0, lo, 0, 0, 0, stream_handle())
            else:
                def k1():
                    if r1 > r0:
                        _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(u), ldu, ptr(flags), l, r0, r1,
                                                            stream_handle()))

                def step():
                    k1()
                    _lib.check(L.pcc_syrk_f64(ptr(u), n, l, ldu, tb, te, 0, ptr(out), 0, lo, 0, 0, 0,
                                              stream_handle()))
            t = timed(step) + exch_ms
            if t > worst:
                worst, worst_k1 = t, timed(k1) + exch_ms
            del out
        if P == 1:
            t1 = worst
        print(f"{cfg} {a.method} k1={a.k1} p={P}: max rank step {worst:9.3f} ms (K1+exchange of that rank "
              f"{worst_k1:7.3f} ms)   efficiency {t1 / (P * worst) * 100:6.1f}%", flush=True)
    del x, u
    torch.cuda.empty_cache()
