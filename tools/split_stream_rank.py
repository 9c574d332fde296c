import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200._device import ptr, stream_handle
from paper_1605_01584_b200.distributed import partition, shard_span
from paper_1605_01584_b200.stream import run_stream
from paper_1605_01584_b200.workloads import CONFIGS, make_config
L = _lib.lib()
for cfg in ("c2", "c4"):
    spec = CONFIGS[cfg]; n, l = spec.n, spec.l
    x = torch.from_numpy(make_config(cfg)).cuda()
    T = int(L.pcc_gpu_tile_count(n))
    dev = x.device
    def timed(fn, reps=3):
        best = 1e30
        for r in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if r: best = min(best, e0.elapsed_time(e1))
        return best
    for P in (1, 8):
        worst_seq = worst_str = 0.0
        for rank in range(P):
            tb, te = partition(T, P)[rank]
            lo, hi = shard_span(n, tb, te)
            out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            flags = torch.empty(n, dtype=torch.uint8, device="cuda")
            def seq():
                con = _lib.Contraction("split", None, n, l, device=dev)
                con.normalize_split(x, l, flags, 0, n, stream_handle())
                con.syrk(tb, te, 0, ptr(out), 0, lo, 0, 0, 0, stream_handle())
            def streamed():
                run_stream(x, n, l, dev, tb, te, out, lo, None, method="split")
            worst_seq = max(worst_seq, timed(seq)); worst_str = max(worst_str, timed(streamed))
            del out
        print(f"{cfg} p={P}: sequential {worst_seq:.3f} ms  streamed {worst_str:.3f} ms", flush=True)
