"""Run K1 (pcc_normalize_rows_f64) on one BASELINE config a few times -- an
ncu target:  ncu -k regex:normalize python tools/k1_once.py --config c2
--split: the fused normaliser -> digit planes (pcc_normalize_split_rows_f64)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1605_01584_b200 import _lib  # noqa: E402
from paper_1605_01584_b200._device import ptr, stream_handle  # noqa: E402
from paper_1605_01584_b200.workloads import make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--split", action="store_true")
a = p.parse_args()
L = _lib.lib()
x = torch.from_numpy(make_config(a.config)).cuda()
n, l = x.shape
fl = torch.empty(n, dtype=torch.uint8, device="cuda")
s = stream_handle()
if a.split:
    con = _lib.Contraction("split", None, n, l, device=x.device)
    for _ in range(a.reps):
        con.normalize_split(x, l, fl, 0, n, s)
else:
    ldu, rows = int(L.pcc_ldu(l)), int(L.pcc_rows_padded(n))
    u = torch.empty((rows, ldu), dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(u), ldu, ptr(fl), l, 0, n, s))
torch.cuda.synchronize()
print("ok", a.config, n, l)
