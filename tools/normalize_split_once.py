"""One fused normalise-to-digit-planes launch (pcc_normalize_split_rows_f64)
on a BASELINE config, for ncu captures:  python tools/normalize_split_once.py --config c2"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200.workloads import make_config

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
a = p.parse_args()
x = torch.from_numpy(make_config(a.config)).cuda()
n, l = x.shape
flags = torch.empty(n, dtype=torch.uint8, device="cuda")
con = _lib.Contraction("split", None, n, l, device=x.device)
for _ in range(2):
    con.normalize_split(x, l, flags, 0, n, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
