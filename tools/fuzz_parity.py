"""Randomised parity sweep on one GPU (a one-off validation run, not a test):
random shapes and value distributions through K1 (U and flags bit for bit
against the CPU oracle, every K1 kernel: staged, chunked, 3-pass) and through
allpairs in the tensor, split and exact modes (within 1e-12 / bit-identical).

    python tools/fuzz_parity.py --seconds 300 --seed 1
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import oracle
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200 import _lib

p = argparse.ArgumentParser()
p.add_argument("--seconds", type=float, default=300.0)
p.add_argument("--seed", type=int, default=1)
a = p.parse_args()
rng = np.random.default_rng(a.seed)
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream


def values(n, l):
    kind = rng.integers(0, 6)
    if kind == 0:
        x = rng.standard_normal((n, l))
    elif kind == 1:
        x = rng.lognormal(2.0, 1.0, (n, l))
    elif kind == 2:  # small integers summing to 0 with -0.0 entries (mean +0, x - mean = -0)
        x = rng.integers(-9, 10, (n, l)).astype(np.float64)
        x[:, rng.integers(0, l, size=min(l, 3))] = -0.0
        x[:, -1] -= x.sum(axis=1)
    elif kind == 3:  # magnitudes spread over many binades
        x = rng.standard_normal((n, l)) * np.exp2(rng.integers(-300, 300, (n, 1)))
    elif kind == 4:  # near-constant rows: tiny spread around a large offset
        x = 1e6 + rng.standard_normal((n, l)) * 1e-9
    else:
        x = rng.random((n, l))
    for r in rng.choice(n, size=min(n, 1 + n // 50), replace=False):  # planted constant rows
        x[r] = x[r, 0]
    return kind, np.ascontiguousarray(x)


t_end = time.time() + a.seconds
cases = fails = 0
while time.time() < t_end:
    big = rng.random() < 0.3
    n = int(rng.integers(1, 64 if big else 1500))
    l = int(rng.choice([rng.integers(2, 300), rng.integers(300, 8192), rng.integers(8192, 20000)] if big else
                       [rng.integers(2, 300), rng.integers(300, 4000)]))
    kind, x = values(n, l)
    cases += 1
    # K1 through the C ABI
    ldu = int(L.pcc_ldu(l))
    xd = torch.from_numpy(x).cuda()
    u = torch.full((n, ldu), float("nan"), dtype=torch.float64, device="cuda")
    zv = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
    _lib.check(L.pcc_normalize_rows_f64(xd.data_ptr(), l, u.data_ptr(), ldu, zv.data_ptr(), l, 0, n, s))
    torch.cuda.synchronize()
    u_ref, zv_ref = oracle.normalize(x)
    got = u.cpu().numpy()
    ok = np.array_equal(got[:, :l].view(np.uint64), u_ref.view(np.uint64)) and \
        np.array_equal(zv.cpu().numpy().astype(bool), zv_ref) and (got[:, l:] == 0.0).all()
    msg = f"K1 n={n} l={l} kind={kind}"
    if ok and n * n * l <= 3e9:
        ref, zref = oracle.allpairs(x, t=4)
        zs = frozenset(np.flatnonzero(zref).tolist())
        for method, tol in (("tensor", 1e-12), ("split", 1e-12), ("exact", 0.0)):
            if method == "split" and l > 8192:
                continue
            kw = {"exact": True} if method == "exact" else {"method": method}
            res = pc.allpairs(pc.Dataset(values=x), **kw)
            dev = float(np.abs(res.packed - ref).max(initial=0.0))
            if not (dev <= tol and res.zero_variance == zs):
                ok = False
                msg += f" {method} dev={dev:.3e} zv_equal={res.zero_variance == zs}"
    if not ok:
        fails += 1
        print("FAIL", msg, flush=True)
    del xd, u, zv
print(f"{cases} cases, {fails} failures", flush=True)
