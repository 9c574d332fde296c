"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists and numba is
installed):

    python tests/golden/make_golden.py

It imports the reference package ``paircorr`` read-only from
/root/reference/pkg/src (bytecode writing disabled, numba cache redirected
to /tmp so nothing is written next to the reference sources), runs its own
public functions on seeded inputs, and writes:

* ``small_cases.npz``   -- per case: x, u, zero-variance flags from
  ``normalize`` (transform.py:99), the packed result of ``allpairs``
  (engine.py:23) at t=4, ``allpairs_naive`` (transform.py:163), and the flat
  ``compute_pass`` buffer at t=3 (tiles.py:133).  Cases mirror the
  reference's own tests (KATs, planted rows, reduction-order lengths,
  zero-variance traps, GPU-tile-ragged shapes).
* ``bijection.npz``     -- ``sym_job_coords`` (indexing.py:128) on random ids
  at large n and ``_kernels.tile_row`` (:301) samples.
* ``partition.json``    -- ``partition(T, p)`` (distributed.py:76).
* ``config_digests.json`` -- for the two configs the reference runs in
  seconds (c1, c3): sha256 of ``allpairs(...).packed`` and of ``normalize(...).u``,
  the zero-variance set and 4096 sampled packed values.

Nothing under tests/ or the product reads /root/reference at run time; only
these committed outputs travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/paircorr_numba_cache")
sys.dont_write_bytecode = True
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import numpy as np  # noqa: E402

import paircorr as pc  # noqa: E402
from paircorr import _kernels  # noqa: E402
from paircorr.indexing import sym_job_coords  # noqa: E402

from paper_1605_01584_b200.workloads import make_config  # noqa: E402


def random_dataset(rng, n, l, special_rows=False):
    """Same recipe as the reference's tests/conftest.py:16-23."""
    values = rng.random((n, l))
    if special_rows and n >= 4:
        values[1] = 3.25
        values[2] = -values[0]
        values[3] = 2.5 * values[0] + 1.0
    return values


def small_cases() -> dict[str, np.ndarray]:
    cases: dict[str, np.ndarray] = {}
    cases["kat_124_135"] = np.array([[1.0, 2.0, 4.0], [1.0, 3.0, 5.0]])
    cases["norm_123"] = np.array([[1.0, 2.0, 3.0]])
    cases["const_then_123"] = np.array([[5.0, 5.0, 5.0], [1.0, 2.0, 3.0]])
    cases["two_samples"] = np.array([[3.0, 9.0]])
    cases["self_reverse"] = np.array([[1.0, 2.0, 3.0], [3.0, 2.0, 1.0]])
    cases["twin"] = np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0]])
    cases["constant_2"] = np.array([[4.0, 4.0]])
    v = np.array([1.46030999e-106, 0.0])
    cases["tiny_magnitude"] = np.stack([v, -v, np.array([0.0, 1.0])])
    # variation only at ~1e-170: squared deviations underflow to 0.0, ssd == 0.0
    # although the row is not constant -> flagged by the ssd guard (_kernels.py:244-247).
    cases["ssd_underflow"] = np.array([[1e-170, 2e-170, 3e-170, 1e-170], [1.0, 2.0, 3.0, 5.0]])
    # variation at ~1e-160: squares are subnormal (not zero) -- the precision-loss
    # regime the reference documents (transform.py:23-26); engine != naive there.
    cases["ssd_subnormal"] = np.array([[1e-160, 2e-160, 3e-160, 1e-160], [1.0, 2.0, 3.0, 5.0]])
    rng = np.random.default_rng(20260810)  # reference conftest seed
    cases["conftest_8x11_special"] = random_dataset(rng, 8, 11, special_rows=True)
    cases["conftest_37x19_special"] = random_dataset(rng, 37, 19, special_rows=True)
    cases["conftest_65x8_special"] = random_dataset(rng, 65, 8, special_rows=True)
    cases["one_row"] = random_dataset(rng, 1, 2)
    for l in [1, 2, 3, 7, 8, 9, 15, 16, 17, 63, 64, 65, 100, 513]:
        if l < 2:
            continue  # Dataset requires l >= 2 (transform.py:66-67)
        r = np.random.default_rng(l)
        scale = 10.0 ** float(r.integers(-3, 4))
        cases[f"lanes_l{l}"] = np.stack([r.standard_normal(l) * scale, r.standard_normal(l),
                                         r.standard_normal(l) * 1e3 + 7.0])
    # log-normal constant rows whose float ssd is NOT zero (the exact-constant trap)
    r = np.random.default_rng(1531)
    x = r.lognormal(2.0, 1.0, (12, 1531))
    x[[0, 5, 11]] = r.lognormal(2.0, 1.0, 3)[:, None]
    cases["lognormal_const_12x1531"] = x
    # GPU-tile-ragged shapes: n crosses the 128-row tile edge, l not a multiple of 8/32
    r = np.random.default_rng(130)
    x = r.standard_normal((130, 37))
    x[127] = 2.0
    x[128] = -x[3]
    cases["ragged_130x37"] = x
    r = np.random.default_rng(257)
    cases["ragged_257x9"] = r.random((257, 9))
    return cases


def extras() -> None:
    """Reference-API helpers outside the engine path: gen_synthetic
    (fileio.py:295-305) values and pcc_naive / pcc_normalized
    (transform.py:134-160) on a few vector pairs, as exact hex floats."""
    gens = {}
    for n, l, seed in [(3, 5, 7), (1, 9, 0), (4, 3, 2**63 + 11)]:
        gens[f"{n},{l},{seed}"] = [float(v).hex() for v in pc.gen_synthetic(n, l, seed=seed).values.ravel()]
    rng = np.random.default_rng(99)
    pairs = []
    vecs = [(np.array([1.0, 2.0, 4.0]), np.array([1.0, 3.0, 5.0])),
            (np.array([3.0, 3.0, 3.0, 3.0]), np.array([1.0, 2.0, 3.0, 4.0])),
            (np.array([1e-160, 2e-160, 4e-160]), np.array([5.0, -1.0, 2.0])),
            (rng.standard_normal(1001), rng.standard_normal(1001)),
            (rng.lognormal(2.0, 1.0, 77), rng.lognormal(2.0, 1.0, 77))]
    for a, b in vecs:
        ua = pc.normalize(pc.Dataset(values=np.stack([a, b])), threads=1).u
        pairs.append({"a": [float(v).hex() for v in a], "b": [float(v).hex() for v in b],
                      "naive": float(pc.pcc_naive(a, b)).hex(),
                      "normalized": float(pc.pcc_normalized(ua[0], ua[1])).hex()})
    # file formats byte for byte (fileio.py:58-63 LPCC, :155-274 LPCR)
    import tempfile

    xs = np.array([[1.0, 2.0, 4.0, 8.0], [3.0, 3.0, 3.0, 3.0], [0.5, -1.5, 2.25, 7.0]])
    d = pc.Dataset(values=xs)
    res = pc.allpairs(d, threads=1)
    with tempfile.TemporaryDirectory() as td:
        pc.save_dataset(f"{td}/d.lpcc", d)
        pc.save_result(f"{td}/r.lpcr", res)
        files = {"x": xs.tolist(), "lpcc_hex": open(f"{td}/d.lpcc", "rb").read().hex(),
                 "lpcr_hex": open(f"{td}/r.lpcr", "rb").read().hex()}
    (HERE / "helpers.json").write_text(json.dumps({"gen_synthetic": gens, "pairs": pairs, "files": files},
                                                  indent=1))


def main() -> None:
    if "--extras" in sys.argv:
        extras()
        print("helper fixtures written to", HERE)
        return
    extras()
    out = {}
    for name, x in small_cases().items():
        d = pc.Dataset(values=x)
        nd = pc.normalize(d, threads=1)
        flags = np.zeros(d.n, dtype=bool)
        flags[list(nd.zero_variance)] = True
        res = pc.allpairs(d, tile_size=4, threads=1)
        naive = pc.allpairs_naive(d)
        geom = pc.TileGeometry(n=d.n, t=3)
        blocks = pc.compute_pass(nd, geom, 0, geom.total_tiles)
        flat = np.concatenate([b.values for b in blocks]) if blocks else np.empty(0)
        out[f"{name}/x"] = d.values
        out[f"{name}/u"] = nd.u
        out[f"{name}/zv"] = flags
        out[f"{name}/packed"] = res.packed
        out[f"{name}/naive"] = naive.packed
        out[f"{name}/pass_t3"] = flat
    np.savez_compressed(HERE / "small_cases.npz", **out)

    # bijection samples (indexing.py:128-171, _kernels.py:301-319)
    rng = np.random.default_rng(1)
    bij = {}
    for n in (10**4, 10**5, 10**6, 2**31 + 7, 2**32 - 1):
        total = n * (n + 1) // 2
        ids = rng.integers(0, total, size=2000, dtype=np.uint64)
        # row boundaries are where the float estimate is most fragile
        ys = rng.integers(0, n, size=500, dtype=np.uint64)
        pref = ys * (np.uint64(2 * n + 1) - ys) // np.uint64(2)
        edge = np.concatenate([pref, np.maximum(pref, np.uint64(1)) - np.uint64(1),
                               np.array([0, total - 1], dtype=np.uint64)])
        ids = np.concatenate([ids, edge])
        y, x = sym_job_coords(n, ids)
        bij[f"n{n}/ids"] = ids
        bij[f"n{n}/y"] = y
        bij[f"n{n}/x"] = x
    tr = []
    for m in (1, 2, 3, 16, 79, 128, 256, 512, 4097, 65536, 2**20 + 3):
        total = m * (m + 1) // 2
        for j in set(rng.integers(0, total, size=64).tolist() + [0, total - 1]):
            tr.append((m, int(j), int(_kernels.tile_row(m, int(j)))))
    bij["tile_row"] = np.array(tr, dtype=np.int64)
    np.savez_compressed(HERE / "bijection.npz", **bij)

    parts = {f"{T},{p}": pc.partition(T, p) for T in range(0, 41) for p in range(1, 10)}
    for T, p in [(136, 8), (3160, 8), (8256, 8), (32896, 8), (131328, 8), (10, 4), (3, 4)]:
        parts[f"{T},{p}"] = pc.partition(T, p)
    (HERE / "partition.json").write_text(json.dumps(parts, sort_keys=True))

    # wire-protocol frames, byte for byte (protocol.py:54-147)
    from paircorr import protocol as rp

    vals = np.arange(2 * 16, dtype=np.float64) / 7.0
    frames = {
        "assign": rp.encode_assign(3, 17, 4, 1000, "/data/expr.lpcc").hex(),
        "assign_unicode": rp.encode_assign(0, 0, 1, 1, "d\u00e9j\u00e0.lpcc").hex(),
        "blocks": rp.encode_blocks(12, vals, 4).hex(),
        "done": rp.encode_done(123456789).hex(),
        "error": rp.encode_error("ValueError: boom").hex(),
        "blocks_values": vals.tolist(),
    }
    (HERE / "protocol_frames.json").write_text(json.dumps(frames, indent=1))

    digests = {}
    threads = len(os.sched_getaffinity(0))
    for name in ("c1", "c3"):
        x = make_config(name)
        d = pc.Dataset(values=x)
        nd = pc.normalize(d, threads=threads)
        res = pc.allpairs(d, threads=threads)
        s = np.random.default_rng(7).integers(0, res.packed.size, size=4096)
        digests[name] = {
            "n": d.n,
            "l": d.l,
            "x_sha256": hashlib.sha256(d.values.tobytes()).hexdigest(),
            "u_sha256": hashlib.sha256(nd.u.tobytes()).hexdigest(),
            "packed_sha256": hashlib.sha256(res.packed.tobytes()).hexdigest(),
            "zero_variance": sorted(res.zero_variance),
            "sample_idx": s.tolist(),
            "sample_val_hex": [float(v).hex() for v in res.packed[s]],
        }
    (HERE / "config_digests.json").write_text(json.dumps(digests, indent=1))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
