"""Host-side logic of the drop-in (no GPU): bijection, geometry, partition,
pass planning, shard ownership, host scatter, result/file containers and
the loud-failure contract."""

import json
import math

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200.distributed import owned_runs, partition, shard_span
from paper_1605_01584_b200.stream import plan_stream
from paper_1605_01584_b200.tiles import _scatter_host

from conftest import GOLDEN, random_values, triangle_walk


# --- bijection (indexing.py) ------------------------------------------------

def test_row_prefix_and_examples():
    assert pc.row_prefix(4, 0) == 0 and pc.row_prefix(4, 4) == 10 and pc.row_prefix(4, 2) == 7
    assert pc.sym_job_id(4, 0, 0) == 0 and pc.sym_job_id(4, 1, 2) == 5 and pc.sym_job_id(4, 3, 3) == 9
    assert pc.sym_job_coord(4, 5) == pc.Coord(1, 2)
    assert pc.nonsym_job_id(4, 1, 2) == 6 and pc.nonsym_job_coord(4, 15) == pc.Coord(3, 3)
    for bad in [(4, -1), (4, 5), (0, 0)]:
        with pytest.raises(ValueError):
            pc.row_prefix(*bad)
    with pytest.raises(ValueError):
        pc.sym_job_id(4, 2, 1)
    with pytest.raises(ValueError):
        pc.sym_job_coord(4, 10)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 16, 33, 64])
def test_bijection_exhaustive(n):
    walk = triangle_walk(n)
    for j, (y, x) in enumerate(walk):
        assert pc.sym_job_id(n, y, x) == j
        assert tuple(pc.sym_job_coord(n, j)) == (y, x)
    ys, xs = pc.sym_job_coords(n, np.arange(len(walk), dtype=np.uint64))
    assert [(int(a), int(b)) for a, b in zip(ys, xs)] == walk
    assert np.array_equal(pc.sym_job_ids(n, ys, xs), np.arange(len(walk), dtype=np.uint64))


def test_bijection_matches_reference_golden_at_scale():
    z = np.load(GOLDEN / "bijection.npz")
    for n in (10**4, 10**5, 10**6, 2**31 + 7, 2**32 - 1):
        ids, y, x = z[f"n{n}/ids"], z[f"n{n}/y"], z[f"n{n}/x"]
        gy, gx = pc.sym_job_coords(n, ids)
        assert np.array_equal(gy, y) and np.array_equal(gx, x)
        for j, yy, xx in list(zip(ids, y, x))[:200]:
            assert tuple(pc.sym_job_coord(n, int(j))) == (int(yy), int(xx))
    for m, j, y in z["tile_row"]:
        assert pc.sym_job_coord(int(m), int(j)).y == int(y)


def _row_bisect(n, j):
    lo, hi = 0, n - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if pc.row_prefix(n, mid) <= j:
            lo = mid
        else:
            hi = mid - 1
    return lo


@given(st.integers(1, 2**20), st.data())
@settings(max_examples=300, deadline=None)
def test_bijection_roundtrip_property(n, data):
    j = data.draw(st.integers(0, n * (n + 1) // 2 - 1))
    y, x = pc.sym_job_coord(n, j)
    assert y == _row_bisect(n, j) and y <= x < n
    assert pc.sym_job_id(n, y, x) == j


def test_max_n_boundaries():
    n = pc.MAX_N
    total = pc.sym_job_count(n)
    assert total == n * (n + 1) // 2 < 2**64
    assert pc.sym_job_coord(n, total - 1) == pc.Coord(n - 1, n - 1)
    assert pc.sym_job_coord(n, 0) == pc.Coord(0, 0)
    with pytest.raises(ValueError):
        pc.sym_job_count(n + 1)


# --- geometry, partition, passes ---------------------------------------------

@pytest.mark.parametrize("n,t,m", [(1, 1, 1), (2, 2, 1), (3, 2, 2), (4, 2, 2), (5, 2, 3), (128, 4, 32), (10, 3, 4)])
def test_geometry(n, t, m):
    g = pc.TileGeometry(n=n, t=t)
    assert g.m == m and g.total_tiles == m * (m + 1) // 2 and g.job_count == n * (n + 1) // 2
    with pytest.raises(ValueError):
        pc.TileGeometry(n=0, t=2)
    with pytest.raises(ValueError):
        pc.TileGeometry(n=4, t=0)


def test_partition_matches_reference_golden():
    ref = json.loads((GOLDEN / "partition.json").read_text())
    for key, ranges in ref.items():
        T, p = map(int, key.split(","))
        assert [list(r) for r in partition(T, p)] == ranges
    with pytest.raises(ValueError):
        partition(5, 0)
    with pytest.raises(ValueError):
        partition(-1, 2)


def test_plan_passes():
    plan = pc.plan_passes(3, 20, 5)
    assert plan.passes == ((3, 8), (8, 13), (13, 18), (18, 20)) and plan.total == 17
    assert pc.plan_passes(4, 4, 3).passes == ()
    with pytest.raises(ValueError):
        pc.plan_passes(0, 5, 0)
    with pytest.raises(ValueError):
        pc.plan_passes(5, 4, 1)


@pytest.mark.parametrize("n", [1, 127, 128, 129, 2000, 10007, 16384, 65536])
@pytest.mark.parametrize("chunk_rows", [1, 3, 8, 64])
@pytest.mark.parametrize("p", [1, 3])
@pytest.mark.parametrize("lead", [None, 0.0, 0.5, 1.0])
def test_stream_plan_covers_range_and_respects_dependencies(n, chunk_rows, p, lead):
    """Streamed passes (stream.plan_stream) tile each partition range exactly
    once, never run before the chunk holding their first tile row is
    normalised, and every row they declare final has all its range tiles done."""
    mg = -(-n // 128)
    T = mg * (mg + 1) // 2
    F = lambda y: (y * (2 * mg + 1 - y)) // 2  # noqa: E731
    for tb, te in partition(T, p):
        sp = plan_stream(n, tb, te, 148, chunk_rows, lead=lead)
        if te == tb:
            assert sp.passes == ()
            continue
        cov = sorted((q[0], q[1]) for q in sp.passes)
        assert cov[0][0] == tb and cov[-1][1] == te
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(cov, cov[1:]))
        assert sp.chunks[0][1] == n and sp.chunks[-1][0] == sp.row_lo
        assert all(c[0] < c[1] for c in sp.chunks)
        done = np.zeros(T, dtype=bool)
        for lo, hi, need, dl_lo, dl_hi, phase in sp.passes:
            assert phase in (1, 2)
            y = pc.sym_job_coord(mg, lo).y
            assert sp.chunks[need - 1][0] <= y * 128  # the pass's rows are normalised first
            done[lo:hi] = True
            for r in range(dl_lo, dl_hi, 128):
                Y = r // 128
                a, b = max(tb, F(Y)), min(te, F(Y + 1))
                assert done[a:b].all(), (lo, hi, dl_lo, dl_hi, Y)


@pytest.mark.parametrize("n", [1, 5, 128, 129, 300, 1000])
@pytest.mark.parametrize("p", [1, 2, 3, 7])
def test_owned_runs_partition_the_packed_triangle(n, p):
    mg = -(-n // 128)
    T = mg * (mg + 1) // 2
    total = n * (n + 1) // 2
    cover = np.zeros(total, dtype=np.int32)
    for lo_t, hi_t in partition(T, p):
        span = shard_span(n, lo_t, hi_t)
        for lo, hi in owned_runs(n, lo_t, hi_t):
            assert span[0] <= lo < hi <= span[1]
            cover[lo:hi] += 1
    assert (cover == 1).all()


def test_owned_runs_equal_cell_enumeration():
    n = 300  # 3 GPU tile rows, 6 tiles
    mg = 3
    for tb in range(6):
        for te in range(tb + 1, 7):
            expect = set()
            for J in range(tb, te):
                Y, X = pc.sym_job_coord(mg, J)
                for y in range(Y * 128, min(n, Y * 128 + 128)):
                    for x in range(max(y, X * 128), min(n, X * 128 + 128)):
                        expect.add(pc.sym_job_id(n, y, x))
            got = set()
            for lo, hi in owned_runs(n, tb, te):
                got.update(range(lo, hi))
            assert got == expect, (tb, te)


# --- results, scatter, containers -------------------------------------------

def test_host_scatter_matches_oracle(rng):
    x = random_values(rng, 23, 7, special_rows=True)
    u, _ = oracle.normalize(x)
    for t in (1, 2, 3, 4, 8):
        g = pc.TileGeometry(n=23, t=t)
        flat = oracle.compute_pass(u, t, 0, g.total_tiles)
        ref = np.full(g.job_count, np.nan)
        oracle.scatter_range(ref, flat, 0, g.total_tiles, g.m, t, 23)
        got = np.full(g.job_count, np.nan)
        _scatter_host(got, flat, 0, g.total_tiles, g)
        assert np.array_equal(got, ref, equal_nan=True)
        # pass-by-pass through the public scatter_pass, with per-block fallback
        res = pc.empty_result(23)
        cut = g.total_tiles // 2
        blocks = pc.BlockList(pc.TileBlock(j, flat[j * t * t:(j + 1) * t * t]) for j in range(cut))
        pc.scatter(blocks, g, res)
        b2 = pc.BlockList(pc.TileBlock(j, flat[j * t * t:(j + 1) * t * t]) for j in range(cut, g.total_tiles))
        b2.flat = flat[cut * t * t:]
        pc.scatter_pass(b2, g, res)
        assert np.array_equal(res.packed, ref)


def test_scatter_errors():
    g = pc.TileGeometry(n=4, t=2)
    res = pc.empty_result(4)
    blk = pc.TileBlock(0, np.zeros(4))
    with pytest.raises(pc.IntegrityError):
        pc.scatter([blk, pc.TileBlock(0, np.zeros(4))], g, res)
    with pytest.raises(ValueError):
        pc.scatter([pc.TileBlock(3, np.zeros(4))], g, res)
    with pytest.raises(ValueError):
        pc.scatter([pc.TileBlock(0, np.zeros(3))], g, res)


def test_correlation_result_get_and_dense():
    packed = np.arange(10, dtype=np.float64)
    r = pc.CorrelationResult(n=4, packed=packed)
    assert r.get(1, 2) == r.get(2, 1) == 5.0
    d = r.to_dense()
    assert np.array_equal(d, d.T) and d[3, 3] == 9.0
    with pytest.raises(ValueError):
        r.get(0, 4)
    with pytest.raises(ValueError):
        r.get(-1, 0)


def test_dataset_validation():
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.array([[np.nan, 1.0]]))
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.array([[np.inf, 1.0], [0.0, 2.0]]))
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.array([[1.0]]))
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.zeros((0, 5)))
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.zeros((2, 3)), ids=["only-one"])
    with pytest.raises(pc.DataError):
        pc.Dataset(values=np.zeros(3))
    with pytest.raises(pc.DataError):
        pc.Dataset(values=torch.tensor([[1.0, float("nan")]]))
    d = pc.Dataset(values=[[1, 2, 3]])
    assert d.values.dtype == np.float64 and d.n == 1 and d.l == 3


def test_estimate_cost():
    assert pc.estimate_cost(1, 1) == 6 and pc.estimate_cost(2, 10) == 130
    for n, l in [(10**6, 999_983), (12345, 678)]:
        assert pc.estimate_cost(n, l) == (10 * l * n + l * n * (n + 1)) // 2
    with pytest.raises(ValueError):
        pc.estimate_cost(0, 5)


def test_file_roundtrip(tmp_path, rng):
    x = random_values(rng, 9, 5)
    pc.save_dataset(tmp_path / "d.lpcc", pc.Dataset(values=x))
    assert np.array_equal(pc.load_dataset(tmp_path / "d.lpcc").values, x)
    packed, zv = oracle.allpairs(x)
    r = pc.CorrelationResult(n=9, packed=packed, zero_variance=frozenset({2, 5}))
    pc.save_result(tmp_path / "r.lpcr", r)
    back = pc.load_result(tmp_path / "r.lpcr")
    assert np.array_equal(back.packed, packed) and back.zero_variance == {2, 5}
    for i, j in [(0, 0), (3, 7), (8, 1)]:
        assert pc.query_pair(tmp_path / "r.lpcr", i, j) == r.get(i, j)
    (tmp_path / "bad.lpcc").write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(pc.DataError):
        pc.load_dataset(tmp_path / "bad.lpcc")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    d = pc.Dataset(values=np.array([[1.0, 2.0, 3.0], [3.0, 1.0, 2.0]]))
    with pytest.raises(pc.DeviceError):
        pc.allpairs(d)
    with pytest.raises(pc.DeviceError):
        pc.normalize(d)


def test_workloads_shapes_and_determinism():
    from paper_1605_01584_b200.workloads import gen_uniform_splitmix64, make_config

    a = make_config("c3", n=500, l=40)
    b = make_config("c3", n=500, l=40)
    assert np.array_equal(a, b) and a.shape == (500, 40)
    const = [i for i in range(500) if (a[i] == a[i, 0]).all()]
    assert len(const) == 5
    c5 = make_config("c5", n=1024, l=64)
    assert c5.shape == (1024, 64)
    # splitmix64 known answers: element k = mix(seed + (k+1) * golden) >> 11 * 2^-53
    def mix(v):
        v &= 2**64 - 1
        v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9 % 2**64
        v = (v ^ (v >> 27)) * 0x94D049BB133111EB % 2**64
        v = v ^ (v >> 31)
        return (v >> 11) * 2.0**-53
    assert gen_uniform_splitmix64(1, 2, seed=0)[0].tolist() == [mix(0x9E3779B97F4A7C15), mix(2 * 0x9E3779B97F4A7C15)]
    assert np.array_equal(gen_uniform_splitmix64(2, 6, seed=9).ravel(), gen_uniform_splitmix64(1, 12, seed=9).ravel())
    u = gen_uniform_splitmix64(3, 4, seed=0)
    assert u.shape == (3, 4) and (0 <= u).all() and (u < 1).all()
    assert math.isclose(float(gen_uniform_splitmix64(1, 1, seed=0)[0, 0]),
                        float(gen_uniform_splitmix64(2, 2, seed=0)[0, 0]))


def test_packed_file_writer_sink_streams_passes(tmp_path, rng):
    """The reference's streaming sink (fileio.py:233-274): passes of tile
    blocks, in any split, land at their bijection offsets in the LPCR file."""
    x = random_values(rng, 41, 9, special_rows=True)
    u, zv = oracle.normalize(x)
    ref, _ = oracle.allpairs(x)
    g = pc.TileGeometry(n=41, t=4)
    path = tmp_path / "s.lpcr"
    with pc.PackedFileWriterSink(path, g, frozenset({1})) as sink:
        for lo, hi in pc.plan_passes(0, g.total_tiles, 17).passes:
            flat = oracle.compute_pass(u, 4, lo, hi)
            blocks = pc.BlockList(pc.TileBlock(lo + k, flat[k * 16:(k + 1) * 16]) for k in range(hi - lo))
            blocks.flat = flat
            sink.consume((lo, hi), blocks)
    back = pc.load_result(path)
    assert np.array_equal(back.packed, ref) and back.zero_variance == {1}
    with pc.PackedResultReader(path) as r:
        assert r.query(3, 0) == ref[pc.sym_job_id(41, 0, 3)]
        assert np.array_equal(r.read_all(), ref)


def test_triangle_indexer_value_object():
    ti = pc.TriangleIndexer(5)
    assert ti.sym_count == 15 and ti.nonsym_count == 25
    assert ti.row_prefix(2) == 9 and ti.job_id(1, 3) == 7 and ti.coord(7) == pc.Coord(1, 3)
    assert ti.nonsym_job_id(2, 1) == 11 and ti.nonsym_coord(11) == pc.Coord(2, 1)
    with pytest.raises(ValueError):
        pc.TriangleIndexer(0)


def test_gen_synthetic_bit_identical_to_reference():
    """fileio.gen_synthetic against the reference's own output (tests/golden/helpers.json)."""
    g = json.loads((GOLDEN / "helpers.json").read_text())["gen_synthetic"]
    for key, vals in g.items():
        n, l, seed = (int(v) for v in key.split(","))
        got = pc.gen_synthetic(n, l, seed=seed).values.ravel()
        assert [float(v).hex() for v in got] == vals, key
    with pytest.raises(ValueError):
        pc.gen_synthetic(0, 3)


def test_load_dataset_tsv_like_reference(tmp_path):
    p = tmp_path / "d.tsv"
    p.write_text("geneA 1 2 3\n\ngeneB 4.5 -1 2e3\n")
    d = pc.load_dataset(p)
    assert d.ids == ["geneA", "geneB"] and d.values.tolist() == [[1, 2, 3], [4.5, -1, 2000.0]]
    p.write_text("1 2\n3 4\n")
    assert pc.load_dataset(p, format="tsv").ids is None
    for bad, msg in [("a 1 2\n3 4 5\n", "expected a label"), ("1 2\n3\n", "ragged"), ("1 x\n", "not a number"),
                     ("1 inf\n", "non-finite"), ("\n\n", "empty")]:
        p.write_text(bad)
        with pytest.raises(pc.DataError, match=msg):
            pc.load_dataset(p)
    with pytest.raises(ValueError):
        pc.load_dataset(p, format="csv")
    b = tmp_path / "d.lpcc"
    pc.save_dataset(b, pc.Dataset(values=np.arange(6.0).reshape(2, 3)))
    assert pc.load_dataset(b).values.tolist() == [[0, 1, 2], [3, 4, 5]]


def test_stream_plan_ends_with_half_wave_passes():
    """The top-down phase ends ..., 1 wave, 1/2, 1/2 (the halves run as one
    round of 64 x 64 quadrants each): a short download after the last pass."""
    n = 16384
    mg = n // 128
    T = mg * (mg + 1) // 2
    sp = plan_stream(n, 0, T, 148, 8)
    sizes = [hi - lo for lo, hi, *_ in sp.passes if _[-1] == 2]
    assert sizes[-2:] == [74, 74] and sizes[-3] == 148
    sp = plan_stream(n, 0, T, 148, 8, half_tail=False)
    assert [hi - lo for lo, hi, *_ in sp.passes][-2:] == [148, 148]


def test_file_formats_byte_identical_to_reference(tmp_path):
    """LPCC dataset and LPCR result files written here equal the reference's
    own files byte for byte (tests/golden/helpers.json, made with
    paircorr.save_dataset / save_result); both load back."""
    g = json.loads((GOLDEN / "helpers.json").read_text())["files"]
    x = np.array(g["x"])
    pc.save_dataset(tmp_path / "d.lpcc", pc.Dataset(values=x))
    assert (tmp_path / "d.lpcc").read_bytes().hex() == g["lpcc_hex"]
    packed, zv = oracle.allpairs(x)
    r = pc.CorrelationResult(n=x.shape[0], packed=packed, zero_variance=frozenset(np.flatnonzero(zv).tolist()))
    pc.save_result(tmp_path / "r.lpcr", r)
    assert (tmp_path / "r.lpcr").read_bytes().hex() == g["lpcr_hex"]
    (tmp_path / "ref.lpcr").write_bytes(bytes.fromhex(g["lpcr_hex"]))
    back = pc.load_result(tmp_path / "ref.lpcr")
    assert np.array_equal(back.packed, packed) and back.zero_variance == r.zero_variance


def test_file_corruption_detected(tmp_path):
    x = np.arange(12.0).reshape(3, 4)
    p = tmp_path / "d.lpcc"
    pc.save_dataset(p, pc.Dataset(values=x))
    raw = p.read_bytes()
    for bad in (raw[:-8], raw + b"\0" * 8, raw[:4] + (2).to_bytes(4, "little") + raw[8:], raw[:10]):
        p.write_bytes(bad)
        with pytest.raises(pc.DataError):
            pc.load_dataset(p, format="binary")
    r = tmp_path / "r.lpcr"
    packed, _ = oracle.allpairs(x)
    pc.save_result(r, pc.CorrelationResult(n=3, packed=packed))
    raw = r.read_bytes()
    for bad in (b"NOPE" + raw[4:], raw[:-8], raw[:6]):
        r.write_bytes(bad)
        with pytest.raises(pc.DataError):
            pc.load_result(r)


def test_contraction_method_resolution():
    from paper_1605_01584_b200 import _lib

    assert _lib.resolve_method() == "tensor"
    assert _lib.resolve_method(exact=True) == "exact"
    assert _lib.resolve_method("split") == "split"
    assert _lib.resolve_method("exact", exact=True) == "exact"
    with pytest.raises(ValueError):
        _lib.resolve_method("split", exact=True)
    with pytest.raises(ValueError):
        _lib.resolve_method("bf16")
    _lib.check_method_shape("split", _lib.SPLIT_MAX_L)
    _lib.check_method_shape("tensor", 10 * _lib.SPLIT_MAX_L)
    with pytest.raises(ValueError, match="split"):
        _lib.check_method_shape("split", _lib.SPLIT_MAX_L + 1)


def test_split_bound_rejected_before_any_device_work():
    import paper_1605_01584_b200 as pc
    from paper_1605_01584_b200 import _lib

    x = np.random.default_rng(0).standard_normal((3, _lib.SPLIT_MAX_L + 1))
    with pytest.raises(ValueError, match="split"):
        pc.allpairs(pc.Dataset(values=x), method="split")
    with pytest.raises(ValueError, match="method"):
        pc.allpairs(pc.Dataset(values=x[:, :10]), method="fp32")


def test_allpairs_routes_backend_like_the_reference(monkeypatch, tmp_path):
    """engine.py:46-56: workers > 1 or backend != "in_process" goes to
    run_workers(dataset, geom, workers, backend, capacity, threads); a path
    stays a path so subprocess workers load the file themselves."""
    from paper_1605_01584_b200 import engine

    calls = []
    monkeypatch.setattr(engine, "resolve_devices", lambda devices=None: [torch.device("cuda", 0)])
    monkeypatch.setattr(engine, "run_workers", lambda *a, **k: calls.append((a, k)) or "routed")
    x = np.random.default_rng(0).random((10, 5))
    ds = pc.Dataset(values=x)
    assert engine.allpairs(ds, workers=2, backend="subprocess", capacity=3, threads=2) == "routed"
    a, k = calls[-1]
    assert a[0] is ds and a[1].n == 10 and a[2:] == (2, "subprocess", 3, 2) and k["method"] == "tensor"
    assert engine.allpairs(ds, backend="subprocess") == "routed"
    a, _ = calls[-1]
    assert a[2:4] == (1, "subprocess") and a[4] == engine.default_capacity(4)
    path = tmp_path / "d.lpcc"
    pc.save_dataset(path, ds)
    engine.allpairs(path, workers=3, backend="subprocess")
    assert calls[-1][0][0] == path
    assert engine.allpairs(ds, workers=2) == "routed"  # in-process workers: the CUDA thread backend
    assert calls[-1][1]["backend"] == "cuda"
    with pytest.raises(ValueError, match="subprocess"):
        engine.allpairs(ds, backend="subprocess", output="dense")
    with pytest.raises(ValueError, match="backend"):
        engine.allpairs(ds, backend="mpi")
