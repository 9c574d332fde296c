"""GPU parity of split mode (``method="split"``): the contraction on the int8
tensor cores (tcgen05.mma kind::i8) over exact radix-128 digit planes of the
normalised rows, against the CPU oracle and the reference's golden outputs.

Tolerance: every coefficient within 1e-12 absolute of the reference's
(the north star's bound; DESIGN.md §3 K2s derives the worst case 9e-13 for
l <= 8192); zero-variance rows/columns exactly 0.0; the same zero-variance
set.  Like the FP64 tensor path, each cell's arithmetic is a pure function
of the kernel (no split-K), so results are bitwise identical across tile
ranges, passes, workers, layouts and the streamed plan.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200.workloads import make_config

from conftest import random_values

pytestmark = pytest.mark.gpu

TOL = 1e-12
SPLIT = dict(method="split")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _normalized(x):
    L = _lib.lib()
    n, l = x.shape
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    rows, ldu = int(L.pcc_rows_padded(n)), int(L.pcc_ldu(l))
    u = torch.full((rows, ldu), float("nan"), dtype=torch.float64, device="cuda")
    zv = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.pcc_normalize_rows_f64(xd.data_ptr(), l, u.data_ptr(), ldu, zv.data_ptr(), l, 0, n, s))
    _lib.check(L.pcc_zero_rows_f64(u.data_ptr(), ldu, n, rows, s))
    return u


def _split_packed(u, n, l, tile_ranges=None):
    """Digit planes + the split contraction straight through the C ABI."""
    L = _lib.lib()
    con = _lib.Contraction("split", u, n, l).prepare_all(torch.cuda.current_stream().cuda_stream)
    T = int(L.pcc_gpu_tile_count(n))
    out = torch.full((n * (n + 1) // 2,), float("nan"), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for tb, te in tile_ranges or [(0, T)]:
        con.syrk(tb, te, _lib.LAYOUT_PACKED, out.data_ptr(), 0, 0, 0, 0, 0, s)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _assert_parity(got, ref, zv_set, n):
    assert got.shape == ref.shape
    assert not np.isnan(got).any(), "unwritten cells"
    dev = np.abs(got - ref)
    assert float(dev.max(initial=0.0)) <= TOL, f"max dev {dev.max():.3e}"
    for i in zv_set:
        for j in range(n):
            lo, hi = min(i, j), max(i, j)
            assert got[(lo * (2 * n + 1 - lo)) // 2 + hi - lo] == 0.0


def test_digit_planes_are_an_exact_expansion(rng):
    """pcc_split_rows_f64: digit ranges ([-127, 127] leading, [-64, 64] after),
    power-of-two scales, and sum_i d_i 128^-(i-1) * scale within max|u|
    2^-49 of every element; pad rows and K padding are all-zero digits."""
    L = _lib.lib()
    x = random_values(rng, 300, 77, special_rows=True)
    x[6, :] = 0.0
    x[6, 3] = 1.0  # one spike: max|u| close to 1
    n, l = x.shape
    u = _normalized(x)
    con = _lib.Contraction("split", u, n, l).prepare_all(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    rows = u.shape[0]
    W = _lib.SPLIT_ROW_BYTES
    kb = -(-l // W)
    d = con.slices.cpu().numpy().view(np.int8).reshape(kb, 7, rows, W)
    d = d.transpose(2, 0, 3, 1).reshape(rows, kb * W, 7).astype(np.float64)  # [row][k][digit]
    assert np.abs(d[:, :, 0]).max() <= 127 and np.abs(d[:, :, 1:]).max() <= 64
    scale = con.scale.cpu().numpy()
    zero_rows = ~np.any(d != 0, axis=(1, 2))
    assert zero_rows[n:].all() and (scale[zero_rows] == 0.0).all(), "all-zero rows have scale 0"
    m, e = np.frexp(scale[~zero_rows])
    assert (m == 0.5).all(), "scales are powers of two"
    w = 128.0 ** -np.arange(7)
    recon = (d @ w) * scale[:, None]
    uh = u.cpu().numpy()
    assert (recon[:, l:] == 0.0).all() and (recon[n:] == 0.0).all()
    umax = np.abs(uh[:n, :l]).max(axis=1)
    err = np.abs(recon[:n, :l] - uh[:n, :l]).max(axis=1)
    assert (err <= umax * 2.0 ** -49 * 1.01).all()  # 2^e <= 2 max|u| (x 128/127.5)


def test_split_allpairs_vs_reference_golden(golden_small):
    for name, case in golden_small.items():
        x = case["x"]
        res = pc.allpairs(pc.Dataset(values=x), **SPLIT)
        zv = frozenset(np.flatnonzero(case["zv"]).tolist())
        assert res.zero_variance == zv, name
        _assert_parity(res.packed, case["packed"], zv, x.shape[0])


def test_split_compute_pass_layout_vs_reference_golden(golden_small):
    for name, case in golden_small.items():
        x = case["x"]
        nd = pc.normalize(pc.Dataset(values=x))
        geom = pc.TileGeometry(n=x.shape[0], t=3)
        flat = pc.compute_pass(nd, geom, 0, geom.total_tiles, **SPLIT).flat
        ref = case["pass_t3"]
        assert flat.shape == ref.shape, name
        assert np.abs(flat - ref).max(initial=0.0) <= TOL, name
        assert (flat[ref == 0.0] == 0.0).all(), name


@pytest.mark.parametrize(
    "n,l",
    [(1, 2), (2, 2), (3, 7), (8, 8), (127, 16), (128, 17), (129, 33), (255, 15), (256, 31), (257, 64),
     (300, 95), (130, 8192)],
)
def test_split_edge_shapes_vs_oracle(rng, n, l):
    x = random_values(rng, n, l, special_rows=True)
    res = pc.allpairs(pc.Dataset(values=x), **SPLIT)
    ref, zv = oracle.allpairs(x, t=4)
    zs = frozenset(np.flatnonzero(zv).tolist())
    assert res.zero_variance == zs
    _assert_parity(res.packed, ref, zs, n)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_split_config_full_vs_oracle(name):
    """c1 whole; c3 (10,007 x 1,531 log-normal, 1 % constant rows) takes the
    streamed plan (digit planes made chunk by chunk)."""
    x = make_config(name)
    n = x.shape[0]
    res = pc.allpairs(pc.Dataset(values=x), **SPLIT)
    ref, zv = oracle.allpairs(x, t=4)
    zs = frozenset(np.flatnonzero(zv).tolist())
    assert res.zero_variance == zs
    dev = np.abs(res.packed - ref)
    assert float(dev.max()) <= TOL, f"{name}: max dev {dev.max():.3e}"
    zl = np.array(sorted(zs), dtype=np.int64)
    for i in zl[:10]:
        assert res.get(int(i), int(i)) == 0.0
    # streamed plan == one direct launch, bit for bit
    u = _normalized(x)
    assert np.array_equal(_split_packed(u, n, x.shape[1]), res.packed)


def test_split_adversarial_spiky_rows_at_max_l():
    """The error bound's worst shape: l = 8,192 (the split limit) and rows
    whose maximum is close to 1 (one spike) so that every small element's
    digits run the full [-64, 64] range -- still within 1e-12."""
    r = np.random.default_rng(3)
    n, l = 200, 8192
    x = r.standard_normal((n, l)) * 1e-3
    x[np.arange(n), r.integers(0, l, n)] += 30.0
    x[::7, 17] += 30.0  # shared spikes: large coefficients
    ref, _ = oracle.allpairs(x, t=4)
    got = pc.allpairs(pc.Dataset(values=x), **SPLIT).packed
    assert float(np.abs(got - ref).max()) <= TOL


def test_split_l_bound_is_enforced(rng):
    x = rng.standard_normal((4, _lib.SPLIT_MAX_L + 1))
    with pytest.raises(ValueError, match="split"):
        pc.allpairs(pc.Dataset(values=x), **SPLIT)
    u = _normalized(x)
    L = _lib.lib()
    rc = L.pcc_syrk_split_f64(u.data_ptr(), u.data_ptr(), 4, _lib.SPLIT_MAX_L + 1, 0, 1, _lib.LAYOUT_PACKED,
                              u.data_ptr(), 0, 0, 0, 0, 0, None)
    assert rc == 1 and b"split" in L.pcc_last_error()


def test_split_schedule_invariance_bitwise(rng):
    x = random_values(rng, 700, 45, special_rows=True)
    n, l = x.shape
    u = _normalized(x)
    T = int(_lib.lib().pcc_gpu_tile_count(n))
    ref = _split_packed(u, n, l)
    for cuts in ([0, 1, T], [0, T // 3, T // 2, T], list(range(T + 1))):
        assert np.array_equal(_split_packed(u, n, l, list(zip(cuts, cuts[1:]))), ref)
    d = pc.Dataset(values=x)
    for workers in (2, 3, 5):
        assert np.array_equal(pc.allpairs(d, workers=workers, **SPLIT).packed, ref)
    for chunk_rows in (1, 2, 7):
        assert np.array_equal(pc.allpairs(d, chunk_rows=chunk_rows, **SPLIT).packed, ref)
    dense, zv = pc.allpairs(d, output="dense", **SPLIT)
    iy, ix = np.triu_indices(n)
    assert np.array_equal(dense[iy, ix], ref) and np.array_equal(dense[ix, iy], ref)
    rd = pc.allpairs(d, keep_on_device=True, **SPLIT)
    assert np.array_equal(rd.packed.cpu().numpy(), ref)


def test_split_workers_pipeline_and_windows_match_single(rng, monkeypatch):
    from paper_1605_01584_b200.distributed import compute_worker, owned_runs, shard_span

    x = random_values(rng, 900, 41, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d, **SPLIT).packed
    n = x.shape[0]
    # subprocess workers on the reference's protocol (PCC_METHOD=split)
    geom = pc.TileGeometry(n=n, t=4)
    res = pc.run_workers(d, geom, 3, backend="subprocess", capacity=700, **SPLIT)
    assert np.array_equal(res.packed, ref) and res.zero_variance == frozenset({1})
    # torchrun-style compute_worker shards
    mg = -(-n // 128)
    T = mg * (mg + 1) // 2
    for p in (2, 3):
        for w in range(p):
            lo_t, hi_t = pc.partition(T, p)[w]
            lo, hi = shard_span(n, lo_t, hi_t)
            host = torch.full((max(1, hi - lo),), float("nan"), dtype=torch.float64).pin_memory()
            compute_worker(pc.Dataset(values=torch.from_numpy(x).pin_memory()), p, w, 0, out=host, **SPLIT)
            for a, b in owned_runs(n, lo_t, hi_t):
                assert np.array_equal(host[a - lo:b - lo].numpy(), ref[a:b])
    # bounded device windows
    monkeypatch.setenv("PCC_DEVICE_RESULT_BUDGET", str(8 * 60_000))
    r = pc.allpairs(d, **SPLIT)
    assert np.array_equal(r.packed, ref)


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_split_full_size_sampled_rows_and_properties(name):
    """BASELINE configs at full size (c4: l = 8,192, the split limit; c5:
    2.1e9 packed entries): sampled rows within 1e-12 of the reference's dot8,
    every coefficient in [-1-1e-12, 1+1e-12], diagonals within 1e-12 of 1."""
    x = make_config(name)
    n, l = x.shape
    d = pc.Dataset(values=torch.from_numpy(x).pin_memory())
    res = pc.allpairs(d, keep_on_device=True, **SPLIT)
    packed = res.packed
    u_ref, zv_ref = oracle.normalize(x)
    assert res.zero_variance == frozenset(np.flatnonzero(zv_ref).tolist())
    rng = np.random.default_rng(13)
    rows = sorted({0, 127, 128, n // 2, n - 129, n - 1, *rng.integers(0, n, 4).tolist()})
    ref_rows = oracle.packed_rows(u_ref, rows)
    worst = 0.0
    for y in rows:
        lo = (y * (2 * n + 1 - y)) // 2
        worst = max(worst, float(np.abs(packed[lo:lo + n - y].cpu().numpy() - ref_rows[y]).max()))
    assert worst <= TOL, f"{name}: max dev {worst:.3e}"
    assert float(packed.min()) >= -1.0 - 1e-12 and float(packed.max()) <= 1.0 + 1e-12
    ys = torch.arange(n, device=packed.device, dtype=torch.int64)
    assert float((packed[(ys * (2 * n + 1 - ys)) // 2] - 1.0).abs().max()) <= 1e-12
    del packed, res
    torch.cuda.empty_cache()


def test_split_full_c2_vs_fp64_tensor_path():
    """Whole c2 packed result (1.3e8 coefficients): split vs the FP64 tensor
    path, both within 1e-12 of the reference, so within 2e-12 of each other
    -- observed ~6e-15."""
    x = make_config("c2")
    d = pc.Dataset(values=torch.from_numpy(x).pin_memory())
    a = pc.allpairs(d, keep_on_device=True, **SPLIT).packed
    b = pc.allpairs(d, keep_on_device=True).packed
    assert float((a - b).abs().max()) <= 2e-14
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("l", [96, 128, 192, 320])
def test_split_many_tiles_per_cta_short_k_vs_oracle(l):
    """More tiles than resident CTAs (each CTA walks 2-3 tiles) with 2-5 K
    blocks: a ring stage is reused by passes that load different numbers of
    digit slices, so every slice barrier must advance in step with its stage
    (regression: the unused slices' barriers fell a phase behind)."""
    r = np.random.default_rng(l)
    n = 128 * 25 + 7  # 26 tile rows: 351 GPU tiles
    x = r.standard_normal((n, l))
    x[300:340, 3] += 300.0  # one tile row at full depth: both pass-1 slice counts
    ref, _ = oracle.allpairs(x, t=4)
    got = pc.allpairs(pc.Dataset(values=x), **SPLIT).packed
    assert float(np.abs(got - ref).max()) <= TOL


def test_split_mixed_depth_tiles_vs_oracle():
    """Adaptive depth decided per tile pair: spiky rows (max|u| near 1) in one
    GPU tile row force full depth (34 products) on every tile touching it,
    the other tiles run at depth 28 -- all within 1e-12 of the reference, and
    the host replica of the decision sees both depths."""
    r = np.random.default_rng(21)
    n, l = 600, 4096
    x = r.standard_normal((n, l))
    x[256:300, 7] += 400.0  # tile row 2: one dominant sample per row
    u = _normalized(x)
    con = _lib.Contraction("split", u, n, l).prepare_all(torch.cuda.current_stream().cuda_stream)
    T = int(_lib.lib().pcc_gpu_tile_count(n))
    prod = _lib.split_products(con.scale, n, l, 0, T)
    assert 28 * T < prod < 34 * T, prod
    ref, _ = oracle.allpairs(x, t=4)
    got = pc.allpairs(pc.Dataset(values=x), **SPLIT).packed
    assert float(np.abs(got - ref).max()) <= TOL


def test_split_to_file_and_pipeline_sink(tmp_path, rng):
    """method='split' through the LPCR file writer and the reference's
    bounded pipeline into its file sink: the same bits as allpairs."""
    x = random_values(rng, 777, 29, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d, **SPLIT).packed
    zv = pc.allpairs_to_file(d, tmp_path / "s.lpcr", **SPLIT)
    back = pc.load_result(tmp_path / "s.lpcr")
    assert np.array_equal(back.packed, ref) and back.zero_variance == zv == frozenset({1})
    nd = pc.normalize(d)
    g = pc.TileGeometry(n=777, t=4)
    with pc.PackedFileWriterSink(tmp_path / "p.lpcr", g, nd.zero_variance) as sink:
        pc.run_pipeline(nd, g, pc.plan_passes(0, g.total_tiles, 5000), sink, **SPLIT)
    assert np.array_equal(pc.load_result(tmp_path / "p.lpcr").packed, ref)


@pytest.mark.parametrize("n,l", [(300, 77), (1, 2), (129, 64), (257, 8192), (1000, 1531)])
def test_fused_normaliser_writes_the_same_digit_planes(rng, n, l):
    """pcc_normalize_split_rows_f64 (K1 straight into digit planes, no U) vs
    K1 + pcc_split_rows_f64: the same flags, scales and digit bytes, pad rows
    and K padding zero; chunked calls (bottom chunk first) give the same."""
    L = _lib.lib()
    x = random_values(rng, n, l, special_rows=True)
    xd = torch.from_numpy(x).cuda()
    u = _normalized(x)
    ref = _lib.Contraction("split", u, n, l).prepare_all(torch.cuda.current_stream().cuda_stream)
    zv_ref = pc.normalize(pc.Dataset(values=x)).zero_flags
    s = torch.cuda.current_stream().cuda_stream
    for cuts in ([0, n], sorted({0, n // 3, (2 * n) // 3, n})):
        con = _lib.Contraction("split", None, n, l, device=xd.device)
        con.slices.fill_(0x55)
        con.scale.fill_(float("nan"))
        flags = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
        for lo, hi in reversed(list(zip(cuts, cuts[1:]))):
            con.normalize_split(xd, l, flags, lo, hi, s)
        torch.cuda.synchronize()
        assert torch.equal(con.slices, ref.slices)
        assert torch.equal(con.scale, ref.scale)
        assert torch.equal(flags.bool().cpu(), zv_ref.bool().cpu())
    rc = L.pcc_normalize_split_rows_f64(xd.data_ptr(), l, n, l, flags.data_ptr(), 0, n + 1, con.slices.data_ptr(),
                                        con.scale.data_ptr(), None)
    assert rc == 1
