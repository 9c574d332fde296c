"""GPU parity: the CUDA path through the C ABI vs the CPU oracle and the
reference's own golden outputs.

Tolerances: normalisation is bit-exact (same IEEE operations in the same
order, no FMA); correlations are within 1e-12 absolute per coefficient (the
north star's bound: the contraction uses FP64 FMA on the tensor pipe in a
fixed but different order than the reference's 8-lane dot8);
zero-variance rows/columns are exactly 0.0; the zero-variance set is equal.
"""

import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200 import _lib
from paper_1605_01584_b200._device import ptr, stream_handle
from paper_1605_01584_b200.workloads import make_config

from conftest import random_values

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _abi_normalize(x):
    """Call pcc_normalize_rows_f64 directly through the C ABI."""
    L = _lib.lib()
    n, l = x.shape
    xd = _dev(x)
    ldu = int(L.pcc_ldu(l))
    rows = int(L.pcc_rows_padded(n))
    u = torch.full((rows, ldu), float("nan"), dtype=torch.float64, device="cuda")
    zv = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.pcc_normalize_rows_f64(xd.data_ptr(), l, u.data_ptr(), ldu, zv.data_ptr(), l, 0, n, s))
    _lib.check(L.pcc_zero_rows_f64(u.data_ptr(), ldu, n, rows, s))
    torch.cuda.synchronize()
    return u, zv


def _abi_packed(u, n, l, tile_ranges=None):
    L = _lib.lib()
    T = int(L.pcc_gpu_tile_count(n))
    out = torch.full((n * (n + 1) // 2,), float("nan"), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for tb, te in tile_ranges or [(0, T)]:
        _lib.check(L.pcc_syrk_f64(u.data_ptr(), n, l, u.shape[1], tb, te, _lib.LAYOUT_PACKED, out.data_ptr(),
                                  0, 0, 0, 0, 0, s))
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


def test_device_info():
    info = _lib.device_info(0)
    assert info.cc_major == 10 and info.sm_count >= 100
    assert info.gpu_tile == 128 and info.syrk_ctas_per_sm >= 1


def test_normalize_bit_exact_vs_reference_golden(golden_small):
    for name, case in golden_small.items():
        x = case["x"]
        n, l = x.shape
        u, zv = _abi_normalize(x)
        uh = u.cpu().numpy()
        assert np.array_equal(uh[:n, :l], case["u"]), name
        assert np.array_equal(zv.cpu().numpy().astype(bool), case["zv"]), name
        assert (uh[:n, l:] == 0.0).all() and (uh[n:] == 0.0).all(), f"{name}: padding not zero"


def test_allpairs_vs_reference_golden(golden_small):
    for name, case in golden_small.items():
        x = case["x"]
        res = pc.allpairs(pc.Dataset(values=x))
        zv = frozenset(np.flatnonzero(case["zv"]).tolist())
        assert res.zero_variance == zv, name
        _assert_parity(res.packed, case["packed"], zv, x.shape[0])
        # also against the reference's naive definition oracle (verify's tolerance
        # is 1e-10), except where the reference engine itself departs from it
        # (subnormal-squared deviations, transform.py:23-26)
        ok = np.abs(case["packed"] - case["naive"]) <= 1e-10
        assert np.abs(res.packed - case["naive"])[ok].max(initial=0.0) <= 1e-10, name


def test_compute_pass_layout_vs_reference_golden(golden_small):
    for name, case in golden_small.items():
        x = case["x"]
        n = x.shape[0]
        nd = pc.normalize(pc.Dataset(values=x))
        geom = pc.TileGeometry(n=n, t=3)
        blocks = pc.compute_pass(nd, geom, 0, geom.total_tiles)
        flat = blocks.flat
        ref = case["pass_t3"]
        assert flat.shape == ref.shape, name
        assert np.abs(flat - ref).max(initial=0.0) <= TOL, name
        # placeholder cells (below the diagonal / past n) are exactly 0.0
        assert (flat[ref == 0.0] == 0.0).all(), name


@pytest.mark.parametrize("t", [1, 2, 3, 4, 5, 8, 16, 130])
def test_compute_pass_subranges_match_oracle(rng, t):
    x = random_values(rng, 150, 21, special_rows=True)
    nd = pc.normalize(pc.Dataset(values=x))
    u_ref, _ = oracle.normalize(x)
    geom = pc.TileGeometry(n=150, t=t)
    total = geom.total_tiles
    cuts = sorted({0, total // 3, total // 2 + 1, total - 1, total})
    for lo, hi in zip(cuts, cuts[1:]):
        got = pc.compute_pass(nd, geom, lo, hi).flat
        ref = oracle.compute_pass(u_ref, t, lo, hi)
        assert np.abs(got - ref).max(initial=0.0) <= TOL
        # exact zeros where the reference writes placeholders
        assert (got[ref == 0.0] == 0.0).all()


@pytest.mark.parametrize(
    "n,l",
    [(1, 2), (2, 2), (3, 7), (8, 8), (127, 16), (128, 17), (129, 33), (255, 15), (256, 31), (257, 64), (300, 1)],
)
def test_edge_shapes_vs_oracle(rng, n, l):
    if l < 2:
        with pytest.raises(pc.DataError):
            pc.Dataset(values=rng.random((n, l)))
        return
    x = random_values(rng, n, l, special_rows=True)
    res = pc.allpairs(pc.Dataset(values=x))
    ref, zv = oracle.allpairs(x, t=4)
    zs = frozenset(np.flatnonzero(zv).tolist())
    assert res.zero_variance == zs
    _assert_parity(res.packed, ref, zs, n)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_config_full_vs_oracle(name):
    x = make_config(name)
    n = x.shape[0]
    res = pc.allpairs(pc.Dataset(values=x))
    ref, zv = oracle.allpairs(x, t=4)
    zs = frozenset(np.flatnonzero(zv).tolist())
    assert res.zero_variance == zs
    if name == "c3":
        assert len(zs) == n // 100
    dev = np.abs(res.packed - ref)
    assert float(dev.max()) <= TOL, f"{name}: max dev {dev.max():.3e}"
    zl = np.array(sorted(zs), dtype=np.int64)
    for i in zl[:10]:
        assert res.get(int(i), int(i)) == 0.0


def test_schedule_invariance_bitwise(rng):
    x = random_values(rng, 700, 45, special_rows=True)
    n, l = x.shape
    u, _ = _abi_normalize(x)
    T = int(_lib.lib().pcc_gpu_tile_count(n))
    ref = _abi_packed(u, n, l)
    for cuts in ([0, 1, T], [0, T // 3, T // 2, T], list(range(T + 1))):
        got = _abi_packed(u, n, l, list(zip(cuts, cuts[1:])))
        assert np.array_equal(got, ref)
    for workers in (2, 3, 5, 8):
        got = pc.allpairs(pc.Dataset(values=x), workers=workers)
        assert np.array_equal(got.packed, ref)
    for chunk_rows in (1, 2, 7):
        got = pc.allpairs(pc.Dataset(values=x), chunk_rows=chunk_rows)
        assert np.array_equal(got.packed, ref)
    for t in (1, 4, 16):
        got = pc.allpairs(pc.Dataset(values=x), tile_size=t, threads=3)
        assert np.array_equal(got.packed, ref)


def test_dense_layout_matches_packed(rng):
    x = random_values(rng, 260, 19, special_rows=True)
    res = pc.allpairs(pc.Dataset(values=x))
    dense, zv = pc.allpairs(pc.Dataset(values=x), output="dense")
    assert zv == res.zero_variance
    assert np.array_equal(dense, res.to_dense())


def test_keep_on_device_and_pinned_out(rng):
    x = random_values(rng, 200, 40, special_rows=True)
    ref = pc.allpairs(pc.Dataset(values=x)).packed
    dres = pc.allpairs(pc.Dataset(values=x), keep_on_device=True)
    assert isinstance(dres.packed, torch.Tensor) and dres.packed.is_cuda
    assert np.array_equal(dres.packed.cpu().numpy(), ref)
    pinned = torch.empty(ref.size, dtype=torch.float64, pin_memory=True)
    xp = torch.from_numpy(x).pin_memory()
    r2 = pc.allpairs(pc.Dataset(values=xp), out=pinned)
    assert r2.packed is pinned
    assert np.array_equal(pinned.numpy(), ref)


def test_device_scatter_range_matches_oracle(rng):
    x = random_values(rng, 37, 11, special_rows=True)
    u, _ = oracle.normalize(x)
    t, n = 4, 37
    geom = pc.TileGeometry(n=n, t=t)
    flat = oracle.compute_pass(u, t, 0, geom.total_tiles)
    ref = np.full(n * (n + 1) // 2, np.nan)
    oracle.scatter_range(ref, flat, 0, geom.total_tiles, geom.m, t, n)
    got = pc.CorrelationResult(n=n, packed=torch.full((ref.size,), float("nan"), dtype=torch.float64, device="cuda"))
    pc.scatter_pass(pc.BlockList([pc.TileBlock(j, flat[j * 16:(j + 1) * 16]) for j in range(geom.total_tiles)]),
                    geom, got)
    assert np.array_equal(got.packed.cpu().numpy(), ref)


def test_run_pipeline_bounded_and_equal(rng):
    x = random_values(rng, 90, 13, special_rows=True)
    d = pc.Dataset(values=x)
    nd = pc.normalize(d)
    geom = pc.TileGeometry(n=90, t=4)
    peak = {"live": 0, "max": 0}

    def alloc(k):
        peak["live"] += k
        peak["max"] = max(peak["max"], peak["live"])
        return np.empty(k)

    asm = pc.ResultAssembler(geom, nd.zero_variance)
    pc.run_pipeline(nd, geom, pc.plan_passes(0, geom.total_tiles, 17), asm, allocator=alloc)
    assert peak["max"] * 8 <= 2 * 17 * 16 * 8
    ref = pc.allpairs(d).packed
    assert np.array_equal(asm.result.packed, ref)


def test_sharded_result_gather_equals_single(rng):
    x = random_values(rng, 600, 12)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d).packed
    for p in (2, 3, 4, 7):
        sh = pc.run_workers(d, None, p, gather=False)
        assert len(sh.shards) == p
        assert np.array_equal(sh.gather().packed, ref)


def test_errors_are_loud():
    L = _lib.lib()
    with pytest.raises(ValueError):
        _lib.check(L.pcc_syrk_f64(None, 10, 5, 16, 0, 1, 0, None, 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError):
        _lib.check(L.pcc_normalize_rows_f64(None, 1, None, 1, None, 1, 0, 1, None))
    u = torch.zeros((128, 32), dtype=torch.float64, device="cuda")
    out = torch.zeros(55, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="tile range"):  # tile range past the end
        _lib.check(L.pcc_syrk_f64(u.data_ptr(), 10, 5, 32, 0, 2, 0, out.data_ptr(), 0, 0, 0, 0, 0, None))
    with pytest.raises(ValueError, match="tile range"):  # reference tile range past the end
        _lib.check(L.pcc_compute_pass_f64(u.data_ptr(), 10, 5, 32, 4, 0, 7, out.data_ptr(), None))
    with pytest.raises(ValueError, match="variant"):
        _lib.check(L.pcc_syrk_f64_variant(99, u.data_ptr(), 10, 5, 32, 0, 1, 0, out.data_ptr(), 0, 0, 0, 0, 0, None))


def test_fp64_probe_reports_plausible_peak():
    tf = _lib.probe_fp64_peak()
    assert 10.0 < tf < 80.0


def test_compute_worker_streamed_shards_match_single(rng):
    from paper_1605_01584_b200.distributed import compute_worker, owned_runs, shard_span

    x = random_values(rng, 1100, 23, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d).packed
    n = x.shape[0]
    mg = -(-n // 128)
    T = mg * (mg + 1) // 2
    for p in (1, 2, 3, 5):
        for w in range(p):
            lo_t, hi_t = pc.partition(T, p)[w]
            lo, hi = shard_span(n, lo_t, hi_t)
            host = torch.full((max(1, hi - lo),), float("nan"), dtype=torch.float64).pin_memory()
            sh = compute_worker(pc.Dataset(values=torch.from_numpy(x).pin_memory()), p, w, 0, out=host)
            for a, b in owned_runs(n, lo_t, hi_t):
                assert np.array_equal(host[a - lo:b - lo].numpy(), ref[a:b])
                assert np.array_equal(sh.values[a - lo:b - lo].cpu().numpy(), ref[a:b])
            if w == 0:
                assert sh.zero_variance == frozenset({1})


def _exchange_rank(rank, world, port, x, q, exchange="collective", method="tensor"):
    import os

    import torch.distributed as dist

    from paper_1605_01584_b200.distributed import compute_worker, owned_runs, partition, shard_span

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = x.shape[0]
        mg = -(-n // 128)
        lo_t, hi_t = partition(mg * (mg + 1) // 2, world)[rank]
        lo, hi = shard_span(n, lo_t, hi_t)
        host = torch.full((max(1, hi - lo),), float("nan"), dtype=torch.float64).pin_memory()
        ds = pc.Dataset(values=torch.from_numpy(x).pin_memory())
        sh = compute_worker(ds, world, rank, 0, out=host, group=dist.group.WORLD, exchange=exchange, method=method)
        first = host.clone()
        # a second call reuses the cached exchange buffers / peer mappings (p2p)
        host.fill_(float("nan"))
        sh = compute_worker(ds, world, rank, 0, out=host, group=dist.group.WORLD, exchange=exchange, method=method)
        runs = owned_runs(n, lo_t, hi_t)
        same = all(torch.equal(first[a - lo:b - lo], host[a - lo:b - lo]) for a, b in runs)
        q.put((rank, [(a, b, host[a - lo:b - lo].numpy().copy()) for a, b in runs], sorted(sh.zero_variance), same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange,method", [("collective", "tensor"), ("p2p", "tensor"), ("p2p", "split")])
@pytest.mark.parametrize("world,n,l", [(2, 1100, 23), (3, 700, 40), (3, 200, 9)])
def test_exchange_mode_workers_match_single(world, n, l, exchange, method):
    """compute_worker(group=...): row-block upload + K1 per rank, U all-gathered
    (here over gloo: the ranks share this box's one GPU, each rank's kernels
    independent), then each rank's contraction -- reassembled bit for bit
    equal to the CPU oracle's packed result, zero-variance set complete on
    every rank."""
    import socket

    import torch.multiprocessing as mp

    x = random_values(np.random.default_rng(11), n, l, special_rows=True)
    ref, zv = oracle.allpairs(x, t=4)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_rank, args=(r, world, port, x, q, exchange, method)) for r in range(world)]
    for p_ in procs:
        p_.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    packed = np.full(ref.size, np.nan)
    for _, runs, zvs, same in got:
        assert same, "second exchange call differs from the first"
        assert zvs == sorted(np.flatnonzero(zv).tolist())
        for a, b, v in runs:
            packed[a:b] = v
    assert np.max(np.abs(packed - ref)) <= 1e-12
    assert np.array_equal(packed, pc.allpairs(pc.Dataset(values=x), method=method).packed)


def test_streamed_upload_from_pageable_and_device_inputs(rng):
    x = random_values(rng, 900, 64, special_rows=True)
    ref, zv = oracle.allpairs(x, t=4)
    for values in (x, torch.from_numpy(x), torch.from_numpy(x).cuda()):
        res = pc.allpairs(pc.Dataset(values=values), chunk_rows=3)
        _assert_parity(res.packed, ref, frozenset(np.flatnonzero(zv).tolist()), 900)


@pytest.mark.parametrize("n,l", [(3, 12_801), (2, 20_000), (1, 1_000_000), (40, 12_800), (33, 4_096), (5, 8_194),
                                 (3, 16_386)])
def test_normalize_long_rows_bit_exact(n, l):
    """Rows beyond the shared-memory budget take the chunked kernel (even l,
    aligned rows) or the three-pass global kernel (odd l); every path must
    equal the reference's normalize_rows bit for bit (the reference tests a
    10^6-sample row, test_transform.py:91-97)."""
    rng = np.random.default_rng(l)
    x = rng.random((n, l))
    if n > 1:
        x[1] = 0.5
    u, zv = _abi_normalize(x)
    u_ref, zv_ref = oracle.normalize(x)
    assert np.array_equal(u.cpu().numpy()[:n, :l], u_ref)
    assert np.array_equal(zv.cpu().numpy().astype(bool), zv_ref)


@pytest.mark.parametrize("l", [4096, 8192, 12_288])
def test_normalize_signed_zero_quotients_bit_exact(l):
    """Integer rows summing to exactly 0 (mean +0) with -0.0 entries: x - mean
    = -0 there, which the one-FMA-correction quotient would turn into +0, so
    those blocks must be written again with IEEE division -- staged (l = 4096)
    and chunked (l >= 8192) kernels, bit for bit with the reference."""
    rng = np.random.default_rng(l + 3)
    n = 24
    x = rng.integers(-9, 10, size=(n, l)).astype(np.float64)
    x[:, 5] = -0.0
    x[:, 77] = -0.0
    x[:, -1] -= x.sum(axis=1)  # every row sums to 0 exactly
    x[7] = -0.0  # a constant (all -0) row
    u, zv = _abi_normalize(x)
    u_ref, zv_ref = oracle.normalize(x)
    got = u.cpu().numpy()[:n, :l]
    assert np.array_equal(got.view(np.uint64), u_ref.view(np.uint64))  # signs of zeros included
    assert np.signbit(got[0, 5])
    assert np.array_equal(zv.cpu().numpy().astype(bool), zv_ref)


@pytest.mark.parametrize("l,ldx,offset", [(1531, 1531, 0), (1531, 1531, 1), (64, 65, 1), (64, 67, 0), (2, 3, 1),
                                          (3, 3, 1), (77, 80, 1), (2048, 2049, 1)])
def test_normalize_any_row_alignment_bit_exact(l, ldx, offset):
    """K1 stages rows by bulk copies of their 16-byte-aligned interior plus
    plain loads of an unaligned first / last element: rows of any length,
    any row stride and an 8-byte-misaligned base pointer (a view one element
    into a buffer), over sub-ranges of rows -- bit-exact to the reference,
    flags included, and every U row outside the range untouched."""
    rng = np.random.default_rng(l * 7 + ldx + offset)
    n = 37
    buf = rng.standard_normal(offset + n * ldx + 5)
    x = np.lib.stride_tricks.as_strided(buf[offset:], shape=(n, l), strides=(8 * ldx, 8)).copy()
    x[3] = -1.25  # a constant row
    for i in range(n):  # the same values inside the strided buffer
        buf[offset + i * ldx: offset + i * ldx + l] = x[i]
    u_ref, zv_ref = oracle.normalize(x)
    L = _lib.lib()
    bd = torch.from_numpy(buf).cuda()
    ldu = int(L.pcc_ldu(l))
    s = torch.cuda.current_stream().cuda_stream
    for lo, hi in ((0, n), (1, n - 1), (5, 6), (n - 1, n)):
        u = torch.full((n, ldu), float("nan"), dtype=torch.float64, device="cuda")
        zv = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
        _lib.check(L.pcc_normalize_rows_f64(bd.data_ptr() + 8 * offset, ldx, u.data_ptr(), ldu, zv.data_ptr(), l,
                                            lo, hi, s))
        torch.cuda.synchronize()
        got = u.cpu().numpy()
        assert np.array_equal(got[lo:hi, :l], u_ref[lo:hi]), (lo, hi)
        assert np.all(got[lo:hi, l:] == 0.0)
        assert np.isnan(got[:lo]).all() and np.isnan(got[hi:]).all()
        assert np.array_equal(zv.cpu().numpy()[lo:hi].astype(bool), zv_ref[lo:hi])


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_full_size_configs_sampled_rows_and_properties(name):
    """BASELINE configs at full size: U bit-exact; sampled packed rows (tile
    edges, first/last, random) within 1e-12 of the reference's dot8; every
    coefficient in [-1-1e-12, 1+1e-12]; every diagonal within 1e-12 of 1."""
    x = make_config(name)
    n, l = x.shape
    d = pc.Dataset(values=torch.from_numpy(x).pin_memory())
    res = pc.allpairs(d, keep_on_device=True)
    packed = res.packed
    nd = pc.normalize(d)
    u_ref, zv_ref = oracle.normalize(x)
    assert torch.equal(nd.u_device[:n, :l].cpu(), torch.from_numpy(u_ref))
    assert res.zero_variance == frozenset(np.flatnonzero(zv_ref).tolist())
    rng = np.random.default_rng(11)
    rows = sorted({0, 1, 127, 128, 129, 255, 256, n // 2, n - 129, n - 128, n - 1,
                   *rng.integers(0, n, 6).tolist()})
    ref_rows = oracle.packed_rows(u_ref, rows)
    worst = 0.0
    for y in rows:
        lo = (y * (2 * n + 1 - y)) // 2
        got = packed[lo:lo + n - y].cpu().numpy()
        worst = max(worst, float(np.abs(got - ref_rows[y]).max()))
    assert worst <= TOL, f"{name}: max dev {worst:.3e}"
    assert float(packed.min()) >= -1.0 - 1e-12 and float(packed.max()) <= 1.0 + 1e-12
    ys = torch.arange(n, device=packed.device, dtype=torch.int64)
    diag = packed[(ys * (2 * n + 1 - ys)) // 2]
    assert float((diag - 1.0).abs().max()) <= 1e-12
    del packed, res, nd
    torch.cuda.empty_cache()


def test_gpu_naive_oracle_bit_exact_vs_reference_golden(golden_small):
    """csrc/verify.cuh restates _kernels.pcc_naive_pair: the reference's own
    allpairs_naive output (golden 'naive') must be reproduced bit for bit."""
    for name, case in golden_small.items():
        d = pc.Dataset(values=case["x"])
        got = pc.naive_pairs(d).cpu().numpy()
        assert np.array_equal(got, case["naive"]), name
        assert pc.naive_zero_variance(d) == frozenset(np.flatnonzero(case["zv"]).tolist()), name


def test_verify_accepts_engine_and_catches_corruption(rng):
    x = random_values(rng, 700, 33, special_rows=True)
    d = pc.Dataset(values=x)
    res = pc.allpairs(d)
    rep = pc.verify(d, res, tolerance=1e-12)
    assert rep.ok and rep.pairs_checked == 700 * 701 // 2 and rep.max_abs_deviation <= 1e-12
    rows = pc.verify(d, res, rows=[0, 5, 699], tolerance=1e-12)
    assert rows.ok and rows.pairs_checked == 700 + 695 + 1
    bad = pc.CorrelationResult(n=700, packed=res.packed.copy(), zero_variance=res.zero_variance)
    bad.packed[pc.sym_job_id(700, 3, 400)] += 1e-9
    with pytest.raises(pc.VerificationError) as ei:
        pc.verify(d, bad, tolerance=1e-10)
    assert ei.value.report.first_bad_pair == (3, 400)
    wrong_zv = pc.CorrelationResult(n=700, packed=res.packed, zero_variance=frozenset())
    assert not pc.verify(d, wrong_zv, raise_on_failure=False).zero_variance_match


def test_verify_full_c3_against_gpu_oracle():
    """Config c3 (ragged, 1% constant rows), every one of its 50 M pairs."""
    x = make_config("c3")
    d = pc.Dataset(values=torch.from_numpy(x).pin_memory())
    res = pc.allpairs(d, keep_on_device=True)
    rep = pc.verify(d, res, tolerance=1e-12)
    assert rep.ok, rep
    assert rep.pairs_checked == x.shape[0] * (x.shape[0] + 1) // 2


def test_streaming_to_file_and_pageable_output(tmp_path, rng):
    x = random_values(rng, 777, 29, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d).packed
    zv = pc.allpairs_to_file(d, tmp_path / "r.lpcr")
    back = pc.load_result(tmp_path / "r.lpcr")
    assert np.array_equal(back.packed, ref) and back.zero_variance == zv == frozenset({1})
    assert pc.query_pair(tmp_path / "r.lpcr", 5, 700) == ref[pc.sym_job_id(777, 5, 700)]
    out = np.full(ref.size, np.nan)               # pageable caller-owned buffer
    r2 = pc.allpairs(d, out=out)
    assert r2.packed is out and np.array_equal(out, ref)
    # the reference's bounded pipeline feeding the streaming file sink
    nd = pc.normalize(d)
    g = pc.TileGeometry(n=777, t=4)
    with pc.PackedFileWriterSink(tmp_path / "p.lpcr", g, nd.zero_variance) as sink:
        pc.run_pipeline(nd, g, pc.plan_passes(0, g.total_tiles, 5000), sink)
    assert np.array_equal(pc.load_result(tmp_path / "p.lpcr").packed, ref)


def test_gpu_worker_serves_assignment_over_the_protocol(tmp_path, rng):
    import io

    from paper_1605_01584_b200 import protocol
    from paper_1605_01584_b200.worker import serve

    x = random_values(rng, 45, 13, special_rows=True)
    path = tmp_path / "d.lpcc"
    pc.save_dataset(path, pc.Dataset(values=x))
    u_ref, _ = oracle.normalize(x)
    buf = io.BytesIO()
    protocol.write_frame(buf, protocol.FRAME_ASSIGN, protocol.encode_assign(3, 40, 4, 10, str(path)))
    buf.seek(0)
    out = io.BytesIO()
    assert serve(buf, out, device=0) == 0
    out.seek(0)
    frames = []
    while (f := protocol.read_frame(out)) is not None:
        frames.append(f)
    assert [k for k, _ in frames] == [protocol.FRAME_BLOCKS] * 4 + [protocol.FRAME_DONE]
    cursor = 3
    for kind, payload in frames[:-1]:
        first, count, vals = protocol.decode_blocks(payload, 4)
        assert first == cursor
        assert np.abs(vals - oracle.compute_pass(u_ref, 4, first, first + count)).max() <= TOL
        cursor += count
    assert protocol.decode_done(frames[-1][1]) == 37


def test_subprocess_gpu_workers_match_single_engine(rng, monkeypatch):
    x = random_values(rng, 333, 21, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d).packed
    geom = pc.TileGeometry(n=333, t=4)
    for p in (1, 3):
        res = pc.run_workers(d, geom, p, backend="subprocess", capacity=700)
        assert np.array_equal(res.packed, ref) and res.zero_variance == frozenset({1})
    monkeypatch.setenv("PAIRCORR_FAIL_AFTER_PASSES", "1")
    with pytest.raises(pc.WorkerError) as ei:
        pc.run_workers(d, geom, 2, backend="subprocess", capacity=700)
    lo, hi = ei.value.unfinished_range
    assert hi - lo > 0 and ei.value.worker_index in (0, 1)


def test_allpairs_backend_subprocess_routes_to_worker_processes(rng, monkeypatch):
    """allpairs(..., backend="subprocess") runs GPU worker processes on the
    reference's protocol, as engine.py:46-56 routes it: same bits as the
    in-process engine, and PAIRCORR_FAIL_AFTER_PASSES reaches the workers
    through the drop-in entry point (WorkerError with the unfinished range)."""
    x = random_values(rng, 300, 20, special_rows=True)
    d = pc.Dataset(values=x)
    ref = pc.allpairs(d)
    for workers in (1, 2):
        got = pc.allpairs(d, workers=workers, backend="subprocess", capacity=500, threads=2)
        assert np.array_equal(got.packed, ref.packed) and got.zero_variance == ref.zero_variance
    monkeypatch.setenv("PAIRCORR_FAIL_AFTER_PASSES", "1")
    with pytest.raises(pc.WorkerError) as ei:
        pc.allpairs(d, workers=2, backend="subprocess", capacity=500)
    lo, hi = ei.value.unfinished_range
    assert hi > lo and ei.value.worker_index in (0, 1)


@pytest.mark.parametrize("method", ["tensor", "split", "exact"])
def test_run_workers_device_slots_exchange_bitwise(rng, method):
    """In-process multi-device workers: each device slot uploads only its row
    block of X and one broadcast K1 kernel writes the normalised rows into
    every slot's U (distributed.normalize_on_devices; peer stores over NVLink
    between GPUs, local stores when slots share a GPU, as here) -- every
    coefficient bitwise equal to the single-device engine."""
    x = random_values(rng, 700, 45, special_rows=True)
    ref = pc.allpairs(pc.Dataset(values=x), method=method)
    for devs, p in (([0, 0], 2), ([0, 0, 0], 5), ([0], 3)):
        for values in (x, torch.from_numpy(x).pin_memory(), torch.from_numpy(x).cuda()):
            got = pc.run_workers(pc.Dataset(values=values), None, p, devices=devs, method=method)
            assert np.array_equal(got.packed, ref.packed), (devs, p, method)
            assert got.zero_variance == ref.zero_variance == frozenset({1})
    n_dev = torch.cuda.device_count()
    if n_dev >= 2:  # the real multi-GPU path: peer access + per-device kernel setup
        got = pc.allpairs(pc.Dataset(values=x), devices=2, method=method)
        assert np.array_equal(got.packed, ref.packed)


def test_normalize_on_devices_rows_bit_exact(rng):
    from paper_1605_01584_b200.distributed import normalize_on_devices

    x = random_values(rng, 1100, 33, special_rows=True)
    u_ref, zv_ref = oracle.normalize(x)
    outs = normalize_on_devices(x, 1100, 33, [torch.device("cuda", 0)] * 3)
    assert len(outs) == 3
    for u, flags in outs:
        assert np.array_equal(u[:1100, :33].cpu().numpy(), u_ref)
        assert float(u[1100:].abs().max()) == 0.0 and float(u[:, 33:].abs().max()) == 0.0
        assert np.array_equal(flags[:1100].cpu().numpy().astype(bool), zv_ref)


def test_acceptance_criterion_2_random_datasets_vs_naive_oracle():
    """The reference's acceptance criterion 2 (test_acceptance.py:88-113):
    50 random datasets with planted constant / negated / affine rows, random
    n, l and scheduling knobs; engine vs the definition oracle <= 1e-10, equal
    zero-variance sets -- here also <= 1e-12 vs the reference engine's order."""
    rng = np.random.default_rng(2)
    worst = 0.0
    for trial in range(50):
        n = int(rng.integers(1, 257))
        l = int(rng.integers(2, 129))
        x = random_values(rng, n, l, special_rows=True)
        t = [1, 2, 3, 4, 5, 8, 16][trial % 7]
        res = pc.allpairs(pc.Dataset(values=x), tile_size=t, threads=int(rng.integers(1, 5)),
                          chunk_rows=int(rng.integers(1, 9)))
        naive, zv = oracle.allpairs_naive(x)
        ref, _ = oracle.allpairs(x, t=4)
        worst = max(worst, float(np.abs(res.packed - naive).max()))
        assert np.abs(res.packed - ref).max() <= TOL
        assert res.zero_variance == frozenset(np.flatnonzero(zv).tolist())
    assert worst <= 1e-10


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402
from hypothesis.extra.numpy import arrays  # noqa: E402


@given(arrays(np.float64, st.tuples(st.integers(1, 5), st.integers(2, 70)),
              elements=st.floats(min_value=-1e6, max_value=1e6, allow_nan=False, width=64)))
@settings(max_examples=150, deadline=None)
def test_normalize_property_bit_exact(x):
    """Hypothesis-generated rows (the reference's test_normalize_row_invariants
    domain, test_transform.py:66-88): K1 equals the reference order bit for bit."""
    u, zv = _abi_normalize(x)
    u_ref, zv_ref = oracle.normalize(x)
    n, l = x.shape
    assert np.array_equal(u.cpu().numpy()[:n, :l], u_ref)
    assert np.array_equal(zv.cpu().numpy().astype(bool), zv_ref)


def test_syrk_launch_count_matches_tail_rule():
    info = _lib.device_info(0)
    wave = info.sm_count * info.syrk_ctas_per_sm
    for n in (16384, 10007, 2000, 129):
        T = int(_lib.lib().pcc_gpu_tile_count(n))
        tail = T % wave
        want = (1 if T > tail or tail == 0 else 0) + (1 if 0 < tail <= wave // 2 else 0)
        if tail > wave // 2:
            want = 1
        assert _lib.syrk_launches(n, 0, T) == want, n
    assert _lib.syrk_launches(16384, 5, 5) == 0
    with pytest.raises(ValueError):
        _lib.syrk_launches(100, 0, 10**6)


def test_reference_pair_helpers_match_reference_outputs():
    """pcc_naive (GPU definition kernel) and pcc_normalized (the bit-exact
    contraction on two rows) bit-identical to the reference's pcc_naive and
    pcc_normalized (tests/golden/helpers.json)."""
    import json

    from conftest import GOLDEN

    pairs = json.loads((GOLDEN / "helpers.json").read_text())["pairs"]
    for case in pairs:
        a = np.array([float.fromhex(v) for v in case["a"]])
        b = np.array([float.fromhex(v) for v in case["b"]])
        assert float(pc.pcc_naive(a, b)).hex() == case["naive"]
        u, _ = oracle.normalize(np.stack([a, b]))
        assert float(pc.pcc_normalized(u[0], u[1])).hex() == case["normalized"]
    with pytest.raises(ValueError):
        pc.pcc_naive([1.0, 2.0], [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        pc.pcc_naive([1.0], [2.0])
    with pytest.raises(ValueError):
        pc.pcc_normalized([1.0, 2.0], [1.0])


def test_allpairs_naive_bit_identical_to_reference_golden(golden_small):
    assert len(golden_small) >= 30
    for name, case in golden_small.items():
        x = case["x"]
        r = pc.allpairs_naive(pc.Dataset(values=x))
        assert np.array_equal(r.packed, case["naive"]), name
        assert r.zero_variance == frozenset(np.flatnonzero(oracle.constant_row_flags(x)).tolist())


# ---------------------------------------------------------------------------
# Exact mode: the dot8 contraction on the FP64 CUDA cores, bit-identical to
# the reference's engine (csrc/exact.cuh).

def test_exact_allpairs_bit_identical_to_reference_golden(golden_small):
    assert len(golden_small) >= 30
    for name, case in golden_small.items():
        r = pc.allpairs(pc.Dataset(values=case["x"]), exact=True)
        assert np.array_equal(r.packed.view(np.uint64), case["packed"].view(np.uint64)), name
        assert r.zero_variance == frozenset(np.flatnonzero(case["zv"]).tolist()), name


def test_exact_pass_buffers_bit_identical_to_reference(golden_small):
    """compute_pass(..., exact=True) reproduces the reference's t = 3 pass
    buffer (zeros outside the triangle included), bit for bit."""
    for name, case in golden_small.items():
        nd = pc.normalize(pc.Dataset(values=case["x"]))
        geom = pc.TileGeometry(n=nd.n, t=3)
        blocks = pc.compute_pass(nd, geom, 0, geom.total_tiles, exact=True)
        flat = blocks.flat if len(blocks) else np.empty(0)
        assert np.array_equal(np.asarray(flat).view(np.uint64), case["pass_t3"].view(np.uint64)), name


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_exact_full_config_matches_reference_sha256(cfg):
    """The whole packed result of c1 / c3 hashes to the reference's own
    (tests/golden/config_digests.json, made by running paircorr.allpairs)."""
    import hashlib
    import json

    from conftest import GOLDEN

    from paper_1605_01584_b200.workloads import make_config

    g = json.loads((GOLDEN / "config_digests.json").read_text())[cfg]
    x = make_config(cfg)
    r = pc.allpairs(pc.Dataset(values=x), exact=True)
    assert hashlib.sha256(np.ascontiguousarray(r.packed).tobytes()).hexdigest() == g["packed_sha256"]
    assert sorted(r.zero_variance) == g["zero_variance"]


@pytest.mark.parametrize("n,l", [(1, 2), (2, 3), (127, 5), (128, 8), (129, 9), (255, 31), (257, 33), (300, 77),
                                 (130, 1531), (520, 64)])
def test_exact_ragged_shapes_bit_identical_to_oracle(n, l, rng):
    x = random_values(rng, n, l, special_rows=n > 3)
    ref, zv = oracle.allpairs(x, t=4)
    r = pc.allpairs(pc.Dataset(values=x), exact=True)
    assert np.array_equal(r.packed.view(np.uint64), ref.view(np.uint64))
    dense, _ = pc.allpairs(pc.Dataset(values=x), exact=True, output="dense")
    iu = np.triu_indices(n)
    assert np.array_equal(dense[iu], ref) and np.array_equal(dense, dense.T)


def test_exact_schedule_invariance(rng):
    """Exact results do not depend on passes, workers or the streamed plan."""
    x = random_values(rng, 700, 45, special_rows=True)
    ref, _ = oracle.allpairs(x, t=4)
    d = pc.Dataset(values=x)
    for kw in ({"workers": 3}, {"chunk_rows": 1}, {"workers": 2, "devices": 1}):
        assert np.array_equal(pc.allpairs(d, exact=True, **kw).packed, ref), kw
    nd = pc.normalize(d)
    geom = pc.TileGeometry(n=700, t=4)
    asm = pc.ResultAssembler(geom, nd.zero_variance)
    pc.run_pipeline(nd, geom, pc.plan_passes(0, geom.total_tiles, 5000), asm, exact=True)
    assert np.array_equal(asm.result.packed, ref)


def test_exact_subprocess_workers_and_device_output(rng, monkeypatch):
    """PCC_EXACT workers over the reference protocol and keep_on_device: still
    the reference's bits."""
    x = random_values(rng, 260, 21, special_rows=True)
    ref, _ = oracle.allpairs(x, t=4)
    r = pc.run_workers(pc.Dataset(values=x), pc.TileGeometry(n=260, t=4), 2, backend="subprocess", exact=True)
    assert np.array_equal(r.packed, ref)
    rd = pc.allpairs(pc.Dataset(values=x), exact=True, keep_on_device=True)
    assert np.array_equal(rd.packed.cpu().numpy(), ref)


@given(st.integers(1, 400), st.integers(2, 160), st.integers(0, 2**32 - 1), st.sampled_from(["normal", "lognormal", "ints"]))
@settings(max_examples=40, deadline=None)
def test_allpairs_property_vs_oracle(n, l, seed, dist):
    """Random shapes and value distributions (incl. small integers: ties,
    constant rows, exact cancellations): the tensor path and split mode within
    1e-12 of the reference order, the exact mode bit-identical, the same
    zero-variance set."""
    r = np.random.default_rng(seed)
    x = {"normal": lambda: r.standard_normal((n, l)),
         "lognormal": lambda: r.lognormal(0.0, 2.0, (n, l)),
         "ints": lambda: r.integers(-2, 3, (n, l)).astype(np.float64)}[dist]()
    ref, zv = oracle.allpairs(x, t=4)
    d = pc.Dataset(values=x)
    fast = pc.allpairs(d)
    assert np.max(np.abs(fast.packed - ref)) <= 1e-12
    assert fast.zero_variance == frozenset(np.flatnonzero(zv).tolist())
    exact = pc.allpairs(d, exact=True)
    assert np.array_equal(exact.packed.view(np.uint64), ref.view(np.uint64))
    split = pc.allpairs(d, method="split")
    assert np.max(np.abs(split.packed - ref)) <= 1e-12
    assert split.zero_variance == fast.zero_variance


@pytest.mark.parametrize("n,l", [(300, 77), (40, 8194)])
def test_normalize_broadcast_writes_every_destination(rng, n, l):
    """pcc_normalize_rows_bcast_f64: one K1 launch stores each row into all
    destinations (the fused normalise + all-gather of the p2p exchange),
    bit-identical to the single-destination K1 -- staged rows and chunked
    rows (l >= 8192, a partial last chunk)."""
    import ctypes

    x = torch.from_numpy(random_values(rng, n, l, special_rows=True)).cuda()
    n, l = x.shape
    L = _lib.lib()
    ldu = int(L.pcc_ldu(l))
    ref_u = torch.zeros((n, ldu), dtype=torch.float64, device="cuda")
    ref_f = torch.zeros(n, dtype=torch.uint8, device="cuda")
    _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(ref_u), ldu, ptr(ref_f), l, 0, n, stream_handle()))
    us = [torch.full((n, ldu), float("nan"), dtype=torch.float64, device="cuda") for _ in range(3)]
    fs = [torch.full((n,), 7, dtype=torch.uint8, device="cuda") for _ in range(3)]
    uarr = (ctypes.c_void_p * 3)(*[ptr(t) for t in us])
    farr = (ctypes.c_void_p * 3)(*[ptr(t) for t in fs])
    _lib.check(L.pcc_normalize_rows_bcast_f64(ptr(x), l, uarr, farr, 3, ldu, l, 0, n, stream_handle()))
    torch.cuda.synchronize()
    for u_, f_ in zip(us, fs):
        assert torch.equal(u_, ref_u) and torch.equal(f_, ref_f)
    with pytest.raises(ValueError):
        _lib.check(L.pcc_normalize_rows_bcast_f64(ptr(x), l, uarr, farr, 0, ldu, l, 0, n, stream_handle()))


def test_device_buffer_ipc_roundtrip_and_lifetime():
    """DeviceBuffer: a cudaMalloc'd buffer viewed as a tensor stays alive as
    long as the view does; its IPC handle is 64 bytes."""
    import gc

    b = _lib.DeviceBuffer(1024 * 8)
    t = b.tensor((1024,), "<f8")
    assert len(b.ipc_handle()) == _lib.IPC_HANDLE_BYTES
    t.fill_(3.0)
    del b
    gc.collect()
    t.add_(1.0)
    assert float(t.sum()) == 4.0 * 1024


def test_pipeline_semantics_match_reference(rng):
    """run_pipeline behaves as the reference's (pipeline.py:109-187,
    tests/test_pipeline.py): one call per pass in plan order, capacity 1
    delivers every tile in order, an empty plan makes no sink call, overlap
    on / off gives identical bits, a failing sink raises PipelineError with
    its pass range, and two pipelines on one device do not interfere."""
    x = random_values(rng, 70, 11, special_rows=True)
    nd = pc.normalize(pc.Dataset(values=x))
    geom = pc.TileGeometry(n=70, t=4)
    T = geom.total_tiles
    ref = pc.allpairs(pc.Dataset(values=x)).packed

    class Recorder(pc.ResultSink):
        def __init__(self):
            self.calls, self.tiles, self.flat = [], [], []

        def consume(self, pass_range, blocks):
            self.calls.append(tuple(pass_range))
            self.tiles += [b.tile_id for b in blocks]
            self.flat.append(np.concatenate([b.values for b in blocks]).copy())

    r = Recorder()
    pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 1), r)
    assert r.calls == [(j, j + 1) for j in range(T)] and r.tiles == list(range(T))
    r = Recorder()
    pc.run_pipeline(nd, geom, pc.plan_passes(5, 5, 3), r)
    assert r.calls == []
    on, off = Recorder(), Recorder()
    pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 37), on, overlap=True)
    pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 37), off, overlap=False)
    assert on.calls == off.calls and all(np.array_equal(a, b) for a, b in zip(on.flat, off.flat))

    class Failing(pc.ResultSink):
        def __init__(self, at):
            self.at, self.n = at, 0

        def consume(self, pass_range, blocks):
            if self.n == self.at:
                raise RuntimeError("disk full")
            self.n += 1

    for overlap in (True, False):
        with pytest.raises(pc.PipelineError) as ei:
            pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 40), Failing(2), overlap=overlap)
        assert tuple(ei.value.pass_range) == (80, 120)
    with pytest.raises(ValueError):
        pc.run_pipeline(nd, geom, pc.plan_passes(0, T + 1, 40), Recorder())
    a1, a2 = pc.ResultAssembler(geom, nd.zero_variance), pc.ResultAssembler(geom, nd.zero_variance)
    pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 29), a1)
    pc.run_pipeline(nd, geom, pc.plan_passes(0, T, 31), a2)
    assert np.array_equal(a1.result.packed, ref) and np.array_equal(a2.result.packed, ref)


@pytest.mark.parametrize("exact", [True, False])
def test_compute_pass_tile_layout_kats(rng, exact):
    """The reference's tile-layout KATs (tests/test_tiles.py): n=2, t=2 gives
    [r00, r01, 0.0, r11]; n=3, t=2 boundary tiles hold r(y, x) for y <= x < n
    and exactly 0.0 elsewhere; an empty range gives no blocks.  Exact mode
    equals pcc_normalized bit for bit, the tensor path within 1e-12."""
    def check(v, want):
        if exact:
            assert v == want
        else:
            assert abs(v - want) <= 1e-12

    nd = pc.normalize(pc.Dataset(values=random_values(rng, 2, 6)))
    blocks = pc.compute_pass(nd, pc.TileGeometry(n=2, t=2), 0, 1, exact=exact)
    assert len(blocks) == 1
    r = lambda i, j: pc.pcc_normalized(nd.u[i], nd.u[j])  # noqa: E731
    v = blocks[0].values
    check(v[0], r(0, 0)), check(v[1], r(0, 1)), check(v[3], r(1, 1))
    assert v[2] == 0.0
    nd = pc.normalize(pc.Dataset(values=random_values(rng, 3, 7)))
    geom = pc.TileGeometry(n=3, t=2)
    blocks = pc.compute_pass(nd, geom, 0, 3, exact=exact)
    assert [b.tile_id for b in blocks] == [0, 1, 2]
    for b in blocks:
        Y, X = pc.tile_coord(geom.m, b.tile_id)
        for off in range(4):
            y, x = Y * 2 + off // 2, X * 2 + off % 2
            if y <= x < 3:
                check(b.values[off], pc.pcc_normalized(nd.u[y], nd.u[x]))
            else:
                assert b.values[off] == 0.0
    nd = pc.normalize(pc.Dataset(values=random_values(rng, 4, 5)))
    assert len(pc.compute_pass(nd, pc.TileGeometry(n=4, t=2), 2, 2, exact=exact)) == 0


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_exact_full_size_sampled_rows_bit_identical(name):
    """Exact mode at full BASELINE size (c2, c4 with l = 8,192, and c5 with
    2.1e9 packed entries = 64-bit offsets): sampled packed rows equal the
    reference's dot8 bit for bit, diagonals of non-constant rows included."""
    x = make_config(name)
    n, l = x.shape
    d = pc.Dataset(values=torch.from_numpy(x).pin_memory())
    res = pc.allpairs(d, keep_on_device=True, exact=True)
    packed = res.packed
    u_ref, _ = oracle.normalize(x)
    rng = np.random.default_rng(5)
    rows = sorted({0, 129, n // 2 + 3, n - 130, n - 1, *rng.integers(0, n, 3).tolist()})
    ref_rows = oracle.packed_rows(u_ref, rows)
    for y in rows:
        lo = (y * (2 * n + 1 - y)) // 2
        got = packed[lo:lo + n - y].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), ref_rows[y].view(np.uint64)), (name, y)
    del packed, res
    torch.cuda.empty_cache()


@pytest.mark.parametrize("exact", [False, True])
def test_windowed_allpairs_when_result_exceeds_device_budget(rng, monkeypatch, exact):
    """A packed result larger than the device budget goes through bounded
    device windows (one GPU tile pass each) -- same bits as the one-shot path."""
    x = random_values(rng, 900, 41, special_rows=True)
    ref = pc.allpairs(pc.Dataset(values=x), exact=exact)
    monkeypatch.setenv("PCC_DEVICE_RESULT_BUDGET", str(8 * 60_000))  # ~15 windows for 405,450 cells
    for out in (None, torch.empty(ref.packed.size, dtype=torch.float64).pin_memory()):
        r = pc.allpairs(pc.Dataset(values=x), exact=exact, out=out)
        got = r.packed.numpy() if isinstance(r.packed, torch.Tensor) else r.packed
        assert np.array_equal(got, ref.packed) and r.zero_variance == ref.zero_variance
