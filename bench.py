#!/usr/bin/env python
"""Benchmark of the all-pairs PCC hot path on B200 (BASELINE.json's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

One step = one pass of the hot path over the config's synthetic dataset:
K1 normalisation of all n rows + K2 symmetric contraction of this rank's
contiguous share of the GPU tile jobs (partition(T, N), distributed.py:76-92)
with the packed epilogue.  Inputs are resident in HBM before the timed
region; X and U (>= 537 MB at c2) exceed the 126 MB L2, so no flush is
needed between steps.  Timing is CUDA events on the launching stream, W
untimed warm-up steps, K timed steps between barrier+synchronize, max over
ranks.  ``e2e`` times the public API (``allpairs`` / the per-worker shard
call) with the pinned-host upload of X and the download of this rank's
packed cells inside the timed region; for N > 1 each rank uploads only its
row block of X and the normalised blocks are all-gathered over NCCL
(distributed.exchange_normalize) before the contraction.

``--impl reference`` times the reference algorithm's CPU implementation
(the bit-exact C port under oracle/, all host threads) on a bounded sample
of the same workload -- the reference itself is Python+numba and not
installable on the box.  Only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# best measured int8 tcgen05.mma throughput on this pool's B200 (tools/i8_mma.cu,
# profiles/r01_i8_mma_peak.log); MEASURED_PEAKS.json carries no int8 figure
I8_PEAK_TOPS = 4122.9
DEFAULT_CONFIG = "c2"  # BASELINE.json configs[1]: the single-GPU headline configuration


def _env_int(name: str, default: int) -> int:
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--config", default=DEFAULT_CONFIG, choices=("c1", "c2", "c3", "c4", "c5"))
    p.add_argument("--e2e-steps", type=int, default=None, help="timed end-to-end API calls (default: max(steps, 5)), median reported")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-exact", action="store_true", help="skip the bit-exact (dot8) mode measurement")
    p.add_argument("--no-split", action="store_true", help="skip the split-mode (int8 tensor core) measurement")
    p.add_argument("--no-pageable", action="store_true", help="skip the numpy-in / numpy-out e2e measurement")
    p.add_argument("--cpu-fraction", type=float, default=None,
                   help="fraction of the reference t=4 tile range in the CPU sample")
    return p.parse_args(argv)


# --------------------------------------------------------------------------- CPU (oracle) leg

def cpu_sample(x: np.ndarray, fraction: float, threads: int) -> dict:
    """Time the reference algorithm (bit-exact C port) on the host: normalize
    all rows, then compute+scatter the first ``fraction`` of the t=4 tile range
    (engine.py:46-52 with capacity = the sample).  Returns pairs/s."""
    import oracle
    from paper_1605_01584_b200.indexing import sym_job_coord

    n, l = x.shape
    t = 4
    m = -(-n // t)
    total = m * (m + 1) // 2
    hi = max(1, int(total * fraction))
    # cells (y <= x < n) inside tiles [0, hi): whole tile rows + a partial one
    yt, xt = sym_job_coord(m, hi - 1)
    pairs = 0
    for r in range(yt + 1):
        x_last = m - 1 if r < yt else xt
        for ry in range(t):
            y = r * t + ry
            if y >= n:
                break
            x_hi = min(n, (x_last + 1) * t)
            pairs += max(0, x_hi - max(y, r * t))
    t0 = time.perf_counter()
    u, _ = oracle.normalize(x, threads=threads)
    flat = oracle.compute_pass(u, t, 0, hi, threads=threads)
    packed = np.empty(n * (n + 1) // 2, dtype=np.float64)
    oracle.scatter_range(packed, flat, 0, hi, m, t, n)
    dt = time.perf_counter() - t0
    return {"pairs": pairs, "seconds": dt, "pairs_per_s": pairs / dt, "tiles": hi, "total_tiles": total}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle
    from paper_1605_01584_b200.workloads import CONFIGS, make_config

    spec = CONFIGS[args.config]
    x = make_config(args.config)
    threads = oracle.default_threads()
    frac = args.cpu_fraction or _default_ref_fraction(args.config)
    for _ in range(args.warmup):
        cpu_sample(x, frac / 4, threads)
    samples = [cpu_sample(x, frac, threads) for _ in range(args.steps)]
    secs = [s["seconds"] for s in samples]
    pairs = samples[0]["pairs"]
    value = pairs / statistics.median(secs)
    sample_desc = (f"normalize all {spec.n} rows + compute_tile_range/scatter_range of reference t=4 tiles "
                   f"[0, {samples[0]['tiles']}) of {samples[0]['total_tiles']} ({pairs} pairs), median of {len(secs)}")
    line = {
        "impl": "reference",
        "metric": "pairs_per_sec",
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": _config_dict(args.config, world),
        "gflops": 2.0 * spec.l * pairs / statistics.median(secs) / 1e9,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port", "sample": sample_desc},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _default_ref_fraction(cfg: str) -> float:
    # ~3 s of 16-thread CPU work per step (the whole --steps/--warmup run ends within ~1 minute)
    return {"c1": 1.0, "c2": 1 / 4, "c3": 1.0, "c4": 1 / 64, "c5": 1 / 64}[cfg]


# --------------------------------------------------------------------------- helpers

def _config_dict(cfg: str, world: int) -> dict:
    from paper_1605_01584_b200.workloads import CONFIGS

    spec = CONFIGS[cfg]
    return {
        "workload": f"{cfg}: n={spec.n} x l={spec.l} FP64, {spec.description}",
        "n": spec.n,
        "l": spec.l,
        "seed": spec.seed,
        "global_batch": spec.n,
        "parallelism": (f"tile-range partition over {world} GPU(s); device step: every rank normalises the "
                        "rows it needs from its resident X, no collective"
                        + ("; e2e: row-block upload + K1 broadcast of U over peer memory" if world > 1 else "")),
        "l2_policy": "inputs larger than L2 (X and U >= 537 MB vs 126 MB L2); no flush",
        "output": "packed upper triangle n(n+1)/2 f64, sharded per GPU range, kept on device",
    }


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                f = [c.strip() for c in line.split(",")]
                if len(f) >= 9:
                    rows.append(f)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load = [s for s in sm if mx and s > 0.3 * max(mx)] or sm
        return {
            "sm_mhz": statistics.median(load) if load else None,
            "sm_max_mhz": max(mx) if mx else None,
            "power_w_max": max(pw) if pw else None,
            "reasons": reasons,
            "samples": len(rows),
        }


def _exchange_label(ndev: int, world: int) -> str:
    ex = os.environ.get("PCC_EXCHANGE", "p2p")
    if ex == "p2p":
        return ("p2p: K1 broadcasts each rank's rows into every rank's U over peer memory (CUDA IPC"
                + (", NVLink)" if ndev >= world else "; ranks share one GPU: functional run)"))
    return "nccl all_gather_into_tensor" if ndev >= world else "gloo via host (ranks share one GPU: functional run)"


def _load_traffic(cfg: str):
    """Per-launch DRAM bytes of the contraction kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_syrk_traffic.json"
    try:
        d = json.loads(p.read_text())
        return d.get(cfg, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------------------- GPU leg

def run_b200(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_1605_01584_b200 as pc
    from paper_1605_01584_b200 import _lib
    from paper_1605_01584_b200._device import ptr, stream_handle
    from paper_1605_01584_b200.distributed import partition, shard_span, owned_runs, compute_worker
    from paper_1605_01584_b200.workloads import CONFIGS, make_config
    from paper_1605_01584_b200.transform import normalize_device

    ndev = torch.cuda.device_count()
    dev_index = local_rank % ndev  # N ranks on fewer GPUs only in functional tests
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    spec = CONFIGS[args.config]
    n, l = spec.n, spec.l
    L = _lib.lib()

    # The process group (gloo, host side) carries only the barrier and the
    # max-over-ranks timing reduction -- nothing in the data path.
    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    x_host = make_config(args.config)
    x_pinned = torch.from_numpy(x_host).pin_memory()
    x = x_pinned.to(dev)
    T = int(L.pcc_gpu_tile_count(n))
    tb, te = partition(T, world)[rank]
    span_lo, span_hi = shard_span(n, tb, te)
    shard = torch.empty(max(1, span_hi - span_lo), dtype=torch.float64, device=dev)
    my_cells = sum(hi - lo for lo, hi in owned_runs(n, tb, te))
    total_pairs = n * (n + 1) // 2
    stream = torch.cuda.current_stream()
    s = stream_handle(stream)

    def step(ev_pair=None):
        u, flags = normalize_device(x)
        if ev_pair is not None:
            ev_pair[0].record(stream)
        if te > tb:
            _lib.check(L.pcc_syrk_f64(ptr(u), n, l, u.shape[1], tb, te, _lib.LAYOUT_PACKED, ptr(shard), 0,
                                      span_lo, 0, 0, 0, s), "syrk")
        if ev_pair is not None:
            ev_pair[1].record(stream)
        return u, flags

    # warm-up (also the first-touch of the allocator)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    syrk_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clocks:
        t0.record(stream)
        for i in range(args.steps):
            step(syrk_events[i])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = t0.elapsed_time(t1)
    syrk_ms = [a.elapsed_time(b) for a, b in syrk_events]
    ms_step = max_over_ranks(elapsed_ms / args.steps)
    syrk_avg_ms = max_over_ranks(sum(syrk_ms) / len(syrk_ms)) if te > tb else 0.0
    clock = clocks.summary()

    # ---- roofline of the dominant kernel (the contraction), per launch
    peak = _lib.probe_fp64_peak()
    flops_launch = 2.0 * l * my_cells                          # algorithmic: 2 l per owned pair
    achieved = flops_launch / (sum(syrk_ms) / len(syrk_ms) * 1e-3) / 1e12 if te > tb else 0.0

    roof = {
        "bound": "tensor",
        "achieved": achieved,
        "peak": peak,
        "unit": "TFLOP/s",
        "frac": achieved / peak if peak else None,
        "traffic": _load_traffic(args.config),
        "kernel": "syrk_tma_kernel<SyrkCfg<2,4,8,4,16,6>, packed, grouped tile order> (TMA ring, DMMA.8x8x4 FP64)",
        "peak_source": "measured live: register-resident mma.sync f64 probe (pcc_probe_fp64_peak); "
                       "MEASURED_PEAKS.json has no FP64 entry",
        "algorithmic_flops_per_launch": flops_launch,
    }

    # ---- bit-exact mode (allpairs(exact=True)): K1 + the dot8 contraction on the
    # FP64 CUDA cores, same shard, device-timed like the step above
    exact_mode = None
    if not args.no_exact and te > tb:
        shard_x = torch.empty_like(shard)

        def step_exact(ev=None):
            u, _ = normalize_device(x)
            if ev is not None:
                ev[0].record(stream)
            _lib.check(L.pcc_syrk_exact_f64(ptr(u), n, l, u.shape[1], tb, te, _lib.LAYOUT_PACKED, ptr(shard_x), 0,
                                            span_lo, 0, 0, 0, s), "syrk_exact")
            if ev is not None:
                ev[1].record(stream)

        ex_steps = max(2, min(args.steps, 3))
        step_exact()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ex_steps)]
        barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(ex_steps):
            step_exact(evs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        ex_ms = max_over_ranks(t0.elapsed_time(t1) / ex_steps)
        ex_syrk_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / ex_steps)
        ex_ach = flops_launch / (ex_syrk_ms * 1e-3) / 1e12
        exact_mode = {
            "what": "allpairs(exact=True): every coefficient bit-identical to the reference's dot8 "
                    "(tests/test_gpu_parity.py::test_exact_*; full c1/c3 results hash to the reference's)",
            "value": total_pairs / (ex_ms * 1e-3), "unit": "pairs/s", "ms_per_step": ex_ms, "steps": ex_steps,
            "roofline": {"bound": "fp64_alu", "achieved": ex_ach, "peak": peak / 2, "unit": "TFLOP/s",
                         "frac": ex_ach / (peak / 2),
                         "kernel": "syrk_exact_kernel<packed> (DMUL + DADD per term, FP64 CUDA cores)",
                         "peak_source": "DMUL/DADD issue at the DFMA rate = half the DMMA probe in FLOP/s "
                                        "(tools/fp64_alu.cu)"},
        }
        torch.cuda.synchronize()
        del shard_x

    # ---- split mode (allpairs(method="split")): K1 + int8 digit planes + the
    # contraction on the int8 tensor cores, same shard, device-timed; plus its
    # own end-to-end call through the public API
    split_mode = None
    if not args.no_split and te > tb and l <= _lib.SPLIT_MAX_L:
        shard_s = torch.empty_like(shard)
        sp_state = {}

        flags_s = torch.empty(n, dtype=torch.uint8, device=dev)

        def step_split(ev=None):
            # K1 fused with the digit planes (what allpairs(method="split") runs)
            con = _lib.Contraction("split", None, n, l, device=dev)
            if ev is not None:
                ev[0].record(stream)
            con.normalize_split(x, l, flags_s, 0, n, s)
            if ev is not None:
                ev[1].record(stream)
            con.syrk(tb, te, _lib.LAYOUT_PACKED, ptr(shard_s), 0, span_lo, 0, 0, 0, s, "syrk_split")
            if ev is not None:
                ev[2].record(stream)
            sp_state["con"] = con

        sp_steps = max(3, args.steps)
        step_split()
        step_split()
        torch.cuda.synchronize()
        evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(sp_steps)]
        barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(sp_steps):
            step_split(evs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        sp_ms = max_over_ranks(t0.elapsed_time(t1) / sp_steps)
        sp_rows_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b, _ in evs) / sp_steps)
        sp_syrk_ms = max_over_ranks(sum(b.elapsed_time(c) for _, b, c in evs) / sp_steps)
        # algorithmic: 2 l ops per owned pair for each int8 digit product the
        # tile pair needs (34, or 28 where its rows allow the adaptive depth)
        products = _lib.split_products(sp_state["con"].scale, n, l, tb, te)
        i8_ops = 2.0 * l * my_cells * products / (te - tb)
        i8_peak = I8_PEAK_TOPS
        i8_ach = i8_ops / (sp_syrk_ms * 1e-3) / 1e12
        diff = float((shard_s[:max(1, span_hi - span_lo)] - shard[:max(1, span_hi - span_lo)]).abs().max())
        del sp_state["con"]
        split_mode = {
            "what": "allpairs(method='split'): Ozaki int8 digit planes on the int8 tensor cores "
                    "(tcgen05.mma kind::i8, s32 in TMEM), every coefficient within 1e-12 of the reference "
                    "(tests/test_gpu_split.py); FP64-accurate, not a reduced-precision result",
            "value": total_pairs / (sp_ms * 1e-3), "unit": "pairs/s", "ms_per_step": sp_ms, "steps": sp_steps,
            "normalize_split_ms": sp_rows_ms, "syrk_ms": sp_syrk_ms,
            "products_per_tile": products / (te - tb),
            "fp64_equivalent_tflops": flops_launch / (sp_syrk_ms * 1e-3) / 1e12,
            "max_abs_diff_vs_fp64_tensor_path": diff,
            "roofline": {"bound": "tensor", "achieved": i8_ach, "peak": i8_peak, "unit": "TOP/s",
                         "frac": i8_ach / i8_peak,
                         "kernel": "syrk_split_kernel<packed> (TMA 3-D boxes per digit slice, tcgen05.mma "
                                   "kind::i8 M128 N256/N128 K32 domino schedule, 4 s32 accumulators in TMEM, 2 K passes "
                                   "per tile, adaptive depth 34/28 products)",
                         "algorithmic_ops_per_launch": i8_ops,
                         "peak_source": "measured int8 tcgen05.mma throughput on this pool's B200 "
                                        "(tools/i8_mma.cu, profiles/r01_i8_mma_peak.log: 128x256x32 shape; "
                                        "the 128x128x32 shape this kernel issues peaks at 3180)"},
        }
        del shard_s
        torch.cuda.synchronize()

    # ---- end to end through the public API (pinned X upload + packed download inside)
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(args.steps, 5)
    host_out = torch.empty(total_pairs if world == 1 else max(1, span_hi - span_lo), dtype=torch.float64,
                           pin_memory=True)
    ds = pc.Dataset(values=x_pinned)
    if world == 1:
        def api_call():
            return pc.allpairs(ds, out=host_out)
    else:
        # U exchange for the e2e leg: by default one broadcast K1 kernel writes
        # each rank's rows into every rank's U over peer memory (CUDA IPC, NVLink
        # between GPUs); PCC_EXCHANGE=collective uses K1 + NCCL all_gather
        # instead (host-staged gloo when ranks share a GPU)
        exchange = os.environ.get("PCC_EXCHANGE", "p2p")
        if exchange == "collective" and ndev >= world:
            exch_group = dist.new_group(backend="nccl")
        else:
            exch_group = dist.group.WORLD

        def api_call():
            return compute_worker(ds, world, rank, dev, out=host_out, group=exch_group, exchange=exchange)
    api_call()  # warm-up
    barrier()
    wall = []
    for _ in range(e2e_steps):
        torch.cuda.synchronize()
        barrier()
        a = time.perf_counter()
        r = api_call()
        wall.append(time.perf_counter() - a)
    e2e_s = max_over_ranks(statistics.median(wall))
    if world == 1:
        # sanity: the API result matches the device-timed shard bit for bit
        assert np.array_equal(r.packed.numpy()[:1000], shard[:1000].cpu().numpy())
    if split_mode is not None:
        # the same public call with method="split"
        if world == 1:
            def api_split():
                return pc.allpairs(ds, out=host_out, method="split")
        else:
            def api_split():
                return compute_worker(ds, world, rank, dev, out=host_out, group=exch_group, exchange=exchange,
                                      method="split")
        api_split()
        wall_s = []
        for _ in range(e2e_steps):
            torch.cuda.synchronize()
            barrier()
            a = time.perf_counter()
            api_split()
            wall_s.append(time.perf_counter() - a)
        e2e_split = max_over_ranks(statistics.median(wall_s))
        split_mode["e2e"] = {"value": total_pairs / e2e_split, "unit": "pairs/s", "ms_per_step": e2e_split * 1e3,
                             "steps": e2e_steps, "h2d_bytes_per_step": n * l * 8, "d2h_bytes_per_step": total_pairs * 8}
    h2d = n * l * 8  # world == 1: all of X; N > 1: one row block of X per rank
    d2h = total_pairs * 8

    # ---- the reference's calling convention: plain numpy in, numpy result
    # allocated by the call (pageable memory, staged through pinned slots)
    e2e_pageable = None
    if world == 1 and not args.no_pageable:
        ds_np = pc.Dataset(values=x_host)
        pc.allpairs(ds_np)  # warm-up
        walls = []
        for _ in range(3):
            torch.cuda.synchronize()
            a = time.perf_counter()
            r_np = pc.allpairs(ds_np)
            walls.append(time.perf_counter() - a)
            del r_np
        t_np = statistics.median(walls)
        e2e_pageable = {"value": total_pairs / t_np, "unit": "pairs/s", "ms_per_step": t_np * 1e3, "steps": 3,
                        "what": "allpairs(Dataset(numpy X)) returning a freshly allocated numpy result"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        threads = oracle.default_threads()
        # ~10-30 s of host work: the whole c1/c2/c3 job, a prefix of c4/c5
        frac = args.cpu_fraction or {"c1": 1.0, "c2": 1.0, "c3": 1.0, "c4": 1 / 16, "c5": 1 / 16}[args.config]
        res = cpu_sample(x_host, frac, threads)
        cpu = {
            "value": res["pairs_per_s"],
            "unit": "pairs/s",
            "cores": threads,
            "kind": "port",
            "sample": (f"bit-exact C port of the reference (oracle/), {threads} threads: normalize all rows + "
                       f"t=4 tiles [0, {res['tiles']}) of {res['total_tiles']} = {res['pairs']} pairs in "
                       f"{res['seconds']:.2f} s"),
        }

    # kernels of the timed region, all ranks: K1 + the contraction's 1-2 launches per step
    launches = args.steps * (1 + (_lib.syrk_launches(n, tb, te) if te > tb else 0))
    if world > 1:
        t = torch.tensor([float(launches)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        launches = int(t.item())
    value = total_pairs / (ms_step * 1e-3)
    if rank == 0:
        line = {
            "metric": "pairs_per_sec",
            "value": value,
            "unit": "pairs/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": dict(_config_dict(args.config, world),
                           **({"u_exchange": _exchange_label(ndev, world)} if world > 1 else {})),
            "gflops": float(n) * n * l / (ms_step * 1e-3) / 1e9,
            "roofline_fp64_frac_of_step": (float(n) * n * l / world / (ms_step * 1e-3) / 1e12) / peak,
            "syrk_ms": syrk_avg_ms,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": total_pairs / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps},
            "gpu_launches": launches,
            "exact_mode": exact_mode,
            "split_mode": split_mode,
            "e2e_pageable": e2e_pageable,
            "clocks": clock,
        }
        print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse_args(argv)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(backend="gloo")
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
