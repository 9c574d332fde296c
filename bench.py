#!/usr/bin/env python
"""Benchmark of the all-pairs PCC hot path on B200 (BASELINE.json's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c4]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Headline workload: c4 (n = 32,768 x l = 8,192 FP64), the configuration
BASELINE.json quotes "at 1/2/4/8 GPUs" and the largest that fits one GPU;
c2 is measured beside it (``extra_configs``).

One step = one pass of the hot path over the config's synthetic dataset:
K1 normalisation of the rows this rank's tiles read + K2 symmetric
contraction of this rank's contiguous share of the GPU tile jobs
(partition(T, N), distributed.py:76-92) with the packed epilogue.  Inputs
are resident in HBM before the timed region; X and U (2.15 GB each at c4) exceed the
126 MB L2, so no flush is needed between steps.  Timing is CUDA events on
the launching stream, W untimed warm-up steps, K timed steps between
barrier+synchronize, max over ranks.  ``e2e`` times the public API
(``allpairs`` / the per-worker shard call) with the pinned-host upload of X
and the download of this rank's packed cells inside the timed region; for
N > 1 each rank uploads only its row block of X and one broadcast K1 kernel
writes the normalised rows into every rank's U over peer memory.

``--impl reference`` times the reference itself -- ``paircorr`` installed
unmodified in baseline/_ref, its stock ``allpairs`` code path (normalize +
run_pipeline over plan_passes + ResultAssembler, all host threads) -- on a
bounded tile-id prefix of the same workload, and the bit-exact C port under
oracle/ beside it.  Only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import ctypes
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

# int8 tcgen05.mma throughput on this pool's B200 (MEASURED_PEAKS.json carries
# no int8 figure).  The split contraction runs back to back inside the bench
# (a long step), so its roofline uses the SUSTAINED rate -- random operands,
# launches back to back under the power cap (tools/i8_mma.cu sustain,
# profiles/r02s2_i8_sustained.log: median 3736 TOP/s at 1541 MHz) -- and
# reports the burst figure beside it (profiles/r01_i8_mma_peak.log)
I8_PEAK_TOPS = 3736.0
I8_PEAK_BURST_TOPS = 4122.9
DEFAULT_CONFIG = "c4"  # BASELINE.json configs[3]: quoted at 1/2/4/8 GPUs, the largest single-GPU config
EXTRA_CONFIGS = "c2"  # device step also measured on these (configs[1])
REF_DIR = ROOT / "baseline" / "_ref"


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
                   help="fraction of the reference t=4 tile range in the CPU sample (default: sized by time)")
    p.add_argument("--ref-seconds", type=float, default=None,
                   help="target seconds of host work per reference-arm step (default 4; cpu_baseline 12)")
    p.add_argument("--extra-configs", default=EXTRA_CONFIGS,
                   help="comma-separated configs whose device step is measured beside the headline ('' = none)")
    p.add_argument("--u-exchange", choices=("local", "p2p"), default="local",
                   help="N > 1 device step: 'local' = each rank normalises the rows its tiles read from its "
                        "resident X; 'p2p' = each rank normalises its 1/N row block and one broadcast K1 kernel "
                        "writes it into every rank's U over peer memory")
    return p.parse_args(argv)


# --------------------------------------------------------------------------- CPU legs

def _prefix_pairs(n: int, t: int, hi: int) -> int:
    """Cells y <= x < n inside reference t x t tiles [0, hi) (whole tile rows + a partial one)."""
    from paper_1605_01584_b200.indexing import sym_job_coord

    m = -(-n // t)
    yt, xt = sym_job_coord(m, hi - 1)
    pairs = 0
    for r in range(yt + 1):
        x_last = m - 1 if r < yt else xt
        x_hi = min(n, (x_last + 1) * t)
        for ry in range(t):
            y = r * t + ry
            if y >= n:
                break
            pairs += max(0, x_hi - max(y, r * t))
    return pairs


def cpu_sample(x: np.ndarray, fraction: float, threads: int) -> dict:
    """Time the bit-exact C port of the reference (oracle/) on the host:
    normalize all rows, then compute+scatter the first ``fraction`` of the
    t=4 tile range (engine.py:46-52 with capacity = the sample)."""
    import oracle

    n, l = x.shape
    t = 4
    m = -(-n // t)
    total = m * (m + 1) // 2
    hi = max(1, int(total * fraction))
    pairs = _prefix_pairs(n, t, hi)
    t0 = time.perf_counter()
    u, _ = oracle.normalize(x, threads=threads)
    flat = oracle.compute_pass(u, t, 0, hi, threads=threads)
    packed = np.empty(n * (n + 1) // 2, dtype=np.float64)
    oracle.scatter_range(packed, flat, 0, hi, m, t, n)
    dt = time.perf_counter() - t0
    return {"pairs": pairs, "seconds": dt, "pairs_per_s": pairs / dt, "tiles": hi, "total_tiles": total}


def import_paircorr():
    """The unmodified reference package from baseline/_ref (its numba cache
    redirected out of the tree), or (None, reason)."""
    if not (REF_DIR / "paircorr" / "__init__.py").exists():
        return None, ("baseline/_ref/paircorr is not installed (python -m pip install --no-index --no-build-isolation "
                      "--no-deps --target baseline/_ref <copy of /root/reference/pkg>)")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "pcc_numba_cache"))
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import paircorr
    except Exception as exc:  # noqa: BLE001 - reported in the JSON line
        return None, f"import paircorr failed: {type(exc).__name__}: {exc}"
    return paircorr, None


class ReferenceSample:
    """``paircorr.allpairs``'s stock single-worker path (engine.py:46-52):
    ``normalize`` + ``run_pipeline(plan_passes(0, hi, default_capacity))``
    into a ``ResultAssembler``, all host threads, over the tile-id prefix
    [0, hi) of the reference's t = 4 tile matrix -- a bounded sample of the
    same workload (tile jobs are equal-cost)."""

    T = 4

    def __init__(self, pc, x: np.ndarray, threads: int):
        from paircorr.pipeline import ResultAssembler, plan_passes, run_pipeline

        self.pc, self.threads = pc, threads
        self._plan, self._run = plan_passes, run_pipeline
        # JIT warm-up on a tiny input first (as test_acceptance.py:268-272)
        pc.allpairs(pc.Dataset(np.random.default_rng(0).random((16, 16))), threads=threads)
        self.ds = pc.Dataset(values=x)
        self.n = x.shape[0]
        self.geom = pc.TileGeometry(n=self.n, t=self.T)
        self.capacity = pc.default_capacity(self.T)
        self.asm = ResultAssembler(self.geom)  # one packed result, reused by every step

    def run(self, hi: int) -> float:
        t0 = time.perf_counter()
        u = self.pc.normalize(self.ds, threads=self.threads)
        self._run(u, self.geom, self._plan(0, hi, self.capacity), self.asm, threads=self.threads)
        return time.perf_counter() - t0

    def size_for(self, seconds: float) -> int:
        """Tile prefix taking about ``seconds`` (one probe run; normalisation is a fixed cost)."""
        total = self.geom.total_tiles
        probe = max(1, min(total, total // 400))
        t_norm = self.run(1)
        t_probe = self.run(probe)
        rate = probe / max(1e-6, t_probe - t_norm)
        return int(max(1, min(total, (seconds - t_norm) * rate)))

    def describe(self, hi: int, extra: str = "") -> str:
        return (f"paircorr {getattr(self.pc, '__version__', '0.1.0')} from baseline/_ref (unmodified), stock allpairs "
                f"path: normalize all {self.n} rows + run_pipeline(plan_passes(0, {hi}, {self.capacity})) + "
                f"ResultAssembler over t=4 tiles [0, {hi}) of {self.geom.total_tiles} "
                f"({_prefix_pairs(self.n, self.T, hi)} pairs), threads={self.threads}{extra}")


def reference_baseline(x: np.ndarray, seconds: float, threads: int, reps: int = 1, warmup: int = 0) -> dict | None:
    """One timed sample (median of ``reps``) of the real reference; None if it is not installed."""
    pc, why = import_paircorr()
    if pc is None:
        return {"unavailable": why}
    rs = ReferenceSample(pc, x, threads)
    hi = rs.size_for(seconds)
    for _ in range(warmup):
        rs.run(hi)
    secs = [rs.run(hi) for _ in range(reps)]
    med = statistics.median(secs)
    pairs = _prefix_pairs(rs.n, rs.T, hi)
    return {"value": pairs / med, "unit": "pairs/s", "cores": threads, "kind": "reference",
            "seconds": med, "steps": reps, "tiles": hi,
            "sample": rs.describe(hi, f"; median of {reps} in {med:.2f} s, extrapolated as a rate")}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle
    from paper_1605_01584_b200.workloads import CONFIGS, make_config

    spec = CONFIGS[args.config]
    x = make_config(args.config)
    threads = oracle.default_threads()
    base = {
        "impl": "reference",
        "metric": "pairs_per_sec",
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": _config_dict(args.config, world),
    }
    # the bit-exact C port beside it (oracle/; ~2.9x faster than numba paircorr)
    frac = args.cpu_fraction or _default_ref_fraction(args.config)
    port = cpu_sample(x, frac, threads)
    port_line = {"value": port["pairs_per_s"], "unit": "pairs/s", "cores": threads, "kind": "port",
                 "sample": f"bit-exact C port (oracle/): normalize + t=4 tiles [0, {port['tiles']}) of "
                           f"{port['total_tiles']} = {port['pairs']} pairs in {port['seconds']:.2f} s"}
    pc, why = import_paircorr()
    if pc is None:
        # fall back to the port as the timed reference implementation
        value = port["pairs_per_s"]
        line = dict(base, value=value, ms_per_step=port["seconds"] * 1e3,
                    gflops=2.0 * spec.l * port["pairs"] / port["seconds"] / 1e9,
                    cpu_baseline=dict(port_line), reference_unavailable=why)
    else:
        rs = ReferenceSample(pc, x, threads)
        hi = rs.size_for(args.ref_seconds or 4.0)
        for _ in range(args.warmup):
            rs.run(max(1, hi // 8))
        secs = [rs.run(hi) for _ in range(args.steps)]
        med = statistics.median(secs)
        pairs = _prefix_pairs(rs.n, rs.T, hi)
        value = pairs / med
        line = dict(base, value=value, ms_per_step=med * 1e3, gflops=2.0 * spec.l * pairs / med / 1e9,
                    cpu_baseline={"value": value, "unit": "pairs/s", "cores": threads, "kind": "reference",
                                  "sample": rs.describe(hi, f"; median of {len(secs)} steps")},
                    port_baseline=port_line)
    line["e2e"] = {"value": line["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def _default_ref_fraction(cfg: str) -> float:
    # ~3-10 s of 16-thread work for the C port
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
        "l2_policy": (f"inputs larger than L2 (X and U {spec.n * spec.l * 8 / 1e6:.0f} MB each vs 126 MB L2); no flush"
                      if spec.n * spec.l * 8 > 126e6 else
                      f"X and U ({spec.n * spec.l * 8 / 1e6:.0f} MB each) fit the 126 MB L2; small-config figure only"),
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


def _device_exchange_label(mode: str) -> str:
    if mode == "local":
        return ("local: X resident on every rank (the reference's worker model, worker.py:68-80); each rank "
                "normalises exactly the rows its tile range reads (rank 0: all), no collective")
    return ("p2p: each rank normalises its 1/N row block; one broadcast K1 kernel stores it into every rank's U "
            "over CUDA IPC peer mappings (NVLink), then a barrier")


def _device_step_config(cfg: str, rank: int, world: int, dev, args, barrier, max_over_ranks, peak: float) -> dict:
    """Device step (K1 of the rows this rank reads + K2 of its tile share) of
    another BASELINE config, timed like the headline: K steps between
    barrier + synchronize, CUDA events, max over ranks."""
    import torch

    from paper_1605_01584_b200 import _lib
    from paper_1605_01584_b200._device import ptr, stream_handle
    from paper_1605_01584_b200.distributed import owned_runs, partition, shard_span
    from paper_1605_01584_b200.indexing import sym_job_coord
    from paper_1605_01584_b200.workloads import CONFIGS, make_config

    L = _lib.lib()
    spec = CONFIGS[cfg]
    n, l = spec.n, spec.l
    x = torch.from_numpy(make_config(cfg)).to(dev)
    T = int(L.pcc_gpu_tile_count(n))
    tb, te = partition(T, world)[rank]
    lo, hi = shard_span(n, tb, te)
    shard = torch.empty(max(1, hi - lo), dtype=torch.float64, device=dev)
    cells = sum(b - a for a, b in owned_runs(n, tb, te))
    ldu, rows_pad = int(L.pcc_ldu(l)), int(L.pcc_rows_padded(n))
    u = torch.empty((rows_pad, ldu), dtype=torch.float64, device=dev)
    flags = torch.zeros(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    s = stream_handle(stream)
    _lib.check(L.pcc_zero_rows_f64(ptr(u), ldu, n, rows_pad, s), "pad rows")
    need_lo = (sym_job_coord(-(-n // _lib.GPU_TILE), tb)[0] * _lib.GPU_TILE) if te > tb else n

    def step(ev=None):
        if need_lo < n:
            _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(u), ldu, ptr(flags), l, need_lo, n, s), "normalize")
        if ev is not None:
            ev[0].record(stream)
        if te > tb:
            _lib.check(L.pcc_syrk_f64(ptr(u), n, l, ldu, tb, te, _lib.LAYOUT_PACKED, ptr(shard), 0, lo, 0, 0, 0, s),
                       "syrk")
        if ev is not None:
            ev[1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)
    syrk_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps if te > tb else 0.0
    ach = 2.0 * l * cells / (syrk_ms * 1e-3) / 1e12 if syrk_ms > 0 else 0.0
    total = n * (n + 1) // 2
    return {"workload": f"{cfg}: n={n} x l={l} FP64, {spec.description}", "value": total / (ms * 1e-3),
            "unit": "pairs/s", "ms_per_step": ms, "steps": args.steps,
            "gflops": float(n) * n * l / (ms * 1e-3) / 1e9, "syrk_ms": max_over_ranks(syrk_ms),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak if peak else None, "traffic": _load_traffic(cfg)}}


# --------------------------------------------------------------------------- GPU leg

def run_b200(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_1605_01584_b200 as pc
    from paper_1605_01584_b200 import _lib
    from paper_1605_01584_b200._device import ptr, stream_handle
    from paper_1605_01584_b200.distributed import partition, shard_span, owned_runs, compute_worker, row_slices
    from paper_1605_01584_b200.indexing import sym_job_coord
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
    ldu = int(L.pcc_ldu(l))
    rows_pad = int(L.pcc_rows_padded(n))

    # K1 of the device step.  N = 1, or --u-exchange local: this rank
    # normalises, from its resident X, exactly the rows its tile range reads
    # (tile rows >= its first one; rank 0 reads all of them).  --u-exchange
    # p2p: this rank normalises only its 1/N row block and one broadcast K1
    # kernel stores the rows into every rank's U over peer memory (CUDA IPC
    # mappings opened once, before the timed region), then a barrier.
    exchange_mode = "local" if world == 1 else args.u_exchange
    peers_opened = 0
    need_lo = (sym_job_coord(-(-n // _lib.GPU_TILE), tb)[0] * _lib.GPU_TILE) if te > tb else n
    if exchange_mode == "local":
        u_dev = torch.empty((rows_pad, ldu), dtype=torch.float64, device=dev)
        flags_dev = torch.zeros(n, dtype=torch.uint8, device=dev)
        _lib.check(L.pcc_zero_rows_f64(ptr(u_dev), ldu, n, rows_pad, s), "pad rows")
        k1_rows = n - need_lo

        def k1():
            if need_lo < n:
                _lib.check(L.pcc_normalize_rows_f64(ptr(x), l, ptr(u_dev), ldu, ptr(flags_dev), l, need_lo, n, s),
                           "normalize")
    else:
        slices, S = row_slices(n, world)
        r0, r1 = slices[rank]
        k1_rows = r1 - r0
        ubuf = _lib.DeviceBuffer(world * S * ldu * 8)
        fbuf = _lib.DeviceBuffer(world * S)
        u_dev = ubuf.tensor((world * S, ldu), "<f8")
        flags_dev = fbuf.tensor((world * S,), "|u1")
        _lib.check(L.pcc_zero_rows_f64(ptr(u_dev), ldu, n, world * S, s), "pad rows")
        flags_dev.zero_()
        handles = [None] * world
        dist.all_gather_object(handles, (ubuf.ipc_handle(), fbuf.ipc_handle()))
        peer_bufs = {q: (_lib.DeviceBuffer(handle=hu), _lib.DeviceBuffer(handle=hf))
                     for q, (hu, hf) in enumerate(handles) if q != rank}
        peers_opened = 2 * len(peer_bufs)
        torch.cuda.synchronize()
        dist.barrier()
        us = [ubuf.address if q == rank else peer_bufs[q][0].address for q in range(world)]
        fs = [fbuf.address if q == rank else peer_bufs[q][1].address for q in range(world)]
        uarr = (ctypes.c_void_p * world)(*[a + 8 * r0 * ldu for a in us])
        farr = (ctypes.c_void_p * world)(*[a + r0 for a in fs])

        def k1():
            if r1 > r0:
                _lib.check(L.pcc_normalize_rows_bcast_f64(ptr(x) + 8 * r0 * l, l, uarr, farr, world, ldu, l, 0,
                                                          r1 - r0, s), "normalize+broadcast")
            stream.synchronize()
            dist.barrier()  # every rank's rows have landed in every U

    def step(ev_pair=None):
        k1()
        if ev_pair is not None:
            ev_pair[0].record(stream)
        if te > tb:
            _lib.check(L.pcc_syrk_f64(ptr(u_dev), n, l, ldu, tb, te, _lib.LAYOUT_PACKED, ptr(shard), 0,
                                      span_lo, 0, 0, 0, s), "syrk")
        if ev_pair is not None:
            ev_pair[1].record(stream)
        return u_dev, flags_dev

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
    with ClockSampler(dev_index) as clocks_e2e:
        for _ in range(e2e_steps):
            torch.cuda.synchronize()
            barrier()
            a = time.perf_counter()
            r = api_call()
            wall.append(time.perf_counter() - a)
    e2e_s = max_over_ranks(statistics.median(wall))
    clock_e2e = clocks_e2e.summary()
    if world == 1:
        # sanity: the API result matches the device-timed shard bit for bit
        assert np.array_equal(r.packed.numpy()[:1000], shard[:1000].cpu().numpy())
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

    # ---- bit-exact mode (allpairs(exact=True)): K1 + the dot8 contraction on the
    # FP64 CUDA cores, same shard, device-timed like the step above
    exact_mode = None
    if not args.no_exact and te > tb:
        shard_x = torch.empty_like(shard)

        def step_exact(ev=None):
            k1()
            if ev is not None:
                ev[0].record(stream)
            _lib.check(L.pcc_syrk_exact_f64(ptr(u_dev), n, l, ldu, tb, te, _lib.LAYOUT_PACKED, ptr(shard_x), 0,
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
            con.normalize_split(x, l, flags_s, need_lo, n, s)
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
                         "peak_burst": I8_PEAK_BURST_TOPS, "frac_burst": i8_ach / I8_PEAK_BURST_TOPS,
                         "kernel": "syrk_split_kernel<packed> (TMA 3-D boxes per digit slice, tcgen05.mma "
                                   "kind::i8 M128 N256/N128 K32 domino schedule, 4 s32 accumulators in TMEM, 2 K passes "
                                   "per tile, adaptive depth 34/28 products)",
                         "algorithmic_ops_per_launch": i8_ops,
                         "peak_source": "measured int8 tcgen05.mma M128 N256 K32 throughput on this pool's "
                                        "B200, random operands, sustained back to back under the power cap "
                                        "(tools/i8_mma.cu sustain, profiles/r02s2_i8_sustained.log: 1541 MHz); "
                                        "peak_burst = the best short launch (profiles/r01_i8_mma_peak.log)"},
        }
        del shard_s
        torch.cuda.synchronize()
        # the same public call with method="split"
        if True:
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

    # ---- CPU baseline (rank 0, N=1 only): the reference itself (paircorr from
    # baseline/_ref, stock allpairs path, all host threads) on a ~12 s tile
    # prefix of the same X; the bit-exact C port (oracle/) if it is absent
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        threads = oracle.default_threads()
        cpu = reference_baseline(x_host, args.ref_seconds or 12.0, threads)
        if "unavailable" in cpu:
            why = cpu["unavailable"]
            frac = args.cpu_fraction or {"c1": 1.0, "c2": 1.0, "c3": 1.0, "c4": 1 / 16, "c5": 1 / 16}[args.config]
            res = cpu_sample(x_host, frac, threads)
            cpu = {
                "value": res["pairs_per_s"], "unit": "pairs/s", "cores": threads, "kind": "port",
                "sample": (f"bit-exact C port of the reference (oracle/), {threads} threads: normalize all rows + "
                           f"t=4 tiles [0, {res['tiles']}) of {res['total_tiles']} = {res['pairs']} pairs in "
                           f"{res['seconds']:.2f} s"),
                "reference_unavailable": why,
            }

    # ---- the device step on the other BASELINE configs (same rank / world)
    extra = {}
    for cfg in [c for c in (args.extra_configs or "").split(",") if c and c != args.config]:
        extra[cfg] = _device_step_config(cfg, rank, world, dev, args, barrier, max_over_ranks, peak)

    # kernels of the timed region, all ranks: K1 + the contraction's 1-2 launches per step
    launches = args.steps * (1 + (_lib.syrk_launches(n, tb, te) if te > tb else 0))
    if world > 1:
        t = torch.tensor([float(launches)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        launches = int(t.item())
    value = total_pairs / (ms_step * 1e-3)
    rank_devices, k1_rows_all = [dev_index], [k1_rows]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (dev_index, k1_rows))
        rank_devices = [g[0] for g in gathered]
        k1_rows_all = [g[1] for g in gathered]
        if rank == 0:
            print(f"bench: world_size={world} rank devices={rank_devices} device-step U exchange={exchange_mode} "
                  f"peer mappings opened on rank 0={peers_opened}", file=sys.stderr, flush=True)
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
                           **({"u_exchange_e2e": _exchange_label(ndev, world),
                               "u_exchange_device_step": _device_exchange_label(exchange_mode),
                               "world_size": world, "rank_devices": rank_devices,
                               "peer_mappings_opened_rank0": peers_opened,
                               "k1_rows_per_rank": k1_rows_all} if world > 1 else {})),
            "gflops": float(n) * n * l / (ms_step * 1e-3) / 1e9,
            "roofline_fp64_frac_of_step": (float(n) * n * l / world / (ms_step * 1e-3) / 1e12) / peak,
            "syrk_ms": syrk_avg_ms,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": total_pairs / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                    "what": "allpairs(Dataset(pinned X), out=pinned host result): upload, K1, K2 and download "
                            "streamed and overlapped (stream.py), wall clock per call, median",
                    "clocks": clock_e2e},
            "gpu_launches": launches,
            "exact_mode": exact_mode,
            "split_mode": split_mode,
            "extra_configs": extra,
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
