"""bench.py's reference arm runs on the CPU (the reference package itself from
baseline/_ref when installed, else the bit-exact C port; all host threads):
check its JSON line carries the contract's keys, and that under torchrun
rank 0 alone reports."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(*args):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                           "--steps", "1", "--warmup", "1", "--cpu-fraction", "0.05", "--ref-seconds", "0.5", *args],
                          capture_output=True, text=True, env=dict(os.environ), cwd=ROOT, timeout=300)


def test_reference_arm_json_line():
    out = _run()
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["unit"] == "pairs/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    if line["cpu_baseline"]["kind"] == "reference":  # paircorr itself timed, the C port beside it
        assert "paircorr" in line["cpu_baseline"]["sample"] and line["port_baseline"]["kind"] == "port"
    else:
        assert "reference_unavailable" in line
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"].startswith("c1")


def test_reference_arm_under_torchrun_prints_one_line():
    """Launched like the driver's N > 1 run (torchrun, gloo on CPU here): rank 0
    alone runs the CPU reference and prints; the other rank exits 0 silently."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "1",
                          "--cpu-fraction", "0.05", "--ref-seconds", "0.5"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2
