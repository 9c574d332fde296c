import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")


def triangle_walk(n):
    """Row-major enumeration of the upper triangle (the reference tests' oracle, conftest.py:7-13)."""
    return [(y, x) for y in range(n) for x in range(y, n)]


def random_values(rng, n, l, special_rows=False):
    """Uniform rows; optionally a constant, a negated and an affine row (conftest.py:16-23)."""
    values = rng.random((n, l))
    if special_rows and n >= 4:
        values[1] = 3.25
        values[2] = -values[0]
        values[3] = 2.5 * values[0] + 1.0
    return values


@pytest.fixture
def rng():
    return np.random.default_rng(20260810)


@pytest.fixture(scope="session")
def golden_small():
    z = np.load(GOLDEN / "small_cases.npz")
    names = sorted({k.split("/")[0] for k in z.files})
    return {nm: {f: z[f"{nm}/{f}"] for f in ("x", "u", "zv", "packed", "naive", "pass_t3")} for nm in names}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
