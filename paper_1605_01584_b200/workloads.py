"""Seeded synthetic datasets with the shapes of BASELINE.json's five configs.

The paper's real data (SEEK GPL570) is not available, and
BASELINE.json quotes its metric on synthetic configurations; these generators
stand in for them (SURVEY.md §8d "Per-config synthetic inputs").  Every
generator is a pure function of its seed, so the GPU path, the CPU oracle and
the golden-fixture script all see the same bytes.

``gen_synthetic`` restates the reference's counter-based splitmix64 uniform
generator (fileio.py:277-305), the generator behind the paper's artificial
uniform [0,1) datasets.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CONFIGS", "ConfigSpec", "make_config", "gen_uniform_splitmix64"]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int
    l: int
    seed: int
    description: str


CONFIGS = {
    "c1": ConfigSpec("c1", 2_000, 500, 1, "i.i.d. N(0,1)"),
    "c2": ConfigSpec("c2", 16_384, 4_096, 2, "rank-32 latent factors N(0,1) x N(0,1) + 0.5 N(0,1)"),
    "c3": ConfigSpec("c3", 10_007, 1_531, 3, "log-normal(2,1), 1% of rows constant"),
    "c4": ConfigSpec("c4", 32_768, 8_192, 4, "rank-64 latent factors + N(0,1)"),
    "c5": ConfigSpec("c5", 65_536, 2_048, 5, "N(0,1) with 256 planted blocks of 64 rows, r~0.8"),
}


def _latent(rng: np.random.Generator, n: int, l: int, rank: int, noise: float) -> np.ndarray:
    # Row-chunked so the float64 product never needs an n x l temporary
    # beyond the output itself.
    loadings = rng.standard_normal((n, rank))
    factors = rng.standard_normal((rank, l))
    x = np.empty((n, l), dtype=np.float64)
    step = 4096
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        np.matmul(loadings[lo:hi], factors, out=x[lo:hi])
        x[lo:hi] += noise * rng.standard_normal((hi - lo, l))
    return x


def make_config(name: str, n: int | None = None, l: int | None = None, seed: int | None = None) -> np.ndarray:
    """Return the C-contiguous float64 n x l matrix of config ``name``.

    ``n``/``l``/``seed`` override the config's shape (same value
    distribution) for reduced-size parity cases.
    """
    spec = CONFIGS[name]
    n = spec.n if n is None else n
    l = spec.l if l is None else l
    rng = np.random.default_rng(spec.seed if seed is None else seed)
    if name == "c1":
        return rng.standard_normal((n, l))
    if name == "c2":
        return _latent(rng, n, l, 32, 0.5)
    if name == "c3":
        x = rng.lognormal(2.0, 1.0, (n, l))
        k = max(1, n // 100)
        rows = rng.choice(n, k, replace=False)
        x[rows] = rng.lognormal(2.0, 1.0, k)[:, None]
        return x
    if name == "c4":
        return _latent(rng, n, l, 64, 1.0)
    if name == "c5":
        x = rng.standard_normal((n, l))
        blocks, rows_per = 256, 64
        if n < blocks * rows_per:
            blocks = n // rows_per
        order = rng.permutation(n)[: blocks * rows_per].reshape(blocks, rows_per)
        f = rng.standard_normal((blocks, l))
        for b in range(blocks):
            x[order[b]] = np.sqrt(0.8) * f[b] + np.sqrt(0.2) * rng.standard_normal((rows_per, l))
        return x
    raise KeyError(name)


_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def gen_uniform_splitmix64(n: int, l: int, seed: int = 0) -> np.ndarray:
    """Uniform [0,1) values, element (r, c) = splitmix64(seed + (r*l+c+1)*golden) >> 11 * 2^-53.

    Restates fileio.py:277-305 (the reference's ``gen_synthetic``).
    """
    if n < 1 or l < 1:
        raise ValueError(f"n and l must be >= 1, got n={n}, l={l}")
    with np.errstate(over="ignore"):
        idx = np.arange(1, n * l + 1, dtype=np.uint64)
        x = np.uint64(seed % 2**64) + idx * _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _MIX1
        x = (x ^ (x >> np.uint64(27))) * _MIX2
        x = x ^ (x >> np.uint64(31))
    return ((x >> np.uint64(11)).astype(np.float64) * 2.0**-53).reshape(n, l)
