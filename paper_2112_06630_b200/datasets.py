"""Seeded synthetic stand-ins for the five BASELINE.json configs.

The reference's own benchmarks used MNIST / Audio, which are not available
here and are not reproduced; these generators follow the shapes, sizes and
value distributions BASELINE.json states.  numpy's PCG64 with a fixed seed,
so a config always yields the same array on the same numpy.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    k: int
    cap: int
    delta: float = 0.001
    seed: int = 0
    description: str = ""

    def scaled(self, n: int) -> "Config":
        return Config(self.name + f"@n={n}", n, self.d, self.k, self.cap, self.delta, self.seed,
                      self.description)


CONFIGS = {
    "C1": Config("C1", 10_000, 8, 20, 20, description="low-dim: i.i.d. U[0,1), rho=1.0"),
    "C2": Config("C2", 70_000, 784, 20, 50,
                 description="image-like: integers 0..255, ~80% zeros, nonzeros U{1..255} in a "
                             "centred 20x20 blob of a 28x28 grid"),
    "C3": Config("C3", 200_000, 128, 30, 50,
                 description="clustered: 100 isotropic Gaussians, centres N(0,10^2 I), sigma=1"),
    "C4": Config("C4", 2_000_000, 96, 10, 50,
                 description="1000 Gaussians, centres N(0,5^2 I), sigma~U[0.5,2]"),
    "C5": Config("C5", 1_000_000, 960, 20, 50,
                 description="Gamma(2,1) features, rows L2-normalised"),
}


def generate(cfg: Config, n: int | None = None) -> np.ndarray:
    """n x d float32 data for the config (n defaults to cfg.n)."""
    n = cfg.n if n is None else n
    rng = np.random.default_rng(cfg.seed)
    base = cfg.name.split("@")[0]
    if base == "C1":
        return rng.random((n, cfg.d), dtype=np.float32)
    if base == "C2":
        side = 28
        x = np.zeros((n, side, side), np.float32)
        # 20x20 blob (rows/cols 4..23); nonzero with p = 0.2*784/400 -> ~157 per row
        p = 0.2 * side * side / 400.0
        mask = rng.random((n, 20, 20)) < p
        vals = rng.integers(1, 256, size=(n, 20, 20)).astype(np.float32)
        x[:, 4:24, 4:24] = np.where(mask, vals, 0.0)
        return x.reshape(n, side * side)
    if base == "C3":
        centres = rng.normal(0.0, 10.0, size=(100, cfg.d)).astype(np.float32)
        lab = rng.integers(0, 100, size=n)
        out = rng.standard_normal((n, cfg.d), dtype=np.float32)
        out += centres[lab]
        return out
    if base == "C4":
        centres = rng.normal(0.0, 5.0, size=(1000, cfg.d)).astype(np.float32)
        sig = rng.uniform(0.5, 2.0, size=1000).astype(np.float32)
        lab = rng.integers(0, 1000, size=n)
        out = np.empty((n, cfg.d), np.float32)
        step = 1 << 18
        for s in range(0, n, step):
            e = min(n, s + step)
            z = rng.standard_normal((e - s, cfg.d), dtype=np.float32)
            out[s:e] = centres[lab[s:e]] + sig[lab[s:e], None] * z
        return out
    if base == "C5":
        out = np.empty((n, cfg.d), np.float32)
        step = 1 << 16
        for s in range(0, n, step):
            e = min(n, s + step)
            g = rng.standard_gamma(2.0, size=(e - s, cfg.d), dtype=np.float32)
            g /= np.linalg.norm(g, axis=1, keepdims=True)
            out[s:e] = g
        return out
    raise KeyError(cfg.name)


def gaussian(n: int, d: int, seed: int, centers: int = 0, spread: float = 10.0) -> np.ndarray:
    """Small test data: i.i.d. N(0,1), or a mixture of `centers` Gaussians."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d), dtype=np.float32)
    if centers:
        c = rng.normal(0.0, spread, size=(centers, d)).astype(np.float32)
        x += c[rng.integers(0, centers, size=n)]
    return x
