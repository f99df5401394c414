"""Seeded synthetic data with the reference generator's stream
(datasets.py:12-44 of the reference): the same numpy default_rng calls in
the same order, so (n, n_queries, dim, clusters, seed) give identical data."""

from __future__ import annotations

import numpy as np


def gaussian_mixture(n: int, n_queries: int, dim: int, clusters: int = 32, seed: int = 0,
                     center_scale: float = 1.0, cluster_scale: float = 1.0,
                     spectrum_decay: float = 0.5, out_dtype=np.float32):
    """out_dtype=np.uint8 converts each chunk with to_u8 as it is drawn (the
    same values as converting the f32 result, without the f32 copy: 51 GB at
    100M x 128)."""
    rng = np.random.default_rng(seed)
    axis = (np.arange(dim) + 1.0) ** -float(spectrum_decay)
    centers = rng.normal(0.0, center_scale, size=(clusters, dim)) * axis

    def draw(count: int, chunk: int = 1 << 20) -> np.ndarray:
        # the normal stream is consumed in row order, so filling the output
        # chunk by chunk yields the reference's values with a bounded f64
        # working set (a 10M x 96 draw would otherwise need ~25 GB)
        which = rng.integers(0, clusters, size=count)
        out = np.empty((count, dim), out_dtype)
        for lo in range(0, count, chunk):
            hi = min(count, lo + chunk)
            noise = rng.normal(0.0, cluster_scale, size=(hi - lo, dim)) * axis
            block = (centers[which[lo:hi]] + noise).astype(np.float32)
            out[lo:hi] = to_u8(block) if out_dtype == np.uint8 else block
        return out

    base = draw(n)
    queries = draw(n_queries) if n_queries else np.zeros((0, dim), np.float32)
    return base, queries


def to_u8(x: np.ndarray, scale: float = 32.0) -> np.ndarray:
    """SURVEY.md 8(d) SIFT-shape recipe: clip(rint(32 x + 128), 0, 255)."""
    return np.clip(np.rint(scale * x + 128.0), 0, 255).astype(np.uint8)


def make_config(name: str, seed: int = 0):
    """(base, queries) of a named benchmark configuration (BASELINE.json)."""
    if name == "C1":   # 100K x 128 f32, clusters=1024
        return gaussian_mixture(100_000, 1_000, 128, clusters=1024, seed=seed)
    if name == "C2":   # SIFT1M-shape 1M x 128 u8, 10K queries
        b, q = gaussian_mixture(1_000_000, 10_000, 128, clusters=10_000, seed=seed)
        return to_u8(b), to_u8(q).astype(np.float32)
    if name == "C3":   # DEEP-shape 10M x 96 f32, 10K queries
        return gaussian_mixture(10_000_000, 10_000, 96, clusters=100_000, seed=seed)
    raise ValueError(f"unknown config {name!r}")
