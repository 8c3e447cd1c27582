"""Shared input generators and comparison helpers for the parity tests
(the generators restate reference tests/test_support.hpp:31-45)."""
from __future__ import annotations

import numpy as np


def quantized_uniform(rng, shape, rng_range: float) -> np.ndarray:
    """Multiples of 2^-10 in [-range, range] (test_support.hpp:31-38): exact
    ties are common, x - max is exact in fp32."""
    lim = int(round(rng_range * 1024))
    return (rng.integers(-lim, lim + 1, size=shape) / 1024.0).astype(np.float32)


def normal(rng, shape, sigma: float = 1.0) -> np.ndarray:
    return (rng.standard_normal(shape) * sigma).astype(np.float32)


def dist(name: str, rng, rows: int, V: int) -> np.ndarray:
    if name == "normal":
        return normal(rng, (rows, V))
    if name == "quantized100":
        return quantized_uniform(rng, (rows, V), 100.0)
    if name == "quantized2":
        return quantized_uniform(rng, (rows, V), 2.0)  # dense ties
    if name == "equal":
        return np.full((rows, V), 1.5, np.float32)
    if name == "ascending":
        return np.tile((-10.0 + 0.125 * np.arange(V)).astype(np.float32), (rows, 1))
    if name == "descending":
        return np.tile((10.0 - 0.125 * np.arange(V)).astype(np.float32), (rows, 1))
    if name == "spikes":
        x = normal(rng, (rows, V))
        pos = rng.integers(0, V, size=(rows, 3))
        for r in range(rows):
            x[r, pos[r]] = 60.0
        return x
    if name == "wide":
        return normal(rng, (rows, V), sigma=30.0)
    raise ValueError(name)


DISTS = ["normal", "quantized100", "quantized2", "equal", "ascending", "descending", "spikes", "wide"]


def max_rel(y: np.ndarray, ref: np.ndarray, floor: float = 1e-30) -> float:
    ref = np.asarray(ref, np.float64)
    y = np.asarray(y, np.float64)
    m = ref > floor
    if not m.any():
        return 0.0
    return float(np.max(np.abs(y[m] - ref[m]) / ref[m]))
