"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The reference measures on UCI datasets that are not in this image (pol,
protein, 3droad, houseelectric shapes); these generators reproduce
their shapes and the distributions BASELINE.json states.  Everything is drawn
in float64 from numpy's PCG64 and rounded to float32 once, so the GPU path
and the CPU oracle see bitwise-identical inputs.  Standardisation follows the
reference's split_standardize (population std, proj/src/dataset.cpp:142-163).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass
class Problem:
    name: str
    X: np.ndarray                 # n x d float32, Fortran order
    y: Optional[np.ndarray]       # n float32
    lengthscales: np.ndarray      # constrained init / fixed values
    signal: float
    noise: float
    V: Optional[np.ndarray] = None  # n x s right-hand sides (H.V microbenchmark)


def _standardize(a):
    mu = a.mean(axis=0)
    sd = np.sqrt(((a - mu) ** 2).mean(axis=0))
    sd = np.where(sd > 0, sd, 1.0)
    return (a - mu) / sd


def _f32(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float32))


def sin_targets(X, rng, noise=0.1):
    """y = sum_j sin(2 x_j) / sqrt(d) + 0.1 eps, standardised (configs 0, 2, 4)."""
    d = X.shape[1]
    y = np.sin(2.0 * X).sum(axis=1) / np.sqrt(d) + noise * rng.standard_normal(X.shape[0])
    return _standardize(y)


def config0(n=2048, d=8, seed=0) -> Problem:
    rng = np.random.default_rng([seed, 0])
    X = _standardize(rng.standard_normal((n, d)))
    y = sin_targets(X, rng)
    return Problem("c0", _f32(X), _f32(y), np.ones(d), 1.0, 0.5)


def config1(n=13500, d=26, s=65, seed=0) -> Problem:
    """Single fused H.V microbenchmark: x~N(0,I), l log-uniform [0.5, 2], sf=1,
    sigma=0.1, V~N(0,1) n x 65."""
    rng = np.random.default_rng([seed, 1])
    X = rng.standard_normal((n, d))
    ls = np.exp(rng.uniform(np.log(0.5), np.log(2.0), d))
    V = rng.standard_normal((n, s))
    return Problem("c1", _f32(X), None, ls, 1.0, 0.1, _f32(V))


def config2(n=41157, d=9, seed=0) -> Problem:
    rng = np.random.default_rng([seed, 2])
    X = _standardize(rng.standard_normal((n, d)))
    y = sin_targets(X, rng)
    return Problem("c2", _f32(X), _f32(y), np.ones(d), 1.0, 0.5)


def config3(n=391386, d=3, seed=0) -> Problem:
    rng = np.random.default_rng([seed, 3])
    X = rng.uniform(size=(n, d))
    y = np.sin(6 * X[:, 0]) * np.cos(4 * X[:, 1]) + X[:, 2] ** 2 + 0.05 * rng.standard_normal(n)
    return Problem("c3", _f32(X), _f32(_standardize(y)), np.ones(d), 1.0, 0.5)


def config4(n=1844352, d=11, seed=0) -> Problem:
    rng = np.random.default_rng([seed, 4])
    X = rng.standard_normal((n, d))
    y = sin_targets(X, rng)
    return Problem("c4", _f32(X), _f32(y), np.ones(d), 1.0, 0.5)


CONFIGS = {"c0": config0, "c1": config1, "c2": config2, "c3": config3, "c4": config4}
